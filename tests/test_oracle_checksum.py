"""Pins for oracle.checksum (reading R14): closed forms, pure-Python brute force
(arbitrary-precision ints reduced mod 2^64, no NumPy wrap-around), additivity
over partitions, and detection of single-element changes and swaps."""
import numpy as np

from oracle import plex_oracle as O

M = 1 << 64


def _brute(bits, base):
    s1 = s2 = 0
    for j, b in enumerate(bits.tolist()):
        s1 += b
        s2 += (base + j + 1) * b
    return s1 % M, s2 % M


def test_closed_form_constant():
    for n, b, dt in ((1000, 0xFFFF, np.uint16), (777, 0xFFFFFFFF, np.uint32), (5, 3, np.uint32)):
        x = np.full(n, b, dtype=dt)
        assert O.checksum(x) == ((n * b) % M, (b * n * (n + 1) // 2) % M)


def test_brute_force():
    rng = np.random.default_rng(0)
    for dt, hi in ((np.uint16, 1 << 16), (np.uint32, 1 << 32)):
        x = rng.integers(0, hi, size=3001, dtype=np.uint64).astype(dt)
        for base in (0, 17, (1 << 32) - 5000):
            assert O.checksum(x, base) == _brute(x, base)


def test_additive_over_partitions():
    rng = np.random.default_rng(1)
    x = rng.integers(0, 1 << 32, size=10_000, dtype=np.uint64).astype(np.uint32)
    full = O.checksum(x)
    cuts = sorted(rng.choice(np.arange(1, x.size), size=37, replace=False).tolist())
    s1 = s2 = 0
    for a, b in zip([0] + cuts, cuts + [x.size]):
        c = O.checksum(x[a:b], a)
        s1, s2 = (s1 + c[0]) % M, (s2 + c[1]) % M
    assert (s1, s2) == full


def test_detects_changes_and_swaps():
    rng = np.random.default_rng(2)
    x = rng.integers(0, 1 << 16, size=4096, dtype=np.uint64).astype(np.uint16)
    c = O.checksum(x)
    for _ in range(200):
        y = x.copy()
        i = rng.integers(0, x.size)
        y[i] ^= np.uint16(1 << rng.integers(0, 16))
        assert O.checksum(y) != c
        i, j = rng.choice(x.size, size=2, replace=False)
        if x[i] != x[j]:
            y = x.copy()
            y[i], y[j] = x[j], x[i]
            assert O.checksum(y)[0] == c[0] and O.checksum(y) != c
