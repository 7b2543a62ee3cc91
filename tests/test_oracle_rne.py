"""Pins for oracle.rne_bf16 (a8/o6, reading R8) against things other than itself:
the golden Appendix C table, torch's CPU fp32->bf16 conversion (a library
routine implementing IEEE RNE), and the textbook nearest-value definition
evaluated in exact float64 arithmetic."""
import os

import numpy as np
import pytest
import torch

from oracle import plex_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "rne_specials.txt")


def _golden():
    rows = []
    for ln in open(GOLD):
        ln = ln.strip()
        if not ln or ln.startswith("#"):
            continue
        a, b = ln.split()[:2]
        rows.append((int(a, 16), int(b, 16)))
    return rows


def test_golden_table():
    rows = _golden()
    u = np.array([a for a, _ in rows], dtype=np.uint32)
    want = np.array([b for _, b in rows], dtype=np.uint16)
    assert np.array_equal(O.rne_bf16(u), want)


def _torch_bf16_bits(u: np.ndarray) -> np.ndarray:
    t = torch.from_numpy(u.view(np.float32).copy()).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16)


def _is_nan(u):
    return ((u & 0x7F800000) == 0x7F800000) & ((u & 0x7FFFFF) != 0)


def test_vs_torch_all_high_halves():
    # every one of the 65536 high halves x the rounding-critical low halves
    hi = np.arange(1 << 16, dtype=np.uint32) << np.uint32(16)
    lows = np.array([0, 1, 0x7FFF, 0x8000, 0x8001, 0xFFFF, 0x1234, 0xC000], dtype=np.uint32)
    u = (hi[:, None] | lows[None, :]).reshape(-1)
    u = u[~_is_nan(u)]
    assert np.array_equal(O.rne_bf16(u), _torch_bf16_bits(u))


def test_vs_torch_random():
    rng = np.random.default_rng(0)
    u = rng.integers(0, 1 << 32, size=1 << 22, dtype=np.uint64).astype(np.uint32)
    u = u[~_is_nan(u)]
    assert np.array_equal(O.rne_bf16(u), _torch_bf16_bits(u))


def test_nan_canonical():
    rng = np.random.default_rng(1)
    m = rng.integers(1, 1 << 23, size=4096, dtype=np.uint64).astype(np.uint32)
    s = rng.integers(0, 2, size=4096, dtype=np.uint64).astype(np.uint32) << np.uint32(31)
    u = s | np.uint32(0x7F800000) | m
    assert (O.rne_bf16(u) == 0x7FC0).all()


def _bf16_value(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def test_vs_nearest_definition():
    """Textbook RNE: pick the nearer of the two bf16 neighbours, ties to the even
    mantissa; beyond the largest finite value the next step is 2^128 (IEEE
    unbounded-exponent rule), which rounds to infinity."""
    rng = np.random.default_rng(2)
    u = np.concatenate([
        rng.integers(0, 1 << 32, size=1 << 20, dtype=np.uint64).astype(np.uint32),
        (rng.integers(0, 1 << 16, size=1 << 16, dtype=np.uint64).astype(np.uint32) << np.uint32(16)) | np.uint32(0x8000),
    ])
    u = u[~_is_nan(u) & ((u & 0x7FFFFFFF) < 0x7F800000)]     # finite only
    sign = u >> np.uint32(31)
    mag = u & np.uint32(0x7FFFFFFF)
    x = mag.view(np.float32).astype(np.float64)
    lo = (mag >> np.uint32(16)).astype(np.uint16)
    hi = (lo + 1).astype(np.uint16)
    lo_v = _bf16_value(lo)
    hi_v = np.where(hi == 0x7F80, 2.0 ** 128, _bf16_value(hi))
    dlo, dhi = x - lo_v, hi_v - x
    pick_hi = (dhi < dlo) | ((dhi == dlo) & ((lo & 1) == 1))
    want = np.where(pick_hi, hi, lo).astype(np.uint16) | (sign.astype(np.uint16) << np.uint16(15))
    assert np.array_equal(O.rne_bf16(u), want)
