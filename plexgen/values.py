"""Counter-based synthetic state generator, NumPy side.

INPUT MODULE. Every element of every synthetic state tensor is a pure function
of (seed, logical key, kind, flat index i in the *logical, unsharded* tensor),
so any rank can produce its own shard and the oracle can produce any slice,
bit-identically.  The CUDA product path implements the same counter-based
generator independently (synth_kernel in paper_2605_20863_b200/csrc/plex_kernels.cu); the two
share no code.  Nothing here is the method's arithmetic: there is no cast, no
layout, no checksum.

Definition (reading of D2):
    h  = FNV1a64(utf8(key))
    x  = (seed * 0xD1B54A32D192ED03) ^ h ^ (kind << 56) ^ i        (mod 2^64)
    z  = splitmix64(x)   -- first output of a SplitMix64 stream whose state is x
    fp32 kinds (MASTER=1, EXP_AVG=2, EXP_AVG_SQ=3):
        bits = sign<<31 | exp<<23 | mant
        mant = (z >> 8) & 0x7FFFFF;  exp = lo[kind] + ((z >> 32) & 7)
        sign = z >> 63 (0 for EXP_AVG_SQ);  lo = 0x76, 0x68, 0x58
    bf16 kind (PARAM=0), drawn independently of MASTER (reading D2'):
        bits = sign<<15 | (0x76 + ((z>>32)&7))<<7 | ((z >> 8) & 0x7F)
    special mode (fp32 kinds only): if (z & (2^k - 1)) == 0 the element is
        SPECIALS[(z >> 20) & 15] (Appendix C corner cases); k = special_bits.
    mutation (multiplex trace, o10): bits ^= (splitmix64(x ^ MUT(step)) & 0xFF).
"""
from __future__ import annotations

import numpy as np

KIND_PARAM, KIND_MASTER, KIND_EXP_AVG, KIND_EXP_AVG_SQ = 0, 1, 2, 3
KINDS = (KIND_PARAM, KIND_MASTER, KIND_EXP_AVG, KIND_EXP_AVG_SQ)
KIND_NAMES = ("param", "master", "exp_avg", "exp_avg_sq")
KIND_DTYPE = {0: np.uint16, 1: np.uint32, 2: np.uint32, 3: np.uint32}
KIND_BYTES = {0: 2, 1: 4, 2: 4, 3: 4}

SEED_MUL = 0xD1B54A32D192ED03
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
MUT_MUL = 0xA24BAED4963EE407
EXP_LO = {KIND_MASTER: 0x76, KIND_EXP_AVG: 0x68, KIND_EXP_AVG_SQ: 0x58}

# Appendix C fp32 corner cases (index = (z >> 20) & 15).
SPECIALS = np.array([
    0x00000000, 0x80000000, 0x00000001, 0x00018000,
    0x007FFFFF, 0x3F808000, 0x3F818000, 0x3F808001,
    0x3F807FFF, 0x7F7FFFFF, 0x7F7F8000, 0x7F800000,
    0xFF800000, 0x7FC00000, 0x7F800001, 0xFFC12345,
], dtype=np.uint32)

_M64 = (1 << 64) - 1


def fnv1a64(key: str) -> int:
    h = 0xCBF29CE484222325
    for b in key.encode("utf-8"):
        h ^= b
        h = (h * 0x100000001B3) & _M64
    return h


def splitmix64(x: np.ndarray) -> np.ndarray:
    """First SplitMix64 output for state x (vectorised, uint64 wrap-around)."""
    with np.errstate(over="ignore"):
        z = x + np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
        return z ^ (z >> np.uint64(31))


def stream_base(seed: int, key: str, kind: int) -> int:
    return ((seed * SEED_MUL) & _M64) ^ fnv1a64(key) ^ ((kind << 56) & _M64)


def gen_bits(seed: int, key: str, kind: int, idx: np.ndarray, special_bits: int = 0) -> np.ndarray:
    """Element bits at logical flat indices ``idx`` (uint64 array)."""
    x = np.uint64(stream_base(seed, key, kind)) ^ idx.astype(np.uint64)
    z = splitmix64(x)
    if kind == KIND_PARAM:
        sign = (z >> np.uint64(63)).astype(np.uint16)
        exp = (np.uint64(0x76) + ((z >> np.uint64(32)) & np.uint64(7))).astype(np.uint16)
        mant = ((z >> np.uint64(8)) & np.uint64(0x7F)).astype(np.uint16)
        return (sign << np.uint16(15)) | (exp << np.uint16(7)) | mant
    sign = (z >> np.uint64(63)).astype(np.uint32)
    if kind == KIND_EXP_AVG_SQ:
        sign[:] = 0
    exp = (np.uint64(EXP_LO[kind]) + ((z >> np.uint64(32)) & np.uint64(7))).astype(np.uint32)
    mant = ((z >> np.uint64(8)) & np.uint64(0x7FFFFF)).astype(np.uint32)
    bits = (sign << np.uint32(31)) | (exp << np.uint32(23)) | mant
    if special_bits > 0:
        sel = (z & np.uint64((1 << special_bits) - 1)) == 0
        if sel.any():
            bits[sel] = SPECIALS[((z[sel] >> np.uint64(20)) & np.uint64(15)).astype(np.int64)]
    return bits


def gen_range(seed: int, key: str, kind: int, start: int, count: int, special_bits: int = 0) -> np.ndarray:
    return gen_bits(seed, key, kind, np.arange(start, start + count, dtype=np.uint64), special_bits)


def gen_tensor(seed: int, key: str, kind: int, shape, special_bits: int = 0) -> np.ndarray:
    n = 1
    for s in shape:
        n *= s
    return gen_range(seed, key, kind, 0, n, special_bits).reshape(shape)


def mutation_bits(job_seed: int, step: int, key: str, kind: int, idx: np.ndarray) -> np.ndarray:
    """XOR mask applied by the multiplex trace's simulated training step (o10):
    the low 8 bits of every element (low mantissa bits of fp32 and bf16)."""
    s = (stream_base(job_seed, key, kind) ^ (((step + 1) * MUT_MUL) & _M64))
    z = splitmix64(np.uint64(s) ^ idx.astype(np.uint64))
    m = (z & np.uint64(0xFF))
    return m.astype(KIND_DTYPE[kind])
