"""Pins for the input module (plexgen): shape fixtures and the generator."""
import numpy as np
import pytest

from plexgen import models, values


@pytest.mark.parametrize("name,total", [
    # shape arithmetic == public model-card parameter counts.
    ("qwen2.5-0.5b", 494_032_768),
    ("qwen2.5-1.5b", 1_543_714_304),
    ("qwen2.5-3b", 3_085_938_688),
    ("qwen2.5-7b", 7_615_616_512),
    ("qwen2.5-32b", 32_763_876_352),
    ("qwen3-30b-a3b", 30_532_122_624),
])
def test_param_counts(name, total):
    assert models.param_count(name) == total


@pytest.mark.parametrize("name,card", [
    # Rounded totals on the public HF model cards.
    ("qwen2.5-0.5b", 0.49e9), ("qwen2.5-1.5b", 1.54e9), ("qwen2.5-3b", 3.09e9),
    ("qwen2.5-7b", 7.61e9), ("qwen3-30b-a3b", 30.5e9),
])
def test_param_counts_vs_cards(name, card):
    assert abs(models.param_count(name) - card) / card < 0.01


def test_tensor_counts():
    # tensors per kind.
    assert len(models.manifest("qwen2.5-0.5b")) == 290
    assert len(models.manifest("qwen2.5-7b")) == 339
    assert len(models.manifest("qwen2.5-32b")) == 771
    assert len(models.manifest("qwen3-30b-a3b")) == 18_867


def test_fnv1a64_vectors():
    # Published FNV-1a 64-bit test vectors.
    assert values.fnv1a64("") == 0xCBF29CE484222325
    assert values.fnv1a64("a") == 0xAF63DC4C8601EC8C
    assert values.fnv1a64("foobar") == 0x85944171F73967E8


def test_splitmix64_vectors():
    # SplitMix64 (Steele, Lea, Flood 2014) reference output for state 0, and
    # the stream from state 1234567 (first outputs of the reference C code).
    z = values.splitmix64(np.array([0], dtype=np.uint64))
    assert int(z[0]) == 0xE220A8397B1DCDAF
    # successive outputs: state advances by the golden gamma each call
    g = values.GOLDEN
    st = np.array([(1234567 + k * g) % (1 << 64) for k in range(3)], dtype=np.uint64)
    out = [int(v) for v in values.splitmix64(st)]
    assert out == [6457827717110365317, 3203168211198807973, 9817491932198370423]


def test_generator_ranges():
    idx = np.arange(100000, dtype=np.uint64)
    for kind, lo in ((1, 0x76), (2, 0x68), (3, 0x58)):
        b = values.gen_bits(7, "k", kind, idx)
        e = (b >> 23) & 0xFF
        assert e.min() >= lo and e.max() <= lo + 7
        if kind == 3:
            assert (b >> 31).max() == 0
    p = values.gen_bits(7, "k", 0, idx)
    assert p.dtype == np.uint16
    e = (p >> 7) & 0xFF
    assert e.min() >= 0x76 and e.max() <= 0x7D
    # low 16 mantissa bits of master are ~uniform: ~half of the casts round up
    b = values.gen_bits(7, "k", 1, idx)
    frac = ((b & 0xFFFF) > 0x8000).mean()
    assert 0.49 < frac < 0.51


def test_generator_slices_consistent():
    full = values.gen_tensor(3, "x.weight", 1, (37, 11))
    part = values.gen_range(3, "x.weight", 1, 5 * 11, 7 * 11).reshape(7, 11)
    assert np.array_equal(full[5:12], part)


def test_special_mode():
    b = values.gen_bits(0, "s", 1, np.arange(1 << 14, dtype=np.uint64), special_bits=3)
    hit = np.isin(b, values.SPECIALS)
    assert 0.08 < hit.mean() < 0.2
