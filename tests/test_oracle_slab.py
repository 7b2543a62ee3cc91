"""Pins for the oracle's slab layout / pack / parse (a3-a7, o4/o5, reading R4):
round-trip identity, byte conservation,
checksum additivity across ranks (R14), 256-B alignment and zero padding."""
import numpy as np
import pytest

from oracle import plex_oracle as O
from plexgen import manifest, numel

from _state import full_state, fsdp_shards


@pytest.mark.parametrize("model", ["toy", "toy-odd", "toy-moe", "toy-tied"])
@pytest.mark.parametrize("world", [1, 2, 3, 5, 8, 13])
@pytest.mark.parametrize("layout", [O.KIND_MAJOR, O.KEY_MAJOR])
def test_roundtrip_and_conservation(model, world, layout):
    man = manifest(model)
    full = full_state(model, seed=world, special_bits=3)
    total = 0
    logical = {kk: O.checksum(x) for kk, x in full.items()}
    acc = {kk: (0, 0) for kk in full}
    for r in range(world):
        sh = fsdp_shards(full, world, r, O.fsdp_rows)
        segs, size = O.slab_layout(man, world, r, layout)
        assert size % 256 == 0
        slab = O.pack_slab(segs, size, sh)
        # segments are 256-B aligned, disjoint, in increasing offset order
        cur = 0
        covered = np.zeros(size, dtype=bool)
        for sg in segs:
            assert sg.offset % 256 == 0 and sg.offset >= cur
            covered[sg.offset:sg.offset + sg.nbytes] = True
            cur = sg.offset + sg.nbytes
        assert (slab[~covered] == 0).all()           # zero padding
        back = O.parse_slab(slab, segs, dict(man))
        for kk, x in sh.items():
            assert np.array_equal(back[kk], x)        # onload(offload(S)) == S
        total += sum(sg.nbytes for sg in segs)
        for sg, c in zip(segs, O.segment_checksums(segs, sh)):
            a = acc[(sg.key, sg.kind)]
            acc[(sg.key, sg.kind)] = ((a[0] + c[0]) % (1 << 64), (a[1] + c[1]) % (1 << 64))
    # byte conservation: sum over ranks = sum numel * size (14 B/param)
    assert total == sum(numel(s) for _, s in man) * 14
    assert acc == logical


def test_layouts_hold_same_segments():
    man = manifest("toy-moe")
    a, _ = O.slab_layout(man, 3, 1, O.KIND_MAJOR)
    b, _ = O.slab_layout(man, 3, 1, O.KEY_MAJOR)
    key = lambda s: (s.key, s.kind, s.nbytes, s.row0, s.row1)
    assert sorted(map(key, a)) == sorted(map(key, b))
    assert [s.kind for s in a[:5]] == [0] * 5
    assert [s.kind for s in b[:4]] == [0, 1, 2, 3]


def test_kind_and_key_subsets():
    man = manifest("toy-moe")
    segs, size = O.slab_layout(man, 2, 0, O.KIND_MAJOR, kinds=O.OPTIM_KINDS)
    assert {s.kind for s in segs} == {1, 2, 3}
    keys = [k for k, _ in man if ".experts.1." in k]
    segs, size = O.slab_layout(man, 2, 0, O.KEY_MAJOR, keys=keys)
    assert {s.key for s in segs} == set(keys) and len(segs) == 4 * len(keys)


def test_empty_shards():
    # N > d0: tail ranks own nothing (R2, torch.chunk semantics)
    assert O.fsdp_rows(6, 8, 6) == (6, 6) and O.fsdp_rows(6, 8, 7) == (6, 6)
    assert O.fsdp_rows(5, 4, 3) == (5, 5)
    assert O.fsdp_rows(6, 8, 2) == (2, 3)
    import torch
    for d0 in (1, 5, 6, 16, 17):
        for n in (1, 2, 3, 5, 8):
            ch = torch.arange(d0).chunk(n)
            for r in range(n):
                a, b = O.fsdp_rows(d0, n, r)
                want = ch[r].tolist() if r < len(ch) else []
                assert list(range(a, b)) == want


def test_real_config_sizes():
    # per-GPU state bytes and segment counts.
    for model, world, S, nseg in (("qwen2.5-0.5b", 1, 6.92e9, 1160),
                                  ("qwen2.5-7b", 8, 13.33e9, 1356),
                                  ("qwen2.5-32b", 8, 57.34e9, 3084)):
        segs, size = O.slab_layout(manifest(model), world, 0)
        assert len(segs) == nseg
        assert abs(size - S) / S < 0.002
