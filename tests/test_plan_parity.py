"""Host planner (a1/a2, C++ in libplex) vs the oracle: slab layout (R4),
FSDP rows (R2), zero-redundancy ledger (o9), rollout tensor names and shapes
(R3) and transition ops.  Pure host code: runs without a GPU."""
import numpy as np
import pytest

from oracle import plex_oracle as O
from plexgen import MODELS, manifest
from paper_2605_20863_b200 import Plan, PlexError, _lib as L

from _state import full_state, master_shards

CASES = [("toy", 1, 1, 1, 1), ("toy", 2, 2, 1, 1), ("toy", 3, 1, 3, 1), ("toy-odd", 5, 1, 5, 1),
         ("toy-moe", 4, 2, 2, 2), ("toy-moe", 8, 2, 4, 4), ("toy-tied", 8, 1, 8, 1), ("toy-kv4", 4, 4, 1, 1),
         ("mid", 4, 2, 2, 1), ("mid-moe", 8, 2, 4, 8), ("toy", 13, 1, 13, 1)]


@pytest.mark.parametrize("model,W,tp,dp,ep", CASES)
@pytest.mark.parametrize("layout", [L.SLAB_KIND_MAJOR, L.SLAB_KEY_MAJOR])
def test_slab_layout_matches_oracle(model, W, tp, dp, ep, layout):
    man = manifest(model)
    p = Plan(man, head_dim=MODELS[model].head_dim, world=W, tp=tp, dp=dp, ep=ep, slab_layout=layout,
             bucket_bytes=4096, tile_bytes=512)
    for r in range(W):
        segs, size = O.slab_layout(man, W, r, layout)
        info = p.rank_info(r)
        assert info.slab_bytes == size
        got = [(s.tensor, s.kind, s.slab_offset, s.nbytes, s.row0, s.row1, s.index_base) for s in p.segments(r)]
        want = [(s.tensor, s.kind, s.offset, s.nbytes, s.row0, s.row1, s.index_base) for s in segs]
        assert got == want
        for t, (_, shp) in enumerate(man):
            assert p.shard_rows(r, t) == O.fsdp_rows(shp[0], W, r)


def test_subsets_and_kind_masks():
    man = manifest("toy-moe")
    keys = [k for k, _ in man if ".experts.2." in k or ".experts.3." in k]
    p = Plan(man, world=4, slab_layout=L.SLAB_KEY_MAJOR, subset=keys, kind_mask=L.KINDMASK_OPTIM)
    for r in range(4):
        segs, size = O.slab_layout(man, 4, r, O.KEY_MAJOR, kinds=O.OPTIM_KINDS, keys=keys)
        got = [(s.tensor, s.kind, s.slab_offset, s.nbytes) for s in p.segments(r)]
        assert got == [(s.tensor, s.kind, s.offset, s.nbytes) for s in segs]
        assert p.rank_info(r).slab_bytes == size


@pytest.mark.parametrize("model,W,tp,dp,ep", CASES)
@pytest.mark.parametrize("rank_map", [L.RANKMAP_TP_FAST, L.RANKMAP_DP_FAST])
def test_rollout_layout_and_ledger_match_oracle(model, W, tp, dp, ep, rank_map):
    man = manifest(model)
    hd = MODELS[model].head_dim
    p = Plan(man, head_dim=hd, world=W, tp=tp, dp=dp, ep=ep, rank_map=rank_map)
    assert np.array_equal(p.ledger(), O.ledger(man, W, tp, dp, ep, rank_map))
    full = full_state(model, kinds=(1,))
    out = O.weight_sync(master_shards(full, W, O.fsdp_rows), tp, dp, ep, rank_map, hd)
    for g in range(W):
        got = [(n, s) for n, _, s in p.dst_tensors(g)]
        want = [(n, x.shape) for n, x in out[g].items()]
        assert got == want
        info = p.rank_info(g)
        assert info.recv_bytes == p.ledger()[:, g].sum() - p.ledger()[g, g]
        offs = [o for _, o, _ in p.dst_tensors(g)]
        assert all(o % 256 == 0 for o in offs) and offs == sorted(offs)


def test_real_config_plans():
    # SURVEY.md Appendix B / §8(d) D1 numbers through the product planner.
    p = Plan(manifest("qwen2.5-7b"), head_dim=128, world=8, tp=2, dp=4)
    L8 = p.ledger()
    off = L8 - np.diag(np.diag(L8))
    assert abs(off.sum(axis=0).max() - 7.33e9) / 7.33e9 < 0.005
    assert p.rank_info(0).n_segments == 1356
    assert abs(p.rank_info(0).slab_bytes - 13.33e9) / 13.33e9 < 0.002
    p = Plan(manifest("qwen3-30b-a3b"), head_dim=128, world=8, tp=2, dp=4, ep=8)
    assert p.rank_info(0).n_segments == 75_468


def test_layout_errors():
    with pytest.raises(PlexError) as e:
        Plan(manifest("toy"), head_dim=4, world=4, tp=4, dp=1)        # kv heads 2 % TP 4
    assert e.value.code == L.E_LAYOUT
    with pytest.raises(PlexError) as e:
        Plan(manifest("toy-moe"), head_dim=4, world=8, tp=1, dp=8, ep=8)   # 4 experts % EP 8
    assert e.value.code == L.E_LAYOUT
    with pytest.raises(PlexError) as e:
        Plan(manifest("toy"), world=4, tp=2, dp=1)                     # tp*dp != world
    assert e.value.code == L.E_INVAL


@pytest.mark.parametrize("resident,incoming,op", [(0, 0, 0), (0, 1, 0), (-1, 1, 0), (2, 2, 3), (1, 2, 3), (3, -1, 0)])
def test_transition_ops_match_oracle(resident, incoming, op):
    p = Plan(manifest("toy"), world=1, resident_job=resident, incoming_job=incoming, op=op)
    want = O.transition_ops(None if resident < 0 else resident, incoming, op == L.OP_SYNC) if incoming >= 0 \
        else [(O.OP_OFFLOAD, resident)]
    assert p.ops() == [(a, b) for a, b in want]


def test_plan_is_deterministic():
    man = manifest("mid-moe")
    a = Plan(man, head_dim=16, world=8, tp=2, dp=4, ep=8)
    b = Plan(man, head_dim=16, world=8, tp=2, dp=4, ep=8)
    assert np.array_equal(a.ledger(), b.ledger())
    for r in range(8):
        assert a.dst_tensors(r) == b.dst_tensors(r)
        sa = [(s.slab_offset, s.nbytes) for s in a.segments(r)]
        assert sa == [(s.slab_offset, s.nbytes) for s in b.segments(r)]


def _busiest(L):
    off = L - np.diag(np.diag(L))
    return max(off.sum(0).max(), off.sum(1).max())


def test_rank_map_auto_picks_lighter_ledger():
    """R10: AUTO resolves to the rank map with the smaller busiest-link bytes;
    for Qwen2.5-7B FSDP-8 -> TP-2 x DP-4 that is DP_FAST (5.99 vs 7.33 GB)."""
    man = manifest("qwen2.5-7b")
    p = Plan(man, head_dim=128, world=8, tp=2, dp=4, rank_map=L.RANKMAP_AUTO)
    assert p.stats().rank_map == L.RANKMAP_DP_FAST
    assert np.array_equal(p.ledger(), O.ledger(man, 8, 2, 4, 1, O.DP_FAST))
    for model, W, tp, dp, ep in CASES:
        q = Plan(manifest(model), head_dim=MODELS[model].head_dim, world=W, tp=tp, dp=dp, ep=ep,
                 rank_map=L.RANKMAP_AUTO)
        m = q.stats().rank_map
        assert np.array_equal(q.ledger(), O.ledger(manifest(model), W, tp, dp, ep, m))
        other = O.ledger(manifest(model), W, tp, dp, ep, 1 - m)
        assert _busiest(q.ledger()) <= _busiest(other)
