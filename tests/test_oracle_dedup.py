"""Pins of the oracle's NEXT-2 canonical dedup of replicated params
("deduplicating replicated state"; ZeRO-2; R18)
and the planner's replica plans against it.  Host-only."""
from collections import OrderedDict

import numpy as np
import pytest

from oracle import plex_oracle as O
from plexgen import MODELS, gen_tensor, manifest
from paper_2605_20863_b200 import Plan, PlexError, _lib as L


def replicas(model, world, seed=3):
    rep = OrderedDict((k, gen_tensor(seed, k, O.KIND_PARAM, s, 0)) for k, s in manifest(model))
    return [OrderedDict((k, v.copy()) for k, v in rep.items()) for _ in range(world)]


def test_param_arena_layout_hand_example():
    # a: 3 bf16 = 6 B at 0; b: 2x2 = 8 B at 256; c: 200 = 400 B at 512 -> end 912 -> 1024
    offs, size = O.param_arena_layout([("a", (3,)), ("b", (2, 2)), ("c", (200,))])
    assert offs == [0, 256, 512] and size == 1024


@pytest.mark.parametrize("model,world", [("toy", 1), ("toy", 2), ("toy-odd", 3), ("toy-moe", 5), ("toy", 13),
                                         ("mid", 8)])
def test_dedup_restore_identity_and_single_copy(model, world):
    reps = replicas(model, world)
    stored = [O.dedup_param_shards(reps, r) for r in range(world)]
    # every replicated byte is stored exactly once across the group
    one = sum(x.nbytes for x in reps[0].values())
    assert sum(x.nbytes for st in stored for x in st.values()) == one
    # and gathering the stored rows restores every replica bit for bit
    back = O.restore_replicas(stored)
    for r in range(world):
        assert list(back[r]) == list(reps[r])
        for k in reps[r]:
            assert np.array_equal(back[r][k], reps[r][k]), (r, k)
    # the stored rows are exactly the sharded plan's PARAM segments (R2)
    for r in range(world):
        for k, s in manifest(model):
            a, b = O.fsdp_rows(s[0], world, r)
            assert np.array_equal(stored[r][k], reps[r][k][a:b])


def test_dedup_rejects_diverged_replicas():
    reps = replicas("toy", 2)
    k = next(iter(reps[1]))
    reps[1][k] = reps[1][k].copy()
    reps[1][k].reshape(-1)[0] ^= 1
    with pytest.raises(AssertionError):
        O.dedup_param_shards(reps, 0)


@pytest.mark.parametrize("model,W", [("toy", 1), ("toy-odd", 3), ("toy-moe", 4), ("mid", 8), ("toy", 13)])
@pytest.mark.parametrize("layout", [L.SLAB_KIND_MAJOR, L.SLAB_KEY_MAJOR])
def test_replica_plan_matches_oracle(model, W, layout):
    man = manifest(model)
    p = Plan(man, world=W, slab_layout=layout, bucket_bytes=4096, tile_bytes=512, replica_param=True)
    plain = Plan(man, world=W, slab_layout=layout, bucket_bytes=4096, tile_bytes=512)
    offs, size = O.param_arena_layout(man)
    assert p.param_arena_bytes == size and p.param_offsets() == offs
    reps = replicas(model, W)
    stored = [sum(x.nbytes for x in O.dedup_param_shards(reps, r).values()) for r in range(W)]
    for r in range(W):
        # the dedup slab is the sharded slab, byte for byte in layout
        assert [bytes(s) for s in p.segments(r)] == [bytes(s) for s in plain.segments(r)]
        info = p.rank_info(r)
        assert info.slab_bytes == plain.rank_info(r).slab_bytes
        assert info.gather_send_bytes == (W - 1) * stored[r]
        assert info.gather_recv_bytes == sum(stored) - stored[r]
        assert (info.n_gather_items == 0) == (W == 1 or stored[r] == 0)


def test_replica_plan_needs_param_kind():
    with pytest.raises(PlexError) as e:
        Plan(manifest("toy"), world=2, kind_mask=L.KINDMASK_OPTIM, replica_param=True)
    assert e.value.code == L.E_INVAL
    with pytest.raises(PlexError):
        Plan(manifest("toy"), world=2).param_arena_bytes


# ---- NEXT-3 checkpoint materialisation (R19) ------------------------------------------
@pytest.mark.parametrize("model,world,layout", [("toy", 1, O.KIND_MAJOR), ("toy-odd", 3, O.KEY_MAJOR),
                                                ("toy-moe", 5, O.KIND_MAJOR), ("toy", 13, O.KIND_MAJOR)])
def test_checkpoints_of_all_ranks_rebuild_the_full_state(model, world, layout):
    """Brute force: the union over ranks of the checkpoint tensors, concatenated
    along dim 0 in rank order, is the full logical state of every (key, kind)."""
    man = manifest(model)
    full = {(k, kd): gen_tensor(7, k, kd, s, 3 if kd else 0) for k, s in man for kd in O.ALL_KINDS}
    per_rank = []
    for r in range(world):
        segs, _ = O.slab_layout(man, world, r, layout)
        sh = {kk: O.shard(x, world, r) for kk, x in full.items()}
        ck = O.checkpoint_tensors(segs, sh)
        assert len(ck) == len(segs) == 4 * len(man)          # names unique, one per segment
        per_rank.append(ck)
    for (k, kd), x in full.items():
        name = O.checkpoint_name(k, kd)
        got = np.concatenate([ck[name] for ck in per_rank], axis=0)
        assert got.dtype == x.dtype and np.array_equal(got, x), name


def test_checkpoint_names_and_metadata():
    assert O.checkpoint_name("model.norm.weight", 0) == "model.norm.weight"
    assert O.checkpoint_name("model.norm.weight", 3) == "optimizer.exp_avg_sq.model.norm.weight"
    md = O.checkpoint_metadata(2, 1, [(1, 0xABC), (2**64 - 1, 0)])
    assert md["plex.checksums"] == "0000000000000001,0000000000000abc,ffffffffffffffff,0000000000000000"
