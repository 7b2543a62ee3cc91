"""a1 + a2 through the bare C ABI (ctypes, no Python Plan wrapper): a C caller
passes only parameter keys and shapes (PLEX_ROLE_AUTO) and the planner derives
every rollout role, fusion group and split unit itself (reading R3,
PAPER.md:576).  The ledger and the destination names / shapes must equal the
oracle's; the transition decision must equal the oracle's op list
(PAPER.md:555).  Pure host code: runs without a GPU."""
import ctypes as C
from collections import OrderedDict

import numpy as np
import pytest

from oracle import plex_oracle as O
from plexgen import MODELS, manifest
from paper_2605_20863_b200 import _lib as L

lib = L.lib
SHAPE_ONLY = np.dtype([])          # zero-byte elements: the oracle's layout rule on shapes alone


def _plan_from_keys(man, world, tp, dp, ep, head_dim, rank_map=L.RANKMAP_TP_FAST):
    keys = [k.encode() for k, _ in man]
    arr = (L.TensorDesc * len(man))()
    for i, (k, s) in enumerate(man):
        d1 = int(np.prod(s[1:])) if len(s) > 1 else 1
        # role AUTO; group / slot / expert / unit deliberately garbage: the planner must ignore them
        arr[i] = L.TensorDesc(keys[i], int(s[0]), d1, len(s), L.ROLE_AUTO, 999, 7, 5, 3)
    req = L.PlanReq(len(man), arr, world, tp, dp, ep, rank_map, L.SLAB_KIND_MAJOR, L.KINDMASK_ALL, 0, None,
                    64 << 20, 64 << 10, -1, -1, L.OP_NONE, 0, None, head_dim)
    h = C.c_void_p()
    code = lib.plex_transition_plan(C.byref(req), C.byref(h))
    return code, h, (keys, arr)


def _dst(h, g):
    info = L.RankInfo()
    assert lib.plex_plan_rank_info(h, g, C.byref(info)) == L.OK
    out = []
    for i in range(info.n_dst_tensors):
        d = L.DstDesc()
        assert lib.plex_plan_dst_tensor(h, g, i, C.byref(d)) == L.OK
        buf = C.create_string_buffer(256)
        n, role, ne = C.c_int32(), C.c_int32(), C.c_int32()
        assert lib.plex_plan_group(h, d.group, buf, 256, C.byref(n), C.byref(role), C.byref(ne)) == L.OK
        out.append((buf.value.decode(), d.rows, d.cols, role.value, ne.value))
    return out


def _want_shapes(man, tp, dp, ep, g, rank_map, head_dim):
    full = OrderedDict((k, np.empty(s if len(s) > 1 else (s[0],), dtype=SHAPE_ONLY)) for k, s in man)
    return [(n, x.shape) for n, x in O.rollout_tensors(full, tp, dp, ep, g, rank_map, head_dim).items()]


@pytest.mark.parametrize("model,W,tp,dp,ep,rank_map", [("qwen2.5-7b", 8, 2, 4, 1, L.RANKMAP_TP_FAST),
                                                       ("qwen2.5-7b", 8, 2, 4, 1, L.RANKMAP_DP_FAST),
                                                       ("qwen3-30b-a3b", 8, 2, 4, 8, L.RANKMAP_TP_FAST),
                                                       ("toy-moe", 4, 2, 2, 2, L.RANKMAP_TP_FAST),
                                                       ("qwen2.5-0.5b", 2, 2, 1, 1, L.RANKMAP_TP_FAST)])
def test_auto_roles_from_keys_and_shapes(model, W, tp, dp, ep, rank_map):
    man = manifest(model)
    hd = MODELS[model].head_dim
    code, h, _keep = _plan_from_keys(man, W, tp, dp, ep, hd, rank_map)
    assert code == L.OK, lib.plex_last_error()
    try:
        buf = (C.c_uint64 * (W * W))()
        assert lib.plex_plan_ledger(h, buf, W * W) == L.OK
        got = np.frombuffer(buf, dtype=np.uint64).reshape(W, W).astype(np.int64)
        assert np.array_equal(got, O.ledger(man, W, tp, dp, ep, rank_map))
        for g in range(W):
            want = _want_shapes(man, tp, dp, ep, g, rank_map, hd)
            have = _dst(h, g)
            assert [n for n, *_ in have] == [n for n, _ in want]
            for (n, rows, cols, role, ne), (_, shp) in zip(have, want):
                if role == L.ROLE_EXPERT:                     # [E/EP, rows/E*EP, cols] stacked experts
                    assert ne % ep == 0 and shp == (ne // ep, rows // (ne // ep), cols), n
                elif len(shp) == 1:
                    assert (rows, cols) == (shp[0], 1), n
                else:
                    assert (rows, cols) == shp, n
    finally:
        lib.plex_plan_destroy(h)


def test_auto_roles_check_head_granularity():
    """unit = head_dim: Qwen2.5-7B's 28 query heads do not split over TP 8
    (E_LAYOUT), although its 3584 q rows are divisible by 8."""
    man = manifest("qwen2.5-7b")
    code, h, _ = _plan_from_keys(man, 8, 8, 1, 1, 128)
    assert code == L.E_LAYOUT and b"q_proj" in lib.plex_last_error()
    code, h, _ = _plan_from_keys(man, 8, 8, 1, 1, 0)          # no head granularity: rows split
    assert code == L.OK
    lib.plex_plan_destroy(h)


def test_mixing_auto_and_explicit_roles_is_rejected():
    man = manifest("toy")
    keys = [k.encode() for k, _ in man]
    arr = (L.TensorDesc * len(man))()
    for i, (k, s) in enumerate(man):
        d1 = int(np.prod(s[1:])) if len(s) > 1 else 1
        arr[i] = L.TensorDesc(keys[i], int(s[0]), d1, len(s), L.ROLE_AUTO if i else L.ROLE_REPLICATED, i, 0, -1, 1)
    req = L.PlanReq(len(man), arr, 1, 1, 1, 1, 0, 0, L.KINDMASK_ALL, 0, None, 0, 0, -1, -1, 0, 0, None, 4)
    h = C.c_void_p()
    assert lib.plex_transition_plan(C.byref(req), C.byref(h)) == L.E_INVAL
    assert b"AUTO" in lib.plex_last_error()


@pytest.mark.parametrize("resident", [None, 0, 1, 5])
@pytest.mark.parametrize("incoming", [0, 1, 7])
@pytest.mark.parametrize("sync", [False, True])
def test_transition_decide_matches_oracle(resident, incoming, sync):
    t = L.Transition()
    assert lib.plex_transition_decide(-1 if resident is None else resident, incoming,
                                      L.OP_SYNC if sync else L.OP_NONE, C.byref(t)) == L.OK
    got = [(t.ops[i], t.op_jobs[i]) for i in range(t.n_ops)]
    assert got == O.transition_ops(resident, incoming, sync)
    assert t.resident_before == (-1 if resident is None else resident)
    assert t.resident_after == incoming and t.mode == L.SWITCH_NONE
