"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact.

Multi-rank layouts are emulated on one GPU (every rank's buffers on cuda:0,
one ctx per rank; the sync's per-rank push kernels write into all ranks'
arenas), so the full W-rank data path is covered without W GPUs.
"""
from collections import OrderedDict

import numpy as np
import pytest
import torch

from oracle import plex_oracle as O
from plexgen import MODELS, gen_bits, gen_range, manifest, mutation_bits

from _state import full_state, fsdp_shards, master_shards

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2605_20863_b200")
from paper_2605_20863_b200 import _lib as L  # noqa: E402
from paper_2605_20863_b200.state import KIND_TORCH  # noqa: E402

U16, U32 = np.uint16, np.uint32


def bits_np(t: torch.Tensor) -> np.ndarray:
    t = t.detach().contiguous().cpu()
    if t.element_size() == 2:
        return t.view(torch.int16).numpy().view(U16)
    return t.view(torch.int32).numpy().view(U32)


def to_dev(a: np.ndarray, kind: int) -> torch.Tensor:
    dt = torch.int16 if kind == 0 else torch.int32
    return torch.from_numpy(a.view(np.int16 if kind == 0 else np.int32).copy()).view(KIND_TORCH[kind]).cuda() \
        if a.size else torch.empty(a.shape, dtype=KIND_TORCH[kind], device="cuda")


def mgr(W=1, r=0, bucket=4096, slots=2, **kw):
    return P.StateManager(device=0, rank=r, world=W, bucket_bytes=bucket, n_slots=slots, bootstrap=False, **kw)


def rank_shards(plan, r, seed, special_bits=0, kinds=(0, 1, 2, 3)):
    out = {}
    for t, (key, shape) in enumerate(plan.manifest):
        a, b = plan.shard_rows(r, t)
        re_ = int(np.prod(shape[1:])) if len(shape) > 1 else 1
        for kd in kinds:
            x = torch.empty((b - a,) + tuple(shape[1:]), dtype=KIND_TORCH[kd], device="cuda")
            P.synth_fill(x, kd, seed, key, a * re_, special_bits if kd else 0)
            out[(key, kd)] = x
    torch.cuda.synchronize()
    return out


# ---- K6 generator parity ----------------------------------------------------------
@pytest.mark.parametrize("model,W", [("toy-odd", 3), ("mid", 4), ("toy-moe", 2)])
def test_synth_matches_generator(model, W):
    plan = P.Plan(manifest(model), world=W)
    for r in range(W):
        sh = rank_shards(plan, r, seed=5, special_bits=3)
        for (key, kd), x in sh.items():
            shape = dict(plan.manifest)[key]
            re_ = int(np.prod(shape[1:])) if len(shape) > 1 else 1
            a, _ = plan.shard_rows(r, plan.index[key])
            want = gen_range(5, key, kd, a * re_, x.numel(), 3 if kd else 0)
            assert np.array_equal(bits_np(x).reshape(-1), want), (key, kd)


# ---- a8 cast parity -------------------------------------------------------------------
def test_cast_matches_oracle_specials_and_random():
    rng = np.random.default_rng(0)
    u = np.concatenate([
        np.array([int(l.split()[0], 16) for l in open(__file__.replace("test_gpu_parity.py", "golden/rne_specials.txt"))
                  if l.strip() and not l.startswith("#")], dtype=U32),
        rng.integers(0, 1 << 32, size=(1 << 24) + 13, dtype=np.uint64).astype(U32)])
    src = to_dev(u, 1)
    for off in (0, 1, 3):                      # aligned and misaligned vector paths
        s = src[off:]
        dst = torch.empty(s.numel(), dtype=torch.bfloat16, device="cuda")
        P.cast_rne(s, dst)
        torch.cuda.synchronize()
        assert np.array_equal(bits_np(dst), O.rne_bf16(u[off:]))


@pytest.mark.slow
def test_cast_exhaustive():
    """All 2^32 fp32 bit patterns (R8), GPU vs oracle, in 2^26 chunks."""
    n = 1 << 26
    dst = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    for c in range(1 << 6):
        u = np.arange(c * n, (c + 1) * n, dtype=np.uint64).astype(U32)
        P.cast_rne(to_dev(u, 1), dst)
        torch.cuda.synchronize()
        assert np.array_equal(bits_np(dst), O.rne_bf16(u)), c


# ---- K7 checksum parity ---------------------------------------------------------------------
@pytest.mark.parametrize("kind,n,base,off", [(0, 100_003, 0, 0), (1, 77_777, 12345, 0), (0, 5000, 7, 3), (3, 1 << 20, 1 << 31, 1)])
def test_checksum_matches_oracle(kind, n, base, off):
    a = gen_range(9, "ck", kind, 0, n + off)
    x = to_dev(a, kind)[off:]
    got = P.checksum(x, base).cpu().numpy().view(np.uint64)
    assert tuple(int(v) for v in got) == O.checksum(a[off:], base)


# ---- a3-a7 suspend/resume round trip ----------------------------------------------------------
RT_CASES = [("toy", 1, L.SLAB_KIND_MAJOR, 4096), ("toy-odd", 3, L.SLAB_KIND_MAJOR, 1024),
            ("toy-moe", 4, L.SLAB_KEY_MAJOR, 2048), ("mid", 2, L.SLAB_KIND_MAJOR, 1 << 16),
            ("mid-moe", 8, L.SLAB_KEY_MAJOR, 1 << 14), ("toy", 13, L.SLAB_KIND_MAJOR, 512),
            ("mid", 1, L.SLAB_KEY_MAJOR, 1 << 20)]


@pytest.mark.parametrize("model,W,layout,bucket", RT_CASES)
def test_offload_onload_roundtrip(model, W, layout, bucket):
    man = manifest(model)
    plan = P.Plan(man, world=W, slab_layout=layout, bucket_bytes=bucket, tile_bytes=512)
    full = full_state(model, seed=11, special_bits=3)
    for r in range(W):
        m = mgr(W, r, bucket=bucket, slots=3)
        sh = rank_shards(plan, r, seed=11, special_bits=3)
        slab = P.Slab(plan, r)
        assert slab.residency == L.RES_DEVICE
        with pytest.raises(P.PlexError) as e:           # never written: E_STATE
            m.onload(plan, slab, sh)
        assert e.value.code == L.E_STATE
        m.offload(plan, sh, slab)
        assert slab.residency == L.RES_HOST
        segs, size = O.slab_layout(man, W, r, layout)
        osh = fsdp_shards(full, W, r, O.fsdp_rows)
        assert np.array_equal(slab.host_bytes(), O.pack_slab(segs, size, osh))
        want_ck = np.array(O.segment_checksums(segs, osh), dtype=np.uint64).reshape(-1, 2)
        assert np.array_equal(slab.checksums(), want_ck)
        # release + re-acquire (a5), then restore into fresh garbage-filled buffers
        new = {k: torch.full_like(v, 7) if v.numel() else torch.empty_like(v) for k, v in sh.items()}
        del sh
        m.offload(plan, new, slab)                      # HOST already: no-op, slab unchanged
        assert np.array_equal(slab.host_bytes(), O.pack_slab(segs, size, osh))
        m.onload(plan, slab, new)
        assert slab.residency == L.RES_DEVICE
        for (key, kd), x in new.items():
            assert np.array_equal(bits_np(x), osh[(key, kd)]), (key, kd)


def test_onload_detects_slab_corruption():
    man = manifest("mid")
    plan = P.Plan(man, world=2, bucket_bytes=1 << 16)
    m = mgr(2, 1, bucket=1 << 16)
    sh = rank_shards(plan, 1, seed=3)
    slab = P.Slab(plan, 1)
    m.offload(plan, sh, slab)
    hb = slab.host_bytes()
    seg = plan.segments(1)[17]
    pos = seg.slab_offset + seg.nbytes // 2
    hb[pos] ^= 0x10
    with pytest.raises(P.PlexError) as e:
        m.onload(plan, slab, sh)
    assert e.value.code == L.E_CHECKSUM
    assert slab.residency == L.RES_HOST                 # no partial state change
    hb[pos] ^= 0x10
    m.onload(plan, slab, sh)
    assert slab.residency == L.RES_DEVICE


def test_job_suspend_resume_releases_memory():
    man = manifest("mid")
    m = mgr(1, 0, bucket=1 << 18)
    plan = m.plan(man)
    job = P.Job(m, plan, seed=4).alloc().init_synthetic()
    before = {k: bits_np(v) for k, v in job.shards.items()}
    job.suspend()
    assert all(v.untyped_storage().nbytes() == 0 for v in job.shards.values())
    job.resume()
    for k, v in job.shards.items():
        assert np.array_equal(bits_np(v), before[k])


# ---- a8-a11 weight sync (emulated W ranks on one GPU) -------------------------------------------
SYNC_CASES = [("toy", 1, 1, 1, 1), ("toy", 2, 2, 1, 1), ("toy-odd", 3, 1, 3, 1), ("toy-tied", 4, 2, 2, 1),
              ("toy-kv4", 4, 4, 1, 1), ("toy-moe", 4, 2, 2, 2), ("toy-moe", 8, 2, 4, 4), ("mid", 4, 2, 2, 1),
              ("mid", 8, 2, 4, 1), ("mid-moe", 8, 2, 4, 8), ("toy", 5, 1, 5, 1)]


@pytest.mark.parametrize("model,W,tp,dp,ep", SYNC_CASES)
@pytest.mark.parametrize("rank_map", [L.RANKMAP_TP_FAST, L.RANKMAP_DP_FAST])
def test_weight_sync_emulated(model, W, tp, dp, ep, rank_map):
    man = manifest(model)
    hd = MODELS[model].head_dim
    plan = P.Plan(man, head_dim=hd, world=W, tp=tp, dp=dp, ep=ep, rank_map=rank_map, tile_bytes=512)
    m = mgr(W, 0)
    masters = [[rank_shards(plan, r, seed=2, special_bits=3, kinds=(1,))[(k, 1)] for k, _ in man]
               for r in range(W)]
    arenas = [torch.full((max(256, plan.rank_info(g).dst_arena_bytes),), 0xAB, dtype=torch.uint8, device="cuda")
              for g in range(W)]
    for r in range(W):
        m.sync_rank(plan, r, masters[r], arenas)
    full = full_state(model, seed=2, kinds=(1,), special_bits=3)
    want = O.weight_sync(master_shards(full, W, O.fsdp_rows), tp, dp, ep, rank_map, hd)
    for g in range(W):
        views = P.StateManager.rollout_views(plan, g, arenas[g])
        assert list(views) == list(want[g])
        for name, v in views.items():
            assert np.array_equal(bits_np(v), want[g][name]), (g, name)


def test_weight_sync_world1_collective_entry():
    man = manifest("mid")
    m = mgr(1, 0)
    plan = m.plan(man, head_dim=32, tp=1, dp=1)
    job = P.Job(m, plan, seed=8, slab=False).alloc(kinds=(1,)).init_synthetic(special_bits=3)
    arena = m.arena(plan)
    job.sync(arena)
    full = full_state("mid", seed=8, kinds=(1,), special_bits=3)
    want = O.weight_sync(master_shards(full, 1, O.fsdp_rows), 1, 1, 1, O.TP_FAST, 32)[0]
    for name, v in P.StateManager.rollout_views(plan, 0, arena).items():
        assert np.array_equal(bits_np(v), want[name]), name


# ---- o10 multiplex trace (emulated 4 ranks, 4 jobs) ----------------------------------------------------
def test_multiplex_emulated():
    """configs[4] multiplex trace through the product's residency authority: one
    plex_group per (emulated) rank decides every switch itself
    and executes it; the op lists must equal the oracle's transition_ops and
    the rollout weights / final states the oracle's multiplex_replay.  Jobs
    release their device storage while suspended (a5) and are re-acquired
    through the group's storage callback."""
    W = 4
    models = ["toy", "toy-tied", "toy-moe", "mid"]
    layouts = [(2, 2, 1), (1, 4, 1), (2, 2, 2), (2, 2, 1)]
    seeds = [0, 1, 2, 3]
    schedule = [0, 1, 2, 3] * 2 + [3, 1]
    plans = [P.Plan(manifest(mo), head_dim=MODELS[mo].head_dim, world=W, tp=tp, dp=dp, ep=ep, bucket_bytes=1 << 14,
                    tile_bytes=1024) for mo, (tp, dp, ep) in zip(models, layouts)]
    mgrs = [mgr(W, r, bucket=1 << 14) for r in range(W)]
    jobs = [[P.Job(mgrs[r], plans[j], seed=seeds[j], rank=r).alloc().init_synthetic() for r in range(W)]
            for j in range(4)]
    for j in range(4):                      # every job starts HOST-resident, device storage released
        for r in range(W):
            jobs[j][r].suspend()
    groups = [P.Group(mgrs[r]) for r in range(W)]
    for r in range(W):
        for j in range(4):
            assert groups[r].add(jobs[j][r]) == j
    resident = None
    steps = [0] * 4
    outs, modes = [], []
    for j in schedule:
        want_ops = O.transition_ops(resident, j)
        for r in range(W):
            res = groups[r].transition(jobs[j][r])                # the product decides and executes
            assert res["ops"] == want_ops, (j, r, res)
            assert res["resident_after"] == j and groups[r].resident is jobs[j][r]
            modes.append(res["mode"])
        for jj in range(4):                                       # a5: only the resident job holds HBM
            for r in range(W):
                held = all(v.untyped_storage().nbytes() > 0 or v.numel() == 0
                           for v in jobs[jj][r].slab_shards().values())
                assert held == (jj == j), (jj, r)
        resident = j
        for r in range(W):
            for t, (key, shape) in enumerate(plans[j].manifest):
                a, _ = plans[j].shard_rows(r, t)
                re_ = int(np.prod(shape[1:])) if len(shape) > 1 else 1
                for kd in range(4):
                    P.synth_mutate(jobs[j][r].shards[(key, kd)], kd, seeds[j], steps[j], key, a * re_)
        steps[j] += 1
        arenas = [mgrs[0].arena(plans[j], g) for g in range(W)]
        for r in range(W):                                        # resident already: [SYNC j] only
            res = groups[r].transition(jobs[j][r], sync=arenas)
            assert res["ops"] == O.transition_ops(j, j, True) and res["mode"] == "none"
        outs.append([{k: bits_np(v) for k, v in P.StateManager.rollout_views(plans[j], g, arenas[g]).items()}
                     for g in range(W)])
    want_modes = ["load"] + ["none" if a == b else "duplex" for a, b in zip(schedule, schedule[1:])]
    assert modes == [m for m in want_modes for _ in range(W)]
    # oracle replay
    ojobs = []
    for mo, sd, (tp, dp, ep) in zip(models, seeds, layouts):
        full = full_state(mo, seed=sd)
        ojobs.append({"manifest": manifest(mo), "tp": tp, "dp": dp, "ep": ep,
                      "shards": [fsdp_shards(full, W, r, O.fsdp_rows) for r in range(W)]})

    def mut(job, step, key, kind, bits, base):
        idx = np.arange(base, base + bits.size, dtype=np.uint64)
        return bits ^ mutation_bits(seeds[job], step, key, kind, idx).reshape(bits.shape)

    # the oracle's sync uses head_dim=None: shapes here are all head-divisible
    visits, final = O.multiplex_replay(ojobs, schedule, W, mut)
    for v, (ops, want) in enumerate(visits):
        for g in range(W):
            for name, x in want[g].items():
                assert np.array_equal(outs[v][g][name], x), (v, g, name)
    for j in range(4):                       # every final state, brought back through the groups
        for r in range(W):
            groups[r].transition(jobs[j][r])
            for k, x in jobs[j][r].shards.items():
                assert np.array_equal(bits_np(x), final[j][r][k]), (j, r, k)


def test_group_modes_and_failures():
    """plex_group_transition picks the switch from what fits (R17):
    LOAD with nothing resident, NONE for the resident job, DUPLEX when the
    incoming storage can be acquired beside the resident one, SEQUENTIAL under
    an HBM budget for one job, SWAP for jobs sharing device storage; a corrupted
    incoming slab leaves no job resident and the outgoing state safe."""
    man = manifest("mid")
    hd = MODELS["mid"].head_dim
    plan = P.Plan(man, head_dim=hd, world=1, tp=1, dp=1, bucket_bytes=1 << 16, tile_bytes=4096)
    m = mgr(1, 0, bucket=1 << 16)
    fx, fy = full_state("mid", seed=31, special_bits=3), full_state("mid", seed=32, special_bits=3)
    segs, size = O.slab_layout(man, 1, 0)
    x = P.Job(m, plan, seed=31).alloc().init_synthetic(special_bits=3)
    y = P.Job(m, plan, seed=32).alloc().init_synthetic(special_bits=3)
    x.suspend()
    y.suspend()
    job_bytes = sum(v.numel() * v.element_size() for v in x.slab_shards().values())
    for budget, mode in ((None, "duplex"), (job_bytes, "sequential")):
        g = P.Group(m, hbm_budget=budget)
        ix, iy = g.add(x), g.add(y)
        assert g.resident is None
        r = g.transition(x)
        assert r["mode"] == "load" and r["ops"] == [(L.OP_ONLOAD, ix)] and r["resident_before"] == -1
        assert g.transition(x)["mode"] == "none"
        r = g.transition(y)
        assert r["mode"] == mode and r["ops"] == [(L.OP_OFFLOAD, ix), (L.OP_ONLOAD, iy)], r
        assert g.resident is y and all(v.untyped_storage().nbytes() == 0 for v in x.slab_shards().values())
        assert np.array_equal(x.slab.host_bytes(), O.pack_slab(segs, size, fx))
        for kk, v in y.shards.items():
            assert np.array_equal(bits_np(v), fy[kk]), kk
        arena = m.arena(plan)
        r = g.transition(y, sync=arena)
        assert r["ops"] == [(L.OP_SYNC, iy)]
        want = O.weight_sync(master_shards(fy, 1, O.fsdp_rows), 1, 1, 1, O.TP_FAST, hd)[0]
        for name, v in P.StateManager.rollout_views(plan, 0, arena).items():
            assert np.array_equal(bits_np(v), want[name]), name
        g.transition(x)                                           # back, then hand both to the next group
        x.suspend()
        g.close()
        del g
    # a corrupted incoming slab: E_CHECKSUM, nothing resident, the outgoing state safe in its slab
    g = P.Group(m)
    ix, iy = g.add(x), g.add(y)
    g.transition(x)
    y.slab.host_bytes()[segs[3].offset] ^= 0x40
    with pytest.raises(P.PlexError) as e:
        g.transition(y)
    assert e.value.code == L.E_CHECKSUM and g.resident is None
    assert np.array_equal(x.slab.host_bytes(), O.pack_slab(segs, size, fx))
    g.transition(x)                                               # x comes back intact
    for kk, v in x.shards.items():
        assert np.array_equal(bits_np(v), fx[kk]), kk
    g.close()
    # SWAP: two jobs sharing one set of device tensors and one slab
    a = P.Job(m, plan, seed=33, slab=False).alloc()
    b = P.Job(m, plan, seed=34)
    b.shards = a.shards
    b.init_synthetic(special_bits=3)
    b.suspend(release=False)
    b.shards = OrderedDict()
    a.init_synthetic(special_bits=3)
    fa, fb = full_state("mid", seed=33, special_bits=3), full_state("mid", seed=34, special_bits=3)
    g = P.Group(m)
    ia = g.add(a, resident=True, storage=0)
    ib = g.add(b, storage=0)
    with pytest.raises(P.PlexError) as e:                        # one resident job per group (R17)
        g.add(P.Job(m, plan, seed=35).alloc(), resident=True)
    assert e.value.code == L.E_STATE
    for k in range(3):
        inc, out, f_in, f_out = (b, a, fb, fa) if k % 2 == 0 else (a, b, fa, fb)
        r = g.transition(inc)
        assert r["mode"] == "swap" and r["ops"] == [(L.OP_OFFLOAD, out.group_id), (L.OP_ONLOAD, inc.group_id)]
        assert inc.slab is None and out.slab is not None and g.resident is inc
        for kk, v in inc.shards.items():
            assert np.array_equal(bits_np(v), f_in[kk]), kk
        assert np.array_equal(out.slab.host_bytes(), O.pack_slab(segs, size, f_out))
    g.close()
    m.close()


# ---- NEXT-1 duplex switch --------------------------------------------------------------------------
@pytest.mark.parametrize("models,buckets", [(("mid", "mid-moe"), (1 << 14, 1 << 16)), (("toy-odd", "toy"), (512, 1024)),
                                            (("mid", "mid"), (1 << 15, 1 << 15))])
def test_duplex_switch_matches_oracle(models, buckets):
    W = 2
    plans = [P.Plan(manifest(mo), world=W, bucket_bytes=b, tile_bytes=512) for mo, b in zip(models, buckets)]
    for r in range(W):
        m = P.StateManager(device=0, rank=r, world=W, bucket_bytes=max(buckets), n_slots=2, bootstrap=False)
        a = P.Job(m, plans[0], seed=30).alloc().init_synthetic(special_bits=3)
        b = P.Job(m, plans[1], seed=31).alloc().init_synthetic(special_bits=3)
        b.suspend()                                   # B waits in its slab, A resident
        for kk, v in b.shards.items():
            assert v.untyped_storage().nbytes() == 0
        for step in range(3):                         # A -> B -> A -> B
            src, dst = (a, b) if step % 2 == 0 else (b, a)
            src.switch_to(dst)
            assert src.slab.residency == L.RES_HOST and dst.slab.residency == L.RES_DEVICE
            for j, (mo, sd) in enumerate(zip(models, (30, 31))):
                full = full_state(mo, seed=sd, special_bits=3)
                osh = fsdp_shards(full, W, r, O.fsdp_rows)
                job = (a, b)[j]
                if job is dst:
                    for kk, x in job.shards.items():
                        assert np.array_equal(bits_np(x), osh[kk]), (step, kk)
                else:
                    segs, size = O.slab_layout(manifest(mo), W, r)
                    assert np.array_equal(job.slab.host_bytes(), O.pack_slab(segs, size, osh))
        m.close()


# ---- NEXT-1 in-place swap (one device copy, one slab) ----------------------------------------------
@pytest.mark.parametrize("model,W,layout,bucket", [("mid", 1, L.SLAB_KIND_MAJOR, 1 << 14),
                                                   ("toy-odd", 3, L.SLAB_KIND_MAJOR, 1024),
                                                   ("mid-moe", 4, L.SLAB_KEY_MAJOR, 1 << 15),
                                                   ("toy", 13, L.SLAB_KIND_MAJOR, 512)])
def test_inplace_swap_matches_oracle(model, W, layout, bucket):
    man = manifest(model)
    plan = P.Plan(man, world=W, slab_layout=layout, bucket_bytes=bucket, tile_bytes=512)
    fa, fb = full_state(model, seed=31, special_bits=3), full_state(model, seed=32, special_bits=3)
    for r in range(W):
        m = mgr(W, r, bucket=bucket, slots=2)
        oa, ob = fsdp_shards(fa, W, r, O.fsdp_rows), fsdp_shards(fb, W, r, O.fsdp_rows)
        segs, size = O.slab_layout(man, W, r, layout)
        dev = {kk: to_dev(x, kk[1]) for kk, x in ob.items()}       # B's state, offloaded into the slab
        slab = P.Slab(plan, r)
        m.offload(plan, dev, slab)
        for kk, x in oa.items():                                    # A resident in the same tensors
            dev[kk].copy_(to_dev(x, kk[1]))
        for it, (now_dev, now_slab) in enumerate(((ob, oa), (oa, ob), (ob, oa))):
            m.swap(plan, dev, slab)
            for kk, x in dev.items():
                assert np.array_equal(bits_np(x), now_dev[kk]), (it, kk)
            assert np.array_equal(slab.host_bytes(), O.pack_slab(segs, size, now_slab)), it
            want_ck = np.array(O.segment_checksums(segs, now_slab), dtype=np.uint64).reshape(-1, 2)
            assert np.array_equal(slab.checksums(), want_ck), it
            assert slab.residency == L.RES_HOST
        # a corrupted incoming state: E_CHECKSUM, and the outgoing state is safe in the slab
        if plan.rank_info(r).payload_bytes:
            seg = next(s_ for s_ in plan.segments(r) if s_.nbytes)
            slab.host_bytes()[seg.slab_offset] ^= 0x01
            with pytest.raises(P.PlexError) as e:
                m.swap(plan, dev, slab)
            assert e.value.code == L.E_CHECKSUM
            assert np.array_equal(slab.host_bytes(), O.pack_slab(segs, size, ob))
        m.close()


@pytest.mark.parametrize("model,W,bucket", [("mid", 1, 1 << 14), ("toy-odd", 3, 1024)])
@pytest.mark.parametrize("a_derived,b_derived", [(True, True), (True, False), (False, True), (False, False)])
def test_inplace_swap_with_elision(model, W, bucket, a_derived, b_derived):
    """NEXT-2 inside the swap: both jobs derivable -> both walk the shifted grid
    (params derived, not moved); only the incoming one elided -> the outgoing
    PARAM prefix goes out first; only the outgoing derivable -> it goes in full."""
    man = manifest(model)
    plan = P.Plan(man, world=W, bucket_bytes=bucket, tile_bytes=512, elide_param=True)

    def state(seed, derived):
        f = full_state(model, seed=seed, special_bits=0 if derived else 3)
        if derived:
            for (k, kd) in list(f):
                if kd == 1:
                    f[(k, 0)] = O.rne_bf16(f[(k, 1)])
        return f

    fa, fb = state(51, a_derived), state(52, b_derived)
    for r in range(W):
        m = mgr(W, r, bucket=bucket, slots=2)
        oa, ob = fsdp_shards(fa, W, r, O.fsdp_rows), fsdp_shards(fb, W, r, O.fsdp_rows)
        segs, size = O.slab_layout(man, W, r)
        cut = plan.rank_info(r).elide_bytes
        dev = {kk: to_dev(x, kk[1]) for kk, x in ob.items()}
        slab = P.Slab(plan, r)
        m.offload(plan, dev, slab)
        assert slab.elided == b_derived
        for kk, x in oa.items():
            dev[kk].copy_(to_dev(x, kk[1]))
        derived = {"a": a_derived, "b": b_derived}
        cur_in, cur_out = "b", "a"
        for it in range(3):
            want_el = slab.elided and derived[cur_out]
            m.swap(plan, dev, slab)
            now_dev = ob if cur_in == "b" else oa
            now_slab = oa if cur_out == "a" else ob
            for kk, x in dev.items():
                assert np.array_equal(bits_np(x), now_dev[kk]), (it, kk)
            assert slab.elided == want_el, it
            c0 = cut if want_el else 0
            assert np.array_equal(slab.host_bytes()[c0:], O.pack_slab(segs, size, now_slab)[c0:]), it
            want_ck = np.array(O.segment_checksums(segs, now_slab), dtype=np.uint64).reshape(-1, 2)
            assert np.array_equal(slab.checksums(), want_ck), it
            cur_in, cur_out = cur_out, cur_in
        m.close()


def test_job_swap_with_shares_one_device_copy():
    man = manifest("mid")
    m = mgr(1, 0, bucket=1 << 16)
    plan = m.plan(man)
    a = P.Job(m, plan, seed=1, slab=False).alloc()
    b = P.Job(m, plan, seed=2)
    b.shards = a.shards
    b.init_synthetic(special_bits=3)
    b.suspend(release=False)
    b.shards = OrderedDict()
    a.init_synthetic(special_bits=3)
    fa, fb = full_state("mid", seed=1, special_bits=3), full_state("mid", seed=2, special_bits=3)
    a.swap_with(b)
    assert a.slab is not None and b.slab is None
    for kk, x in b.shards.items():
        assert np.array_equal(bits_np(x), fb[kk]), kk
    b.swap_with(a)
    for kk, x in a.shards.items():
        assert np.array_equal(bits_np(x), fa[kk]), kk
    with pytest.raises(ValueError):
        a.swap_with(a)
    m.close()


# ---- NEXT-2 derived-param elision ----------------------------------------------------------------
@pytest.mark.parametrize("model,W,bucket", [("mid", 1, 4096), ("mid", 3, 1 << 14), ("toy-odd", 2, 512)])
def test_param_elision(model, W, bucket):
    man = manifest(model)
    plan = P.Plan(man, world=W, bucket_bytes=bucket, tile_bytes=512, elide_param=True)
    for r in range(W):
        m = mgr(W, r, bucket=bucket)
        info = plan.rank_info(r)
        assert info.elide_buckets >= 1
        # params == RNE(master): the leading buckets are derived, not moved
        job = P.Job(m, plan, seed=40, rank=r).alloc().init_synthetic(special_bits=3, derived_param=True)
        before = {k: bits_np(v) for k, v in job.shards.items()}
        full = full_state(model, seed=40, kinds=(1, 2, 3), special_bits=3)
        for (k, kd) in list(full):
            if kd == 1:
                full[(k, 0)] = O.rne_bf16(full[(k, 1)])
        osh = fsdp_shards(full, W, r, O.fsdp_rows)
        for kk, x in before.items():
            assert np.array_equal(x, osh[kk]), kk            # GPU inputs == oracle inputs
        job.suspend()
        assert job.slab.elided
        segs, size = O.slab_layout(man, W, r)
        want = O.pack_slab(segs, size, osh)
        cut = info.elide_bytes
        assert np.array_equal(job.slab.host_bytes()[cut:], want[cut:])     # stored part
        want_ck = np.array(O.segment_checksums(segs, osh), dtype=np.uint64).reshape(-1, 2)
        assert np.array_equal(job.slab.checksums(), want_ck)
        job.resume()
        for kk, x in job.shards.items():
            assert np.array_equal(bits_np(x), osh[kk]), kk
        # break the invariant on one element: full offload, still bit-exact
        p0 = next(v for (k, kd), v in job.shards.items() if kd == 0 and v.numel())
        p0.view(-1)[0:1].view(torch.int16).add_(1)
        state = {k: bits_np(v) for k, v in job.shards.items()}
        job.suspend()
        assert not job.slab.elided
        job.resume()
        for kk, x in job.shards.items():
            assert np.array_equal(bits_np(x), state[kk]), kk
        m.close()


# ---- NEXT-2 canonical dedup of replicated (ZeRO-2) params -------------------------------------------
@pytest.mark.parametrize("model,W,layout,elide", [("mid", 3, L.SLAB_KIND_MAJOR, False),
                                                  ("toy-moe", 4, L.SLAB_KEY_MAJOR, False),
                                                  ("toy-odd", 5, L.SLAB_KIND_MAJOR, True),
                                                  ("toy", 13, L.SLAB_KIND_MAJOR, False),
                                                  ("mid", 2, L.SLAB_KIND_MAJOR, True)])
def test_replica_param_dedup(model, W, layout, elide):
    """Each rank offloads only its FSDP rows of the replicated bf16 params; onload
    + the NVLink all-gather (emulated: every rank's push into all W arenas)
    restores every replica bit for bit (oracle dedup_param_shards / restore_replicas)."""
    man = manifest(model)
    plan = P.Plan(man, world=W, slab_layout=layout, bucket_bytes=1 << 14, tile_bytes=512, replica_param=True,
                  elide_param=elide)
    full = full_state(model, seed=21, special_bits=0 if elide else 3)
    if elide:                                   # params == RNE(master): the derivable case
        for (k, kd) in list(full):
            if kd == 1:
                full[(k, 0)] = O.rne_bf16(full[(k, 1)])
    reps = [OrderedDict((k, full[(k, 0)]) for k, _ in man) for _ in range(W)]
    stored = [O.dedup_param_shards(reps, r) for r in range(W)]
    want_rep = O.restore_replicas(stored)
    mgrs = [mgr(W, r, bucket=1 << 14) for r in range(W)]
    slabs = []
    for r in range(W):
        arena = mgrs[r].param_arena(plan)
        views = plan.param_views(arena)
        osh = fsdp_shards(full, W, r, O.fsdp_rows)
        sh = OrderedDict()
        for k, _ in man:
            for kd in range(4):
                if kd == 0:
                    views[k].copy_(to_dev(full[(k, 0)], 0))
                    sh[(k, 0)] = views[k]
                else:
                    sh[(k, kd)] = to_dev(osh[(k, kd)], kd)
        slab = P.Slab(plan, r)
        mgrs[r].offload(plan, sh, slab)
        # the dedup slab == the sharded slab of the oracle (params: own rows only)
        for k, _ in man:
            osh[(k, 0)] = stored[r][k]
        segs, size = O.slab_layout(man, W, r, layout)
        cut = plan.rank_info(r).elide_bytes if slab.elided else 0
        assert slab.elided == (elide and layout == L.SLAB_KIND_MAJOR)
        assert np.array_equal(slab.host_bytes()[cut:], O.pack_slab(segs, size, osh)[cut:])
        assert np.array_equal(slab.checksums(), np.array(O.segment_checksums(segs, osh), dtype=np.uint64).reshape(-1, 2))
        slabs.append((slab, osh))
    # restore into fresh, garbage-filled arenas and optimizer buffers
    arenas = [torch.full((max(256, plan.param_arena_bytes),), 0xAB, dtype=torch.uint8, device="cuda")
              for _ in range(W)]
    opt = []
    for r in range(W):
        views = plan.param_views(arenas[r])
        slab, osh = slabs[r]
        sh = OrderedDict()
        for k, _ in man:
            sh[(k, 0)] = views[k]
            for kd in (1, 2, 3):
                sh[(k, kd)] = torch.full_like(to_dev(osh[(k, kd)], kd), 3) if osh[(k, kd)].size \
                    else to_dev(osh[(k, kd)], kd)
        mgrs[r].onload(plan, slab, sh)
        opt.append(sh)
    for r in range(W):
        mgrs[r].param_allgather_rank(plan, r, arenas)
    for g in range(W):
        views = plan.param_views(arenas[g])
        for k, _ in man:
            assert np.array_equal(bits_np(views[k]), want_rep[g][k]), (g, k)
            for kd in (1, 2, 3):
                assert np.array_equal(bits_np(opt[g][(k, kd)]), slabs[g][1][(k, kd)]), (g, k, kd)
    for m in mgrs:
        m.close()


def test_replica_job_release_resume_world1():
    man = manifest("mid")
    m = mgr(1, 0, bucket=1 << 16)
    plan = m.plan(man, replica_param=True)
    job = P.Job(m, plan, seed=6).alloc().init_synthetic(special_bits=3)
    assert job.param_arena is not None
    before = {k: bits_np(v) for k, v in job.shards.items()}
    full = full_state("mid", seed=6, special_bits=3)
    for kk, x in before.items():
        assert np.array_equal(x, full[kk]), kk      # world 1: shards are the full tensors
    job.suspend()
    assert job.param_arena.untyped_storage().nbytes() == 0
    job.resume()
    for kk, v in job.shards.items():
        assert np.array_equal(bits_np(v), before[kk]), kk
    m.close()


# ---- NEXT-3 checkpoint materialisation from the offloaded slab ------------------------------------
def _load_ckpt(path):
    import json
    import struct

    from safetensors.torch import load_file
    with open(path, "rb") as f:
        n = struct.unpack("<Q", f.read(8))[0]
        hdr = json.loads(f.read(n))
    meta = hdr.pop("__metadata__")
    order = sorted(hdr, key=lambda k: hdr[k]["data_offsets"])     # data order in the file
    return load_file(path), meta, order


@pytest.mark.parametrize("model,W,layout", [("mid", 3, L.SLAB_KIND_MAJOR), ("toy-moe", 4, L.SLAB_KEY_MAJOR),
                                            ("toy", 13, L.SLAB_KIND_MAJOR)])
def test_slab_checkpoint_and_restore(tmp_path, model, W, layout):
    man = manifest(model)
    plan = P.Plan(man, world=W, slab_layout=layout, bucket_bytes=1 << 14, tile_bytes=512)
    full = full_state(model, seed=17, special_bits=3)
    for r in (0, W - 1):
        m = mgr(W, r, bucket=1 << 14)
        sh = rank_shards(plan, r, seed=17, special_bits=3)
        slab = P.Slab(plan, r)
        with pytest.raises(P.PlexError) as e:                  # nothing offloaded yet
            slab.checkpoint(str(tmp_path / "x.safetensors"))
        assert e.value.code == L.E_STATE
        m.offload(plan, sh, slab)
        path = str(tmp_path / f"{model}-r{r}.safetensors")
        th = slab.checkpoint(path, threads=4, background=True)
        m.onload(plan, slab, sh)                # resuming from the slab while it is written out is fine
        th.join()
        assert not th.errors
        # a standard safetensors file holding exactly the oracle's tensors, in slab order
        segs, _ = O.slab_layout(man, W, r, layout)
        osh = fsdp_shards(full, W, r, O.fsdp_rows)
        want = O.checkpoint_tensors(segs, osh)
        got, meta, order = _load_ckpt(path)
        assert order == list(want) and sorted(got) == sorted(want)
        for name, x in want.items():
            assert tuple(got[name].shape) == x.shape, name
            assert got[name].dtype == (torch.bfloat16 if x.dtype == U16 else torch.float32), name
            assert np.array_equal(bits_np(got[name]), x), name
        assert meta == O.checkpoint_metadata(W, r, O.segment_checksums(segs, osh))
        # restore into a fresh slab, onload into fresh buffers
        slab2 = P.Slab(plan, r)
        slab2.restore(path)
        assert slab2.residency == L.RES_HOST
        new = {k: torch.full_like(v, 5) if v.numel() else torch.empty_like(v) for k, v in sh.items()}
        m.onload(plan, slab2, new)
        for (key, kd), x in new.items():
            assert np.array_equal(bits_np(x), osh[(key, kd)]), (key, kd)
        if not plan.rank_info(r).payload_bytes:    # all shards empty: no data to corrupt
            m.close()
            continue
        # a flipped data byte is caught by the next onload
        raw = bytearray(open(path, "rb").read())
        raw[-3] ^= 0x40
        bad = str(tmp_path / "bad.safetensors")
        open(bad, "wb").write(bytes(raw))
        slab3 = P.Slab(plan, r)
        slab3.restore(bad)
        with pytest.raises(P.PlexError) as e:
            m.onload(plan, slab3, new)
        assert e.value.code == L.E_CHECKSUM
        # another plan's checkpoint is refused, the slab untouched
        other = P.Plan(man, world=W + 1, slab_layout=layout, bucket_bytes=1 << 14)
        with pytest.raises(P.PlexError) as e:
            P.Slab(other, 0).restore(path)
        assert e.value.code == L.E_LAYOUT
        m.close()


def test_checkpoint_refuses_elided_slab(tmp_path):
    man = manifest("mid")
    plan = P.Plan(man, world=1, bucket_bytes=4096, tile_bytes=512, elide_param=True)
    m = mgr(1, 0, bucket=4096)
    job = P.Job(m, plan, seed=2).alloc().init_synthetic(derived_param=True)
    job.suspend()
    assert job.slab.elided
    with pytest.raises(P.PlexError) as e:
        job.slab.checkpoint(str(tmp_path / "e.safetensors"))
    assert e.value.code == L.E_STATE
    m.close()


# ---- NEXT-3 sync straight from the offloaded slab ----------------------------------------------------
@pytest.mark.parametrize("model,W,tp,dp,ep,elide", [("mid", 4, 2, 2, 1, False), ("mid-moe", 4, 2, 2, 4, True),
                                                     ("toy-odd", 3, 1, 3, 1, False)])
def test_sync_from_slab(model, W, tp, dp, ep, elide):
    man = manifest(model)
    hd = MODELS[model].head_dim
    plan = P.Plan(man, head_dim=hd, world=W, tp=tp, dp=dp, ep=ep, bucket_bytes=1 << 14, tile_bytes=1024,
                  elide_param=elide)
    mgrs = [mgr(W, r, bucket=1 << 14) for r in range(W)]
    jobs = [P.Job(mgrs[r], plan, seed=50, rank=r).alloc().init_synthetic(special_bits=3, derived_param=elide)
            for r in range(W)]
    for j in jobs:
        j.suspend()                                   # training state leaves the GPU
    arenas = [torch.full((max(256, plan.rank_info(g).dst_arena_bytes),), 0xEE, dtype=torch.uint8, device="cuda")
              for g in range(W)]
    with pytest.raises(P.PlexError):                  # wrong rank's slab
        mgrs[0].sync_rank_from_slab(plan, 1, jobs[0].slab, arenas)
    for r in range(W):
        mgrs[r].sync_rank_from_slab(plan, r, jobs[r].slab, arenas)
    full = full_state(model, seed=50, kinds=(1,), special_bits=3)
    want = O.weight_sync(master_shards(full, W, O.fsdp_rows), tp, dp, ep, O.TP_FAST, hd)
    for g in range(W):
        for name, v in P.StateManager.rollout_views(plan, g, arenas[g]).items():
            assert np.array_equal(bits_np(v), want[g][name]), (g, name)
    jobs[0].resume()
    with pytest.raises(P.PlexError) as e:             # device-resident again: nothing to read in the slab
        mgrs[0].sync_rank_from_slab(plan, 0, jobs[0].slab, arenas)
    assert e.value.code == L.E_STATE


def test_sync_from_slab_refuses_carried_buckets():
    """A rank whose buckets are carried by a peer (NEXT-1 link balancing) does
    not hold its tail master rows in its own slab: sync-from-slab must refuse
    instead of reading stale bytes (E_INVAL before any residency check)."""
    man = manifest("mid")
    plan = P.Plan(man, head_dim=MODELS["mid"].head_dim, world=2, tp=2, dp=1, bucket_bytes=1 << 14,
                  tile_bytes=1024, link_weights=[1.0, 0.05])
    assert plan.rank_info(1).carried_out > 0
    m = mgr(2, 1, bucket=1 << 14)
    slab = P.Slab(plan, 1)
    arenas = [m.arena(plan, g) for g in range(2)]
    with pytest.raises(P.PlexError) as e:
        m.sync_rank_from_slab(plan, 1, slab, arenas)
    assert e.value.code == L.E_INVAL and "carried" in str(e.value)
    m.close()


def test_background_checkpoint_marks_slab_before_returning(tmp_path):
    """plex_slab_checkpoint_start: the slab is read-only from the moment the
    call returns (swap into it / restore refused with E_STATE) until join();
    onload from it proceeds meanwhile; afterwards the slab is writable again."""
    man = manifest("mid")
    plan = P.Plan(man, world=1, bucket_bytes=1 << 16, tile_bytes=4096)
    m = mgr(1, 0, bucket=1 << 16)
    sh = rank_shards(plan, 0, seed=23)
    slab = P.Slab(plan, 0)
    m.offload(plan, sh, slab)
    want = slab.host_bytes().copy()
    path = str(tmp_path / "bg.safetensors")
    th = slab.checkpoint(path, threads=2, background=True)
    with pytest.raises(P.PlexError) as e:
        m.swap(plan, sh, slab)                        # would overwrite the slab being written out
    assert e.value.code == L.E_STATE
    with pytest.raises(P.PlexError) as e:
        slab.restore(path)
    assert e.value.code == L.E_STATE
    m.onload(plan, slab, sh)                          # reading the slab is fine
    th.join()
    assert not th.errors
    assert np.array_equal(slab.host_bytes(), want)
    slab2 = P.Slab(plan, 0)
    slab2.restore(path)                               # the file is complete and consistent
    assert np.array_equal(slab2.host_bytes(), want)
    m.close()


# ---- NEXT-4 NVMe cold tier ----------------------------------------------------------------------
def test_slab_nvme_tier(tmp_path):
    man = manifest("mid")
    plan = P.Plan(man, world=2, bucket_bytes=1 << 16, tile_bytes=1024)
    m = mgr(2, 1, bucket=1 << 16)
    job = P.Job(m, plan, seed=60, rank=1).alloc().init_synthetic(special_bits=3)
    before = {k: bits_np(v) for k, v in job.shards.items()}
    job.suspend()
    slab_bytes = job.slab.host_bytes().copy()
    path = str(tmp_path / "slab.bin")
    try:
        job.slab.spill(path, threads=4)
    except P.PlexError as e:                        # filesystem without O_DIRECT
        pytest.skip(f"O_DIRECT unavailable here: {e}")
    assert job.slab.residency == L.RES_DISK and job.slab.host_bytes().size == 0
    with pytest.raises(P.PlexError) as e:
        job.resume()
    assert e.value.code == L.E_STATE
    job.slab.fill(path, threads=3)
    assert job.slab.residency == L.RES_HOST
    assert np.array_equal(job.slab.host_bytes(), slab_bytes)
    job.resume()
    for k, v in job.shards.items():
        assert np.array_equal(bits_np(v), before[k])
    # a corrupted file is caught by the onload checksum
    job.suspend()
    job.slab.spill(path)
    with open(path, "r+b") as f:
        f.seek(plan.segments(1)[5].slab_offset + 3)
        b = f.read(1)
        f.seek(-1, 1)
        f.write(bytes([b[0] ^ 0x40]))
    job.slab.fill(path)
    with pytest.raises(P.PlexError) as e:
        job.resume()
    assert e.value.code == L.E_CHECKSUM
    m.close()


def test_binding_rejects_mis_sized_tensors():
    """A wrong-size / wrong-dtype / non-contiguous shard or arena is refused by
    the binding before any kernel could write out of bounds."""
    man = manifest("mid")
    plan = P.Plan(man, head_dim=32, world=2, tp=2, dp=1, bucket_bytes=1 << 16)
    m = mgr(2, 0, bucket=1 << 16)
    sh = rank_shards(plan, 0, seed=1)
    slab = P.Slab(plan, 0)
    key = man[3][0]
    bad = dict(sh)
    bad[(key, 1)] = torch.empty(sh[(key, 1)].numel() + 1, dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        m.offload(plan, bad, slab)
    bad[(key, 1)] = sh[(key, 1)].to(torch.float16) if sh[(key, 1)].numel() else sh[(key, 1)]
    with pytest.raises(ValueError):
        m.offload(plan, bad, slab)
    assert slab.residency == L.RES_DEVICE                      # nothing happened
    masters = [sh[(k, 1)] for k, _ in man]
    small = torch.empty(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        m.sync_rank(plan, 0, masters, [small, small])
    with pytest.raises(ValueError):
        m.sync_rank(plan, 0, masters[:-1], [m.arena(plan, 0), m.arena(plan, 1)])


# ---- NEXT-1 async prefetch / drain ---------------------------------------------------------------
@pytest.mark.parametrize("elide", [False, True])
def test_async_prefetch_and_drain(elide):
    """B is prefetched while A keeps computing, then A is drained while B
    computes and syncs; both end bit-identical to the oracle's replay."""
    W, r = 2, 1
    models = ("mid", "mid-moe")
    plans = [P.Plan(manifest(mo), head_dim=MODELS[mo].head_dim, world=W, tp=2, dp=1, ep=2 if "moe" in mo else 1,
                    bucket_bytes=1 << 14, tile_bytes=1024, elide_param=elide) for mo in models]
    m = mgr(W, r, bucket=1 << 14)
    a = P.Job(m, plans[0], seed=70, rank=r).alloc().init_synthetic(special_bits=3, derived_param=elide)
    b = P.Job(m, plans[1], seed=71, rank=r).alloc().init_synthetic(special_bits=3, derived_param=elide)
    b.suspend()
    # while B's state comes back, A "trains": one mutation step on every shard
    b.prefetch()
    with pytest.raises(P.PlexError) as e:              # blocking transfers must wait for the async one
        a.suspend()
    assert e.value.code == L.E_STATE
    for t, (key, shape) in enumerate(plans[0].manifest):
        a0, _ = plans[0].shard_rows(r, t)
        re_ = int(np.prod(shape[1:])) if len(shape) > 1 else 1
        for kd in range(4):
            if not elide or kd != 0:
                P.synth_mutate(a.shards[(key, kd)], kd, 70, 0, key, a0 * re_)
    if elide:                                           # keep params == RNE(master)
        for key, _ in plans[0].manifest:
            if a.shards[(key, 0)].numel():
                P.cast_rne(a.shards[(key, 1)], a.shards[(key, 0)])
    b.wait_prefetch()
    assert b.slab.residency == L.RES_DEVICE
    a.drain()
    arena = torch.zeros(plans[1].rank_info(r).dst_arena_bytes + 256, dtype=torch.uint8, device="cuda")
    arenas = [torch.zeros_like(arena) for _ in range(W)]
    arenas[r] = arena
    m.sync_rank(plans[1], r, b.masters(), arenas)       # sync of B runs while A drains
    a.wait_drain()
    assert a.slab.residency == L.RES_HOST and a.slab.elided == elide
    # oracle: B unchanged, A mutated once
    for j, (mo, sd, job) in enumerate(zip(models, (70, 71), (a, b))):
        full = full_state(mo, seed=sd, kinds=(1, 2, 3), special_bits=3)
        if not elide:
            full.update({(k, 0): x for (k, kd), x in full_state(mo, seed=sd, kinds=(0,)).items()})
        if j == 0:
            for (key, kd), x in list(full.items()):
                idx = np.arange(x.size, dtype=np.uint64)
                full[(key, kd)] = x ^ mutation_bits(70, 0, key, kd, idx).reshape(x.shape)
        if elide:
            for (key, kd) in [kk for kk in full if kk[1] == 1]:
                full[(key, 0)] = O.rne_bf16(full[(key, 1)])
        osh = fsdp_shards(full, W, r, O.fsdp_rows)
        if job is a:
            segs, size = O.slab_layout(manifest(mo), W, r)
            want = O.pack_slab(segs, size, osh)
            cut = plans[0].rank_info(r).elide_bytes if elide else 0
            assert np.array_equal(job.slab.host_bytes()[cut:], want[cut:])
            job.resume()
        for kk, x in job.shards.items():
            assert np.array_equal(bits_np(x), osh[kk]), (j, kk)
    m.close()


def test_timeline_records_cover_the_switch():
    """Launch records (PLEX_CTX_TIMING) carry start times per blocking call: every
    bucket of a duplex switch has its pack, D2H, H2D and unpack, each inside the call."""
    man = manifest("mid")
    m = mgr(1, 0, bucket=1 << 15, timing=True)
    plans = [m.plan(man) for _ in range(2)]
    a = P.Job(m, plans[0], seed=1).alloc().init_synthetic()
    b = P.Job(m, plans[1], seed=2).alloc().init_synthetic()
    b.suspend()
    m.reset_stats()
    a.switch_to(b)
    recs = m.timeline()
    nb = plans[0].rank_info(0).n_buckets
    kinds = [r["kind"] for r in recs]
    for k in ("pack", "d2h", "h2d", "unpack"):
        assert kinds.count(k) == nb, k
    assert {r["call"] for r in recs} == {0}
    t0 = min(r["start_ms"] for r in recs)
    assert t0 == 0.0 and all(r["ms"] >= 0 for r in recs)
    # per bucket: the D2H starts after its pack ended, the unpack after its H2D ended
    packs = [r for r in recs if r["kind"] == "pack"]
    d2hs = [r for r in recs if r["kind"] == "d2h"]
    h2ds = [r for r in recs if r["kind"] == "h2d"]
    unps = [r for r in recs if r["kind"] == "unpack"]
    for p_, d_ in zip(packs, d2hs):
        assert d_["start_ms"] >= p_["start_ms"] + p_["ms"] - 0.01
    for h_, u_ in zip(h2ds, unps):
        assert u_["start_ms"] >= h_["start_ms"] + h_["ms"] - 0.01
    m.close()


def test_swap_with_replica_params_world1():
    """In-place swap of two ZeRO-2 (replica_param) jobs: the full replicated
    params travel with the device tensors; a non-replica plan is refused by
    the all-gather."""
    man = manifest("mid")
    m = mgr(1, 0, bucket=1 << 15)
    plan = m.plan(man, replica_param=True)
    a = P.Job(m, plan, seed=61, slab=False).alloc()
    b = P.Job(m, plan, seed=62)
    b.shards, b.param_arena = a.shards, a.param_arena
    b.init_synthetic(special_bits=3)
    b.suspend(release=False)
    b.shards, b.param_arena = OrderedDict(), None
    a.init_synthetic(special_bits=3)
    fa, fb = full_state("mid", seed=61, special_bits=3), full_state("mid", seed=62, special_bits=3)
    a.swap_with(b)
    assert b.param_arena is not None and a.param_arena is None
    for kk, x in b.shards.items():
        assert np.array_equal(bits_np(x), fb[kk]), kk
    b.swap_with(a)
    for kk, x in a.shards.items():
        assert np.array_equal(bits_np(x), fa[kk]), kk
    plain = m.plan(man)
    with pytest.raises(ValueError):
        m.param_allgather(plain, a.param_arena)
    with pytest.raises(P.PlexError) as e:
        P._lib.check(P._lib.lib.plex_param_allgather(m.h, plain.h, a.param_arena.data_ptr(), None))
    assert e.value.code == L.E_INVAL
    m.close()


def test_workspace_is_the_callers_and_bounded():
    """SURVEY §8(b) ownership: the library keeps every device table in the
    workspace the caller hands to plex_ctx_create (it never calls cudaMalloc).
    Too small a workspace is refused at creation; a plan whose tables do not
    fit fails with E_TIER_FULL before anything moves; destroying the plan
    gives its tables back."""
    import gc
    with pytest.raises(P.PlexError) as e:
        P.StateManager(device=0, bucket_bytes=4096, bootstrap=False, workspace_bytes=4096)
    assert e.value.code == L.E_INVAL
    man = [("w", (4096, 16384))]                              # 64 M elements; 4 KiB buckets -> 230 k work items
    small = P.StateManager(device=0, bucket_bytes=4096, bootstrap=False, workspace_bytes=1 << 20)
    plan = small.plan(man)
    job = P.Job(small, plan, seed=3).alloc().init_synthetic()
    before = {k: P.checksum(v).cpu() for k, v in job.shards.items()}
    with pytest.raises(P.PlexError) as e:
        job.suspend(release=False)
    assert e.value.code == L.E_TIER_FULL and "workspace" in str(e.value)
    assert job.slab.residency == L.RES_DEVICE                 # nothing moved
    assert all(torch.equal(P.checksum(v).cpu(), before[k]) for k, v in job.shards.items())
    big = P.StateManager(device=0, bucket_bytes=4096, bootstrap=False, workspace_bytes=64 << 20)
    base, _ = big.workspace_usage()
    plan2 = big.plan(man)
    job2 = P.Job(big, plan2, seed=3).alloc().init_synthetic()
    job2.suspend()
    job2.resume()                                              # checksum-verified round trip
    assert all(torch.equal(P.checksum(v).cpu(), before[k]) for k, v in job2.shards.items())
    used, hw = big.workspace_usage()
    assert used > base and hw >= used
    del job2, plan2
    gc.collect()
    assert big.workspace_usage()[0] < used                     # the plan's tables went back
    del job, plan
    gc.collect()
    small.close()
    big.close()
