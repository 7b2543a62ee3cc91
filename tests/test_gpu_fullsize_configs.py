"""Full-size parity at the BASELINE.json configs that do not fit the default
tier, all on ONE B200 (slow tier):

* M2  Qwen2.5-7B FSDP-8 -> TP-2 x DP-4 with the bench's AUTO rank map: all 8
      ranks' pushes emulated on one GPU (every rank's masters and arena in its
      HBM); the ledger equals O.ledger and the (S1, S2) of EVERY rollout tensor
      of EVERY rank equals the oracle's gather -> RNE -> slice/fuse, plus
      element-by-element compares of sampled tensors;
* M1/M2 slab: the whole Qwen2.5-7B FSDP-1 state (the bench's N=1 workload):
      every slab byte against the oracle's regeneration and the oracle's
      (S1, S2) of every segment against what offload recorded;
* M4  one rank's FSDP-8 shard of the Qwen3-30B-A3B KEY_MAJOR plan (75,468
      segments, 32-B ones included) through pack / offload / onload / unpack:
      every slab byte and checksum against the oracle, restored tensors
      compared byte for byte for 64 random tensors and the largest;
* M3  the Qwen2.5-32B optimizer-only (master / m / v) round trip of rank 0's
      FSDP-8 shard at k = 1, with the oracle's checksums of every segment.

The oracle work is fanned out over the host's cores (tests/_oracle_pool.py).
"""
import gc

import numpy as np
import pytest
import torch

from oracle import plex_oracle as O
from plexgen import MODELS, gen_range, manifest, mutation_bits

import _oracle_pool as OP

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

P = pytest.importorskip("paper_2605_20863_b200")
from paper_2605_20863_b200 import _lib as L  # noqa: E402


def bits_np(t: torch.Tensor) -> np.ndarray:
    t = t.detach().contiguous().cpu()
    return t.view(torch.int16).numpy().view(np.uint16) if t.element_size() == 2 else \
        t.view(torch.int32).numpy().view(np.uint32)


def _need(gb: float):
    if not torch.cuda.is_available() or torch.cuda.get_device_properties(0).total_memory < gb * 1e9:
        pytest.skip(f"needs a GPU with >= {gb} GB")


def _free(*objs):
    del objs
    gc.collect()
    torch.cuda.empty_cache()


def _emulated_sync_every_tensor(model, seed, W, tp, dp, ep, sample_keys, want_rmap=None):
    """All W source ranks' pushes emulated on one B200, one source rank at a
    time (its master shard generated, pushed into all W arenas, freed), so only
    the W arenas + one master shard are resident.  Checks: ledger == O.ledger;
    (S1, S2) of EVERY rollout tensor of EVERY rank == the oracle's gather -> RNE
    -> slice/fuse (c1.3); element by element for ``sample_keys`` (each list is
    one set of keys fused together, e.g. q/k/v) on every rank."""
    torch.cuda.set_device(0)
    man = manifest(model)
    hd = MODELS[model].head_dim
    plan = P.Plan(man, head_dim=hd, world=W, tp=tp, dp=dp, ep=ep, rank_map=L.RANKMAP_AUTO, bucket_bytes=1 << 20)
    rmap = plan.stats().rank_map
    if want_rmap is not None:
        assert rmap == want_rmap
    assert np.array_equal(plan.ledger(), O.ledger(man, W, tp, dp, ep, rmap))
    mgr = P.StateManager(device=0, rank=0, world=W, bucket_bytes=1 << 20, bootstrap=False)
    arenas = [torch.full((plan.rank_info(g).dst_arena_bytes,), 0xEE, dtype=torch.uint8, device="cuda")
              for g in range(W)]
    for r in range(W):                                       # source rank r's push into all W arenas
        job = P.Job(mgr, plan, seed=seed, rank=r, slab=False).alloc(kinds=(1,)).init_synthetic()
        mgr.sync_rank(plan, r, job.masters(), arenas)
        torch.cuda.synchronize()
        del job
        gc.collect()
        torch.cuda.empty_cache()
    want = OP.rollout_checksums(seed, man, tp, dp, ep, rmap, hd)
    views = [P.StateManager.rollout_views(plan, g, arenas[g]) for g in range(W)]
    assert sorted(want) == sorted((g, n) for g in range(W) for n in views[g])
    names = [(g, n) for g in range(W) for n in views[g]]
    ck = torch.zeros((len(names), 2), dtype=torch.int64, device="cuda")
    for i, (g, n) in enumerate(names):
        P.checksum(views[g][n], 0, out=ck[i])
    got = ck.cpu().numpy().view(np.uint64)
    bad = [names[i] for i in range(len(names)) if tuple(int(v) for v in got[i]) != want[names[i]]]
    assert not bad, bad[:10]
    shapes = dict(man)
    n_cmp = 0
    for keys in sample_keys:                                 # element by element, every rank
        full = {k: gen_range(seed, k, 1, 0, int(np.prod(shapes[k]))).reshape(shapes[k]) for k in keys}
        cast = {k: O.rne_bf16(v) for k, v in full.items()}
        for g in range(W):
            for name, x in O.rollout_tensors(cast, tp, dp, ep, g, rmap, hd).items():
                assert np.array_equal(bits_np(views[g][name]), x), (g, name)
                n_cmp += 1
    assert n_cmp > 0
    del views, arenas
    mgr.close()
    _free()
    return len(names)


def test_m2_qwen7b_fsdp8_to_tp2dp4_every_rollout_tensor():
    """configs[1]: Qwen2.5-7B FSDP-8 -> TP-2 x DP-4 with the bench's AUTO rank
    map (R10 picks DP_FAST: 5.99 vs 7.33 GB over the busiest link)."""
    _need(150)
    qkv = [f"model.layers.0.self_attn.{n}_proj.weight" for n in "qkv"]
    _emulated_sync_every_tensor("qwen2.5-7b", 1, 8, 2, 4, 1,
                                [qkv, ["model.layers.27.mlp.down_proj.weight"], ["lm_head.weight"],
                                 ["model.layers.13.self_attn.o_proj.weight"]], want_rmap=L.RANKMAP_DP_FAST)


def test_m3_qwen32b_fsdp8_to_tp4dp2_every_rollout_tensor():
    """configs[2] sync: Qwen2.5-32B FSDP-8 -> TP-4 x DP-2 (Table 1 32B row,
    PAPER.md:615): 8 arenas (131 GB) + one 16.4 GB master shard at a time."""
    _need(150)
    qkv = [f"model.layers.7.self_attn.{n}_proj.weight" for n in "qkv"]
    gu = [f"model.layers.40.mlp.{n}_proj.weight" for n in ("gate", "up")]
    _emulated_sync_every_tensor("qwen2.5-32b", 2, 8, 4, 2, 1,
                                [qkv, gu, ["model.layers.63.mlp.down_proj.weight"],
                                 ["model.layers.31.self_attn.o_proj.weight"]])


def test_m4_qwen3_30b_a3b_fsdp8_to_tp2dp4_ep8_every_rollout_tensor():
    """configs[3] sync: Qwen3-30B-A3B FSDP-8 -> attention TP-2 x DP-4 + experts
    EP-8 (Table 1): every rollout tensor (w13 / w2 expert stacks
    included) against the oracle; attention, router and q/k norms element by
    element."""
    _need(150)
    qkv = [f"model.layers.11.self_attn.{n}_proj.weight" for n in "qkv"]
    _emulated_sync_every_tensor("qwen3-30b-a3b", 3, 8, 2, 4, 8,
                                [qkv, ["model.layers.47.self_attn.o_proj.weight"],
                                 ["model.layers.5.mlp.gate.weight"], ["model.layers.5.self_attn.q_norm.weight"]])


def test_m1m2_qwen7b_fsdp1_every_slab_byte():
    _need(150)
    torch.cuda.set_device(0)
    model, seed = "qwen2.5-7b", 1
    man = manifest(model)
    mgr = P.StateManager(device=0, bucket_bytes=2 << 30, n_slots=2, bootstrap=False)
    plan = mgr.plan(man, head_dim=MODELS[model].head_dim, tp=1, dp=1)
    job = P.Job(mgr, plan, seed=seed).alloc().init_synthetic()
    job.suspend()                                            # offload + release device storage
    segs = plan.segments(0)
    host = job.slab.host_bytes()
    cks, bad = OP.check_slab(seed, man, segs, host)
    assert not bad, bad[:10]
    assert np.array_equal(job.slab.checksums(), cks)         # offload's R14 == the oracle's, every segment
    ends = [s.slab_offset + s.nbytes for s in segs]          # zero padding (R4)
    starts = [s.slab_offset for s in segs[1:]] + [host.size]
    for e, nxt in zip(ends, starts):
        assert nxt - e < 256 and not host[e:nxt].any()
    job.resume()                                             # checksum-verified against the oracle's values
    for key in ("model.embed_tokens.weight", "model.layers.5.mlp.gate_proj.weight"):
        for kd in range(4):
            x = job.shards[(key, kd)]
            assert np.array_equal(bits_np(x).reshape(-1), gen_range(seed, key, kd, 0, x.numel())), (key, kd)
    del host, job, plan
    mgr.close()
    _free()


def _shard_roundtrip(model, seed, W, rank, layout, kind_mask, n_sample):
    torch.cuda.set_device(0)
    man = manifest(model)
    mgr = P.StateManager(device=0, rank=rank, world=W, bucket_bytes=2 << 30, n_slots=2, bootstrap=False)
    plan = mgr.plan(man, slab_layout=layout, kind_mask=kind_mask)
    kinds = tuple(k for k in range(4) if kind_mask & (1 << k))
    job = P.Job(mgr, plan, seed=seed, rank=rank).alloc(kinds=kinds).init_synthetic()
    job.suspend()
    segs = plan.segments(rank)
    host = job.slab.host_bytes()
    cks, bad = OP.check_slab(seed, man, segs, host)
    assert not bad, bad[:10]
    assert np.array_equal(job.slab.checksums(), cks)
    want_segs, size = O.slab_layout(man, W, rank, layout, kinds=kinds)
    assert host.size == size
    assert [(s.tensor, s.kind, s.slab_offset, s.nbytes) for s in segs] == \
        [(s.tensor, s.kind, s.offset, s.nbytes) for s in want_segs]
    job.resume()
    shapes = dict(man)
    for key in OP.sample_keys(man, n_sample, seed):
        t = plan.index[key]
        a, _ = plan.shard_rows(rank, t)
        re_ = int(np.prod(shapes[key][1:])) if len(shapes[key]) > 1 else 1
        for kd in kinds:
            x = job.shards[(key, kd)]
            assert np.array_equal(bits_np(x).reshape(-1), gen_range(seed, key, kd, a * re_, x.numel())), (key, kd)
    n_seg = len(segs)
    del host, job, plan
    mgr.close()
    _free()
    return n_seg


def test_m4_qwen3_30b_a3b_key_major_rank_shard():
    """One rank's FSDP-8 shard of the 30B-A3B KEY_MAJOR plan: 75,468 segments
    (per-expert units contiguous, 32-B segments included), 53.4 GB."""
    _need(150)
    n = _shard_roundtrip("qwen3-30b-a3b", 3, 8, 3, L.SLAB_KEY_MAJOR, L.KINDMASK_ALL, 64)
    assert n == 75_468


def test_m3_qwen32b_optimizer_only_roundtrip_k1():
    """configs[2] at k = 1: the optimizer kinds (master / m / v, 49.15 GB) of
    rank 0's FSDP-8 shard of Qwen2.5-32B, offloaded and restored."""
    _need(150)
    n = _shard_roundtrip("qwen2.5-32b", 2, 8, 0, L.SLAB_KIND_MAJOR, L.KINDMASK_OPTIM, 64)
    assert n == 3 * len(manifest("qwen2.5-32b"))


def test_m5_multiplex_trace_fullsize():
    """configs[4] at full size: 4 jobs shaped Qwen2.5-0.5B / 1.5B / 3B / 7B
    (seeds 0..3) time-slice one GPU group for R = 5
    round-robin rounds (20 visits, 19 switches).  D1's FSDP-8 emulated on one
    B200 (one plex_group per rank, all 8 ranks' shards and arenas in its HBM:
    7B state 106.6 GB + 8 arenas 61 GB at the widest point); rollout TP-1 x
    DP-8 for 0.5B, TP-2 x DP-4 for the rest.  (FSDP-4, TP-2 x DP-2, when the
    device reports less than 185e9 bytes.)  Every switch is decided and executed by the library's residency
    authority (op lists == O.transition_ops), every visit mutates
    the state (o10 reading M1) and syncs it.  Checks:
      * per visit, element by element on every rank: the fused q/k/v, o_proj
        and input norm of one layer against the oracle's rollout of the
        mutated masters (init XOR every mask so far, the multiplex_replay
        closed form pinned in tests/test_oracle_multiplex.py);
      * at the end, EVERY (key, kind) of every job: each job is brought back
        through its group, its masks are XOR-ed out again, and the R14
        checksum (additive over the 4 shards) equals the oracle's checksum of
        the regenerated initial state -- any byte the 19 switches lost or
        moved fails it."""
    _need(150)
    torch.cuda.set_device(0)
    W = 8 if torch.cuda.get_device_properties(0).total_memory >= 185e9 else 4
    print(f"M5 trace: FSDP-{W} emulated, device total_memory {torch.cuda.get_device_properties(0).total_memory}")
    models = ["qwen2.5-0.5b", "qwen2.5-1.5b", "qwen2.5-3b", "qwen2.5-7b"]
    seeds = [0, 1, 2, 3]
    rounds = 5
    schedule = list(range(4)) * rounds
    mgrs = [P.StateManager(device=0, rank=r, world=W, bucket_bytes=128 << 20, n_slots=2, bootstrap=False)
            for r in range(W)]
    plans, jobs = [], []
    for mo in models:
        tp = 1 if mo == "qwen2.5-0.5b" else 2
        plans.append(P.Plan(manifest(mo), head_dim=MODELS[mo].head_dim, world=W, tp=tp, dp=W // tp,
                            bucket_bytes=128 << 20))
    groups = [P.Group(mgrs[r]) for r in range(W)]
    for j, mo in enumerate(models):                        # every job starts HOST-resident
        row = []
        for r in range(W):
            jb = P.Job(mgrs[r], plans[j], seed=seeds[j], rank=r).alloc().init_synthetic()
            jb.suspend()
            row.append(jb)
        jobs.append(row)
        torch.cuda.synchronize()
        _free()
        for r in range(W):
            assert groups[r].add(jobs[j][r]) == j
    resident, steps, modes = None, [0] * 4, []

    def mutate(j, step):
        for r in range(W):
            for t, (key, shape) in enumerate(plans[j].manifest):
                a, _ = plans[j].shard_rows(r, t)
                re_ = int(np.prod(shape[1:])) if len(shape) > 1 else 1
                for kd in range(4):
                    P.synth_mutate(jobs[j][r].shards[(key, kd)], kd, seeds[j], step, key, a * re_)

    rng = np.random.default_rng(5)
    for v, j in enumerate(schedule):
        want_ops = O.transition_ops(resident, j)
        for r in range(W):
            res = groups[r].transition(jobs[j][r])
            assert res["ops"] == want_ops, (v, j, r, res)
            assert res["resident_after"] == j
            modes.append(res["mode"])
        resident = j
        mutate(j, steps[j])
        steps[j] += 1
        arenas = [mgrs[0].arena(plans[j], g) for g in range(W)]
        for r in range(W):
            res = groups[r].transition(jobs[j][r], sync=arenas)
            assert res["ops"] == O.transition_ops(j, j, True) and res["mode"] == "none"
        torch.cuda.synchronize()
        # oracle: one layer's q/k/v + o_proj + input norm after every mask so far
        mo = models[j]
        man = dict(manifest(mo))
        layer = int(rng.integers(MODELS[mo].layers))
        keys = [f"model.layers.{layer}.self_attn.{n}_proj.weight" for n in "qkvo"] + \
            [f"model.layers.{layer}.input_layernorm.weight"]
        cast = {}
        for k in keys:
            n = int(np.prod(man[k]))
            x = gen_range(seeds[j], k, 1, 0, n)
            idx = np.arange(n, dtype=np.uint64)
            for s in range(steps[j]):
                x = x ^ mutation_bits(seeds[j], s, k, 1, idx)
            cast[k] = O.rne_bf16(x).reshape(man[k])
        tp = plans[j].stats().tp
        for g in range(W):
            views = P.StateManager.rollout_views(plans[j], g, arenas[g])
            for name, x in O.rollout_tensors(cast, tp, W // tp, 1, g, L.RANKMAP_TP_FAST,
                                             MODELS[mo].head_dim).items():
                assert np.array_equal(bits_np(views[name]), x), (v, j, g, name)
        del arenas, views
        _free()
    want_modes = ["load"] + ["none" if a == b else ("duplex", "sequential") for a, b in zip(schedule, schedule[1:])]
    for i, m in enumerate(modes):
        w = want_modes[i // W]
        assert m == w if isinstance(w, str) else m in w, (i, m, w)
    # every byte of every job: undo the masks, R14 per (key, kind) == oracle of the initial state
    for j, mo in enumerate(models):
        for r in range(W):
            groups[r].transition(jobs[j][r])
        for s in range(steps[j]):
            mutate(j, s)                                   # XOR is an involution
        man = manifest(mo)
        names = [(k, kd) for k, _ in man for kd in range(4)]
        ck = torch.zeros((W, len(names), 2), dtype=torch.int64, device="cuda")
        for r in range(W):
            for i, (k, kd) in enumerate(names):
                t = plans[j].index[k]
                a, _ = plans[j].shard_rows(r, t)
                shape = dict(man)[k]
                re_ = int(np.prod(shape[1:])) if len(shape) > 1 else 1
                P.checksum(jobs[j][r].shards[(k, kd)], a * re_, out=ck[r, i])
        got = ck.cpu().numpy().view(np.uint64).astype(object).sum(axis=0)
        want = OP.tensor_checksums(seeds[j], man)
        bad = [names[i] for i in range(len(names))
               if (int(got[i][0]) & OP.M64, int(got[i][1]) & OP.M64) != want[names[i]]]
        assert not bad, (mo, bad[:10])
    for g in groups:
        g.close()
    for m in mgrs:
        m.close()
    _free()
