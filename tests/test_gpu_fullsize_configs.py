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
from plexgen import MODELS, gen_range, manifest

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


def test_m2_qwen7b_fsdp8_to_tp2dp4_every_rollout_tensor():
    _need(150)
    torch.cuda.set_device(0)
    model, seed, W, tp, dp = "qwen2.5-7b", 1, 8, 2, 4
    man = manifest(model)
    hd = MODELS[model].head_dim
    plan = P.Plan(man, head_dim=hd, world=W, tp=tp, dp=dp, rank_map=L.RANKMAP_AUTO, bucket_bytes=1 << 20)
    rmap = plan.stats().rank_map
    assert rmap == L.RANKMAP_DP_FAST                         # R10: the lighter ledger (5.99 vs 7.33 GB)
    assert np.array_equal(plan.ledger(), O.ledger(man, W, tp, dp, 1, rmap))
    mgrs = [P.StateManager(device=0, rank=r, world=W, bucket_bytes=1 << 20, bootstrap=False) for r in range(W)]
    masters = [P.Job(mgrs[r], plan, seed=seed, rank=r, slab=False).alloc(kinds=(1,)).init_synthetic().masters()
               for r in range(W)]
    arenas = [torch.full((plan.rank_info(g).dst_arena_bytes,), 0xEE, dtype=torch.uint8, device="cuda")
              for g in range(W)]
    for r in range(W):                                       # every source rank's push into all 8 arenas
        mgrs[r].sync_rank(plan, r, masters[r], arenas)
    torch.cuda.synchronize()
    del masters
    gc.collect()
    torch.cuda.empty_cache()
    want = OP.rollout_checksums(seed, man, tp, dp, 1, rmap, hd)
    views = [P.StateManager.rollout_views(plan, g, arenas[g]) for g in range(W)]
    assert sorted(want) == sorted((g, n) for g in range(W) for n in views[g])
    names = [(g, n) for g in range(W) for n in views[g]]
    ck = torch.zeros((len(names), 2), dtype=torch.int64, device="cuda")
    for i, (g, n) in enumerate(names):
        P.checksum(views[g][n], 0, out=ck[i])
    got = ck.cpu().numpy().view(np.uint64)
    bad = [names[i] for i in range(len(names)) if tuple(int(v) for v in got[i]) != want[names[i]]]
    assert not bad, bad[:10]
    # element by element on sampled tensors, every rank
    shapes = dict(man)
    for key in ("model.layers.0.self_attn.q_proj.weight", "model.layers.27.mlp.down_proj.weight",
                "lm_head.weight", "model.layers.13.self_attn.o_proj.weight"):
        full = {key: gen_range(seed, key, 1, 0, int(np.prod(shapes[key]))).reshape(shapes[key])}
        if ".q_proj." in key:
            for n in "kv":
                k2 = key.replace(".q_proj.", f".{n}_proj.")
                full[k2] = gen_range(seed, k2, 1, 0, int(np.prod(shapes[k2]))).reshape(shapes[k2])
        cast = {k: O.rne_bf16(v) for k, v in full.items()}
        for g in range(W):
            for name, x in O.rollout_tensors(cast, tp, dp, 1, g, rmap, hd).items():
                assert np.array_equal(bits_np(views[g][name]), x), (g, name)
    del views, arenas
    for m in mgrs:
        m.close()
    _free()


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
