"""torchrun worker: full-size (Qwen2.5-7B-shaped) parity at N GPUs, the
launch configuration bench.py times: FSDP-N -> TP-min(2,N) x DP weight sync
through the collective NVLink push, and a duplex switch between two jobs.

Checks (see tests/test_gpu_fullsize.py for the rationale):
* sampled rollout tensors of every rank == oracle gather -> RNE -> slice/fuse;
* after switch A->B->A, every shard's device checksum (K7) equals its value
  before the switches (round-trip identity at full size), and the checksums
  recorded in the slab equal K7 over the source shards;
* sampled slab segments == oracle bytes.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2605_20863_b200 as P  # noqa: E402
from oracle import plex_oracle as O  # noqa: E402
from plexgen import MODELS, gen_range, gen_tensor, manifest  # noqa: E402

MODEL = os.environ.get("PLEX_FULL_MODEL", "qwen2.5-7b")
SAMPLE = ["model.layers.0.input_layernorm.weight", "model.layers.0.self_attn.q_proj.weight", "model.layers.5.self_attn.o_proj.weight",
          "model.layers.27.mlp.gate_proj.weight", "model.layers.13.mlp.down_proj.weight", "model.norm.weight",
          "model.layers.3.self_attn.q_proj.bias"]


def bits_np(t):
    t = t.detach().contiguous().cpu()
    return t.view(torch.int16).numpy().view(np.uint16) if t.element_size() == 2 else t.view(torch.int32).numpy().view(np.uint32)


def dev_checksums(plan, job, rank):
    man = plan.manifest
    segs = plan.segments(rank)
    ck = torch.zeros((len(segs), 2), dtype=torch.int64, device="cuda")
    for i, s in enumerate(segs):
        P.checksum(job.shards[(man[s.tensor][0], s.kind)], s.index_base, out=ck[i])
    return ck


def main():
    import faulthandler
    faulthandler.dump_traceback_later(900, exit=True)     # never hang a GPU box silently
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    shape = MODELS[MODEL]
    man = manifest(MODEL)
    tp = min(2, world)
    dp = world // tp
    mgr = P.StateManager(device=local, rank=rank, world=world)
    # bench.py's launch configuration: AUTO rank map, host-link balancing (here
    # with rank 0's link twice as fast, so the other ranks' buckets are carried)
    weights = [2.0 if r == 0 else 1.0 for r in range(world)]
    plans = [mgr.plan(man, head_dim=shape.head_dim, tp=tp, dp=dp, rank_map=2, link_weights=weights)
             for _ in range(2)]
    for pl in plans:
        mgr.enable_carry(pl)
    rmap = plans[0].stats().rank_map
    b = P.Job(mgr, plans[1], seed=2).alloc().init_synthetic()
    ck_b = dev_checksums(plans[1], b, rank)
    b.suspend()
    a = P.Job(mgr, plans[0], seed=1).alloc().init_synthetic()
    ck_a = dev_checksums(plans[0], a, rank)
    bad = 0
    # duplex switches A -> B -> A
    a.switch_to(b)
    if not torch.equal(dev_checksums(plans[1], b, rank), ck_b):
        print(f"[rank {rank}] B restore mismatch", flush=True)
        bad += 1
    rec = a.slab.checksums()
    if not np.array_equal(rec, ck_a.cpu().numpy().view(np.uint64)):
        print(f"[rank {rank}] A slab checksums != K7", flush=True)
        bad += 1
    slab = a.slab.host_bytes()
    # bytes of carried buckets live in the carrier's carry region (checked by
    # mp_carry_worker); sample the segments that stay in this rank's own slab
    carried = [(c.slab_offset, c.slab_offset + c.bytes) for c in plans[0].carry() if c.owner == rank]
    for i, s in enumerate(plans[0].segments(rank)):
        key = man[s.tensor][0]
        if any(lo < s.slab_offset + s.nbytes and s.slab_offset < hi for lo, hi in carried):
            continue
        if key in SAMPLE[:3]:
            want = gen_range(1, key, s.kind, s.index_base, s.nbytes // (2 if s.kind == 0 else 4))
            if not np.array_equal(slab[s.slab_offset:s.slab_offset + s.nbytes].view(want.dtype), want):
                print(f"[rank {rank}] slab bytes mismatch {key}/{s.kind}", flush=True)
                bad += 1
    b.switch_to(a)
    if not torch.equal(dev_checksums(plans[0], a, rank), ck_a):
        print(f"[rank {rank}] A restore mismatch", flush=True)
        bad += 1
    # collective weight sync of A
    arena = mgr.arena(plans[0])
    a.sync(arena)
    views = P.StateManager.rollout_views(plans[0], rank, arena)
    shapes = dict(man)
    for key in SAMPLE:
        keys = [key]
        if ".q_proj." in key:
            keys += [key.replace(".q_proj.", ".k_proj."), key.replace(".q_proj.", ".v_proj.")]
        if ".gate_proj." in key:
            keys += [key.replace(".gate_proj.", ".up_proj.")]
        cast = {k: O.rne_bf16(gen_tensor(1, k, 1, shapes[k])) for k in keys}
        want = O.rollout_tensors(cast, tp, dp, 1, rank, rmap, shape.head_dim)
        for name, x in want.items():
            if not np.array_equal(bits_np(views[name]), x):
                print(f"[rank {rank}] sync mismatch {name}", flush=True)
                bad += 1
    # the NCCL-baseline transport must produce the same bytes at full size
    mgr_nccl = P.StateManager(device=local, rank=rank, world=world, sync_nccl=True, duplex=False)
    arena.fill_(0x5A)
    mgr_nccl.sync(plans[0], a.masters(), arena)
    views = P.StateManager.rollout_views(plans[0], rank, arena)
    for key in SAMPLE:
        keys = [key]
        if ".q_proj." in key:
            keys += [key.replace(".q_proj.", ".k_proj."), key.replace(".q_proj.", ".v_proj.")]
        if ".gate_proj." in key:
            keys += [key.replace(".gate_proj.", ".up_proj.")]
        cast = {k: O.rne_bf16(gen_tensor(1, k, 1, shapes[k])) for k in keys}
        want = O.rollout_tensors(cast, tp, dp, 1, rank, rmap, shape.head_dim)
        for name, x in want.items():
            if not np.array_equal(bits_np(views[name]), x):
                print(f"[rank {rank}] nccl sync mismatch {name}", flush=True)
                bad += 1
    mgr_nccl.close()
    if rank == 0:
        print(f"carried buckets per job: {len(plans[0].carry())}, rank map {rmap}", flush=True)
    del a, b, arena, views
    torch.cuda.empty_cache()
    # NEXT-2 ZeRO-2 replicas at full size: dedup slab + NVLink all-gather
    rp = mgr.plan(man, replica_param=True)
    r = P.Job(mgr, rp, seed=3).alloc().init_synthetic()
    ck_p = torch.zeros((len(man), 2), dtype=torch.int64, device="cuda")
    for t_, (key, _) in enumerate(man):
        P.checksum(r.shards[(key, 0)], 0, out=ck_p[t_])
    r.suspend()
    r.resume()
    ck_p2 = torch.zeros_like(ck_p)
    for t_, (key, _) in enumerate(man):
        P.checksum(r.shards[(key, 0)], 0, out=ck_p2[t_])
    if not torch.equal(ck_p, ck_p2):
        print(f"[rank {rank}] replica restore mismatch", flush=True)
        bad += 1
    for key in SAMPLE[:3]:
        if not np.array_equal(bits_np(r.shards[(key, 0)]).reshape(-1), gen_tensor(3, key, 0, shapes[key]).reshape(-1)):
            print(f"[rank {rank}] replica sample mismatch {key}", flush=True)
            bad += 1
    del r
    t = torch.tensor([bad], device=f"cuda:{local}")
    dist.all_reduce(t)
    mgr.close()
    dist.destroy_process_group()
    if rank == 0:
        print(f"mp_fullsize_worker {MODEL} world={world} mismatches={int(t.item())}", flush=True)
    sys.exit(1 if int(t.item()) else 0)


if __name__ == "__main__":
    main()
