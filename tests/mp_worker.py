"""torchrun worker for the multi-GPU parity test (tests/test_gpu_multi.py).

Each rank: bootstraps the library's NCCL communicator over torch.distributed,
runs the real collective plex_weight_sync (CUDA-IPC peer-mapped arenas, fused
cast + NVLink push) and a suspend/resume round trip of its own shards, and
checks both bit-exactly against the CPU oracle.  Exit code 0 = all ranks ok.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import paper_2605_20863_b200 as P  # noqa: E402
from oracle import plex_oracle as O  # noqa: E402
from plexgen import MODELS, manifest  # noqa: E402
from _state import full_state, fsdp_shards, master_shards  # noqa: E402


def bits_np(t):
    t = t.detach().contiguous().cpu()
    return t.view(torch.int16).numpy().view(np.uint16) if t.element_size() == 2 else t.view(torch.int32).numpy().view(np.uint32)


def main():
    import faulthandler
    faulthandler.dump_traceback_later(900, exit=True)     # never hang a GPU box silently
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    mgr = P.StateManager(device=local, rank=rank, world=world, bucket_bytes=1 << 16, n_slots=2)
    # NCCL-baseline transport; tiny staging forces many exchange rounds
    mgr_nccl = P.StateManager(device=local, rank=rank, world=world, bucket_bytes=1 << 16, n_slots=2, sync_nccl=True)
    bad = 0
    cases = [("mid", 2 if world % 2 == 0 else 1, 1), ("mid-moe", 2 if world % 2 == 0 else 1, world),
             ("toy-odd", 1, 1)]
    for model, tp, ep in cases:
        dp = world // tp
        hd = MODELS[model].head_dim
        for rank_map in (0, 1):
            plan = mgr.plan(manifest(model), head_dim=hd, tp=tp, dp=dp, ep=ep, rank_map=rank_map, tile_bytes=2048)
            job = P.Job(mgr, plan, seed=21).alloc().init_synthetic(special_bits=3)
            arena = mgr.arena(plan)
            arena.fill_(0xCD)
            for _ in range(2):                              # second call reuses mapped peers
                job.sync(arena)
            full = full_state(model, seed=21, special_bits=3)
            want = O.weight_sync(master_shards(full, world, O.fsdp_rows), tp, dp, ep, rank_map, hd)[rank]
            for name, v in P.StateManager.rollout_views(plan, rank, arena).items():
                if not np.array_equal(bits_np(v), want[name]):
                    print(f"[rank {rank}] sync mismatch {model} map={rank_map} {name}", flush=True)
                    bad += 1
            arena.fill_(0xCD)
            for _ in range(2):
                mgr_nccl.sync(plan, job.masters(), arena)
            for name, v in P.StateManager.rollout_views(plan, rank, arena).items():
                if not np.array_equal(bits_np(v), want[name]):
                    print(f"[rank {rank}] nccl-sync mismatch {model} map={rank_map} {name}", flush=True)
                    bad += 1
            # suspend / resume of this rank's shards
            before = {k: bits_np(v) for k, v in job.shards.items()}
            job.suspend()
            segs, size = O.slab_layout(manifest(model), world, rank)
            osh = fsdp_shards(full, world, rank, O.fsdp_rows)
            if not np.array_equal(job.slab.host_bytes(), O.pack_slab(segs, size, osh)):
                print(f"[rank {rank}] slab mismatch {model}", flush=True)
                bad += 1
            job.resume()
            for k, v in job.shards.items():
                if not np.array_equal(bits_np(v), before[k]):
                    print(f"[rank {rank}] restore mismatch {model} {k}", flush=True)
                    bad += 1
            del arena
    # NEXT-2 replicated (ZeRO-2) params: dedup slab + collective NVLink all-gather,
    # interleaved with a rollout sync so both peer-mapped arena roles stay live
    for model in ("mid", "toy-odd"):
        man = manifest(model)
        hd = MODELS[model].head_dim
        plan = mgr.plan(man, head_dim=hd, tp=1, dp=world, replica_param=True, tile_bytes=2048)
        job = P.Job(mgr, plan, seed=33).alloc().init_synthetic(special_bits=3)
        arena = mgr.arena(plan)
        full = full_state(model, seed=33, special_bits=3)
        want_sync = O.weight_sync(master_shards(full, world, O.fsdp_rows), 1, world, 1, 0, hd)[rank]
        osh = fsdp_shards(full, world, rank, O.fsdp_rows)
        segs, size = O.slab_layout(man, world, rank)
        for it in range(2):
            job.sync(arena)
            for name, v in P.StateManager.rollout_views(plan, rank, arena).items():
                if not np.array_equal(bits_np(v), want_sync[name]):
                    print(f"[rank {rank}] replica-plan sync mismatch {model} {name}", flush=True)
                    bad += 1
            job.suspend()
            if not np.array_equal(job.slab.host_bytes(), O.pack_slab(segs, size, osh)):
                print(f"[rank {rank}] dedup slab mismatch {model}", flush=True)
                bad += 1
            job.resume()                                    # onload own rows + all-gather
            for (k, kd), v in job.shards.items():
                want = full[(k, kd)] if kd == 0 else osh[(k, kd)]
                if not np.array_equal(bits_np(v), want):
                    print(f"[rank {rank}] replica restore mismatch {model} {k}/{kd} iter {it}", flush=True)
                    bad += 1
        del arena, job
    # NEXT-1 in-place swap of two same-layout jobs on every rank, then the collective sync
    man = manifest("mid")
    plan = mgr.plan(man, head_dim=MODELS["mid"].head_dim, tp=1, dp=world, tile_bytes=2048)
    ja = P.Job(mgr, plan, seed=41, slab=False).alloc()
    jb = P.Job(mgr, plan, seed=42)
    jb.shards = ja.shards
    jb.init_synthetic(special_bits=3)
    jb.suspend(release=False)
    jb.shards = type(ja.shards)()
    ja.init_synthetic(special_bits=3)
    arena = mgr.arena(plan)
    for it, (out, inc, seed_in) in enumerate(((ja, jb, 42), (jb, ja, 41))):
        out.swap_with(inc)
        inc.sync(arena)
        full = full_state("mid", seed=seed_in, special_bits=3)
        osh = fsdp_shards(full, world, rank, O.fsdp_rows)
        for k, v in inc.shards.items():
            if not np.array_equal(bits_np(v), osh[k]):
                print(f"[rank {rank}] swap restore mismatch {k} iter {it}", flush=True)
                bad += 1
        want = O.weight_sync(master_shards(full, world, O.fsdp_rows), 1, world, 1, 0, MODELS["mid"].head_dim)[rank]
        for name, v in P.StateManager.rollout_views(plan, rank, arena).items():
            if not np.array_equal(bits_np(v), want[name]):
                print(f"[rank {rank}] sync after swap mismatch {name} iter {it}", flush=True)
                bad += 1
    del arena, ja, jb
    # a1 through the library's group executor with the real collectives: three
    # jobs (one with replicated ZeRO-2 params) time-slicing the group; the op
    # lists must equal the oracle's transition_ops, every sync the oracle's
    # weight_sync, every restored state the oracle's shards
    specs = [("mid", 2 if world % 2 == 0 else 1, 1, False, 51), ("mid-moe", 2 if world % 2 == 0 else 1, world, False, 52),
             ("toy", 1, 1, True, 53)]
    group = P.Group(mgr)
    gjobs, garenas, gwant = [], [], []
    for model, tp, ep, rep, seed in specs:
        hd = MODELS[model].head_dim
        plan = mgr.plan(manifest(model), head_dim=hd, tp=tp, dp=world // tp, ep=ep, replica_param=rep,
                        tile_bytes=2048)
        job = P.Job(mgr, plan, seed=seed).alloc().init_synthetic(special_bits=3)
        job.suspend()                                        # every job starts HOST-resident
        group.add(job)
        full = full_state(model, seed=seed, special_bits=3)
        gjobs.append(job)
        garenas.append(mgr.arena(plan))
        gwant.append((full, O.weight_sync(master_shards(full, world, O.fsdp_rows), tp, world // tp, ep, 0, hd)[rank]))
    resident = None
    for j in (0, 1, 2, 0, 2, 1, 1):
        res = group.transition(gjobs[j])
        if res["ops"] != O.transition_ops(resident, j):
            print(f"[rank {rank}] group ops {res['ops']} != oracle {O.transition_ops(resident, j)}", flush=True)
            bad += 1
        resident = j
        garenas[j].fill_(0xCD)
        res = group.transition(gjobs[j], sync=garenas[j])        # collective sync through the executor
        if res["ops"] != [(O.OP_SYNC, j)]:
            bad += 1
        full, want = gwant[j]
        for name, v in P.StateManager.rollout_views(gjobs[j].plan, rank, garenas[j]).items():
            if not np.array_equal(bits_np(v), want[name]):
                print(f"[rank {rank}] group sync mismatch job {j} {name}", flush=True)
                bad += 1
        osh = fsdp_shards(full, world, rank, O.fsdp_rows)
        for (k, kd), v in gjobs[j].shards.items():
            w = full[(k, kd)] if (kd == 0 and specs[j][3]) else osh[(k, kd)]
            if not np.array_equal(bits_np(v), w):
                print(f"[rank {rank}] group restore mismatch job {j} {k}/{kd}", flush=True)
                bad += 1
    group.close()
    del gjobs, garenas
    t = torch.tensor([bad], device=f"cuda:{local}")
    dist.all_reduce(t)
    mgr.close()
    mgr_nccl.close()
    dist.destroy_process_group()
    if rank == 0:
        print(f"mp_worker world={world} mismatches={int(t.item())}", flush=True)
    sys.exit(1 if int(t.item()) else 0)


if __name__ == "__main__":
    main()
