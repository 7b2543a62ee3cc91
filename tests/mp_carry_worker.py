"""torchrun worker: NEXT-1 host-link balancing (carried buckets), bit-exact.

Rank 0 is given a 4x slower host link, so it hands its last buckets over NVLink
to the other ranks, which keep them in their carry regions.  Checked: every
owner slab byte that it stores itself and every carried byte in the carriers'
regions equal the oracle's canonical slab; resume restores every shard; the
duplex switch between two jobs with carried buckets restores both.
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
from _state import full_state, fsdp_shards  # noqa: E402


def bits_np(t):
    t = t.detach().contiguous().cpu()
    return t.view(torch.int16).numpy().view(np.uint16) if t.element_size() == 2 else t.view(torch.int32).numpy().view(np.uint32)


def main():
    import faulthandler
    faulthandler.dump_traceback_later(600, exit=True)
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    bad = 0
    for carry_nccl in (False, True):          # peer-memory transport (default), NCCL baseline
        bad += run(rank, world, local, carry_nccl)
    t = torch.tensor([bad], device=f"cuda:{local}")
    dist.all_reduce(t)
    dist.destroy_process_group()
    if rank == 0:
        print(f"mp_carry_worker world={world} mismatches={int(t.item())}", flush=True)
    sys.exit(1 if int(t.item()) else 0)


def run(rank, world, local, carry_nccl):
    bucket = 1 << 16
    mgr = P.StateManager(device=local, rank=rank, world=world, bucket_bytes=bucket, n_slots=2, carry_nccl=carry_nccl)
    weights = [1.0] + [4.0] * (world - 1)
    bad = 0
    models = ("mid", "mid-moe")
    plans = [mgr.plan(manifest(mo), head_dim=MODELS[mo].head_dim, bucket_bytes=bucket, tile_bytes=2048,
                      link_weights=weights) for mo in models]
    for pl in plans:
        mgr.enable_carry(pl)
    assert plans[0].carry(), "expected carried buckets"
    jobs = [P.Job(mgr, pl, seed=80 + j).alloc().init_synthetic(special_bits=3) for j, pl in enumerate(plans)]
    fulls = [full_state(mo, seed=80 + j, special_bits=3) for j, mo in enumerate(models)]

    def check_slabs(j):
        nonlocal bad
        man = manifest(models[j])
        pl = plans[j]
        # every rank's canonical slab from the oracle
        want = []
        for r in range(world):
            segs, size = O.slab_layout(man, world, r)
            want.append(O.pack_slab(segs, size, fsdp_shards(fulls[j], world, r, O.fsdp_rows)))
        carried = pl.carry()
        own = jobs[j].slab.host_bytes()
        for b in range(pl.rank_info(rank).n_buckets):
            lo = b * bucket
            if any(x.owner == rank and x.bucket == b for x in carried):
                continue
            hi = min(lo + bucket, own.size)
            if not np.array_equal(own[lo:hi], want[rank][lo:hi]):
                print(f"[rank {rank}] own bucket {b} mismatch job {j}", flush=True)
                bad += 1
        reg = jobs[j].slab.carry_bytes()
        for x in carried:
            if x.carrier == rank:
                got = reg[x.carry_offset:x.carry_offset + x.bytes]
                if not np.array_equal(got, want[x.owner][x.slab_offset:x.slab_offset + x.bytes]):
                    print(f"[rank {rank}] carried bucket {x.owner}/{x.bucket} mismatch job {j}", flush=True)
                    bad += 1

    def check_shards(j):
        nonlocal bad
        osh = fsdp_shards(fulls[j], world, rank, O.fsdp_rows)
        for k, v in jobs[j].shards.items():
            if not np.array_equal(bits_np(v), osh[k]):
                print(f"[rank {rank}] shard mismatch job {j} {k}", flush=True)
                bad += 1

    jobs[1].suspend()                       # collective: carried buckets cross NVLink
    check_slabs(1)
    jobs[0].suspend()
    check_slabs(0)
    jobs[0].resume()
    check_shards(0)
    jobs[0].switch_to(jobs[1])              # duplex switch, both halves carrying
    check_slabs(0)
    check_shards(1)
    jobs[1].switch_to(jobs[0])
    check_shards(0)
    for _ in range(3):                      # repeated calls reuse the carry slots and flags
        jobs[0].switch_to(jobs[1])
        jobs[1].switch_to(jobs[0])
    check_shards(0)
    check_slabs(1)
    mgr.close()
    if rank == 0:
        print(f"transport={'nccl' if carry_nccl else 'peer-memory'} carried={len(plans[0].carry())} "
              f"mismatches(rank0)={bad}", flush=True)
    return bad


if __name__ == "__main__":
    main()
