#!/usr/bin/env python
"""nccl-tests-style context rows: plain NCCL all-gather and
all-to-all over the GPUs of one box at the message sizes of the weight sync,
timed with CUDA events (max over ranks).  Context for the sync's NVLink
roofline, not part of the product path.

    torchrun --nproc-per-node N tools/nccl_context.py [--model qwen2.5-7b]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2605_20863_b200 import Plan  # noqa: E402
from plexgen import MODELS, manifest  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / reps], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-7b")
    ap.add_argument("--tp", type=int, default=2)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    tp = min(a.tp, world)
    plan = Plan(manifest(a.model), head_dim=MODELS[a.model].head_dim, world=world, tp=tp, dp=world // tp,
                rank_map=2)
    infos = [plan.rank_info(g) for g in range(world)]
    recv_max = max(i.recv_bytes for i in infos)
    send_max = max(i.send_bytes for i in infos)
    # all-gather of each rank's bf16 shard of the whole model (the TP-1 sync, N2)
    shard = plan.stats().total_params * 2 // world
    shard -= shard % 256
    x = torch.empty(shard, dtype=torch.uint8, device="cuda")
    y = torch.empty(shard * world, dtype=torch.uint8, device="cuda")
    ms_ag = timed(lambda: dist.all_gather_into_tensor(y, x))
    # uniform all-to-all moving the sync's max(send, recv) per rank (N1/N3)
    per_peer = max(recv_max, send_max) // max(1, world - 1)
    per_peer -= per_peer % 256
    s = torch.empty(per_peer * world, dtype=torch.uint8, device="cuda")
    r = torch.empty_like(s)
    ms_a2a = timed(lambda: dist.all_to_all_single(r, s))
    if rank == 0:
        line = {"tool": "nccl_context", "model": a.model, "n_gpus": world,
                "all_gather": {"bytes_in_per_rank": shard, "ms": round(ms_ag, 3),
                               "recv_GBs_per_rank": round(shard * (world - 1) / (ms_ag * 1e-3) / 1e9, 1)},
                "all_to_all": {"bytes_per_peer": per_peer, "ms": round(ms_a2a, 3),
                               "recv_GBs_per_rank": round(per_peer * (world - 1) / (ms_a2a * 1e-3) / 1e9, 1)},
                "sync_ledger": {"layout": f"FSDP-{world}->TP-{tp}xDP-{world // tp}", "recv_max": recv_max,
                                "send_max": send_max}}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
