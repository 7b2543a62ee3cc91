#!/usr/bin/env python
"""Fused cast + reshard push (a8-a11) driven from ONE process over N GPUs.

Every rank r of an FSDP-N -> TP x DP sync gets its own ctx on cuda:r; the
destination arenas live on their own GPUs and every rank's push kernel stores
into them through CUDA peer access (NVLink), exactly the kernel and items of
plex_weight_sync, without NCCL barriers.  Because it is a single process, the
push kernels can be captured by ncu with DRAM and NVLink counters (never wrap
a multi-rank torchrun command in ncu; B200_PROFILING.md):

    python tools/push_probe.py --gpus 4 --model qwen2.5-7b --tp 2
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
nvltx__bytes.sum,nvlrx__bytes.sum -k regex:push_kernel python tools/push_probe.py --gpus 4 --steps 1 --warmup 0

--only row restricts the manifest to the row-parallel tensors (o_proj,
down_proj: the strided 2-D rectangles), --only col to the rest.  One JSON line
per run: per-rank push time (library CUDA events), the NVLink bytes of the
busiest rank and the kernel's roofline (slower of HBM and NVLink).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_20863_b200 as P  # noqa: E402
from paper_2605_20863_b200 import _lib as L  # noqa: E402
from plexgen import MODELS, manifest  # noqa: E402


def enable_peers(n: int) -> None:
    from cuda.bindings import runtime as rt
    for r in range(n):
        torch.cuda.set_device(r)
        for g in range(n):
            if g != r:
                err, ok = rt.cudaDeviceCanAccessPeer(r, g)
                if not ok:
                    raise SystemExit(f"cuda:{r} cannot access cuda:{g}")
                (e,) = rt.cudaDeviceEnablePeerAccess(g, 0)
                if e not in (rt.cudaError_t.cudaSuccess, rt.cudaError_t.cudaErrorPeerAccessAlreadyEnabled):
                    raise SystemExit(f"cudaDeviceEnablePeerAccess({r}->{g}): {e}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=4)
    ap.add_argument("--model", default="qwen2.5-7b")
    ap.add_argument("--tp", type=int, default=2)
    ap.add_argument("--ep", type=int, default=1)
    ap.add_argument("--rank-map", default="auto", choices=["tp", "dp", "auto"])
    ap.add_argument("--only", default="all", choices=["all", "row", "col"])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--tile-kb", type=int, default=64)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    N = a.gpus
    assert torch.cuda.device_count() >= N, torch.cuda.device_count()
    man = manifest(a.model)
    row = lambda k: k.endswith(("self_attn.o_proj.weight", "mlp.down_proj.weight")) and ".experts." not in k  # noqa: E731
    if a.only == "row":
        man = [(k, s) for k, s in man if row(k)]
    elif a.only == "col":
        man = [(k, s) for k, s in man if not row(k)]
    rank_map = {"tp": L.RANKMAP_TP_FAST, "dp": L.RANKMAP_DP_FAST, "auto": L.RANKMAP_AUTO}[a.rank_map]
    plan = P.Plan(man, head_dim=MODELS[a.model].head_dim, world=N, tp=a.tp, dp=N // a.tp, ep=a.ep,
                  rank_map=rank_map, tile_bytes=a.tile_kb << 10)
    enable_peers(N)
    mgrs, masters, arenas = [], [], []
    for r in range(N):
        torch.cuda.set_device(r)
        m = P.StateManager(device=r, rank=r, world=N, bucket_bytes=1 << 20, bootstrap=False, timing=True)
        job = P.Job(m, plan, seed=1, rank=r, slab=False).alloc(kinds=(1,)).init_synthetic()
        mgrs.append(m)
        masters.append(job.masters())
        arenas.append(m.arena(plan, r))
    for r in range(N):
        torch.cuda.synchronize(r)
    bar = threading.Barrier(N)
    wall = []

    def rank_loop(r: int, n: int):
        torch.cuda.set_device(r)
        for _ in range(n):
            bar.wait()
            t0 = time.perf_counter()
            mgrs[r].sync_rank(plan, r, masters[r], arenas)         # blocking; stores land in peers' HBM
            bar.wait()
            if r == 0:
                wall.append(time.perf_counter() - t0)

    def run(n: int):
        th = [threading.Thread(target=rank_loop, args=(r, n)) for r in range(N)]
        for t in th:
            t.start()
        for t in th:
            t.join()

    run(a.warmup)
    for m in mgrs:
        m.reset_stats()
    wall.clear()
    run(a.steps)
    per_rank = []
    for r in range(N):
        st = mgrs[r].stats()["push"]
        info = plan.rank_info(r)
        ms = st["ms"] / max(1, st["launches"])
        per_rank.append({"rank": r, "push_ms": round(ms, 3), "send_bytes": info.send_bytes,
                         "recv_bytes": info.recv_bytes, "local_bytes": info.local_bytes,
                         "src_read_bytes": info.src_read_bytes, "items": info.n_push_items})
    t_max = max(p["push_ms"] for p in per_rank)
    link = max(max(p["send_bytes"], p["recv_bytes"]) for p in per_rank)
    hbm = max(p["src_read_bytes"] + p["local_bytes"] + p["recv_bytes"] for p in per_rank)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    t_hbm = hbm / (peaks["hbm_gbs"] * 1e9) * 1e3
    t_nvl = link / 770e9 * 1e3
    line = {"probe": "push", "model": a.model, "only": a.only, "n_gpus": N, "tp": a.tp, "dp": N // a.tp,
            "ep": a.ep, "rank_map": ["tp_fast", "dp_fast"][plan.stats().rank_map], "tile_kb": a.tile_kb,
            "steps": a.steps, "push_ms_max_rank": t_max, "wall_ms_median": round(1e3 * sorted(wall)[len(wall) // 2], 3),
            "nvlink_bytes_max_rank": link, "nvlink_gbs": round(link / (t_max * 1e-3) / 1e9, 1),
            "nvlink_frac_of_770": round(link / (t_max * 1e-3) / 1e9 / 770.0, 4),
            "hbm_bytes_max_rank": hbm, "hbm_gbs": round(hbm / (t_max * 1e-3) / 1e9, 1),
            "lower_bound_ms": round(max(t_hbm, t_nvl), 3), "bound": "nvlink" if t_nvl >= t_hbm else "hbm",
            "frac_of_bound": round(max(t_hbm, t_nvl) / t_max, 4), "per_rank": per_rank}
    print(json.dumps(line), flush=True)
    if a.out:
        with open(a.out, "a") as f:
            f.write(json.dumps(line) + "\n")
    for m in mgrs:
        m.close()


if __name__ == "__main__":
    main()
