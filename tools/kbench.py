#!/usr/bin/env python
"""Kernel micro-benchmark: K1 pack / K2 unpack / push throughput per launch
(CUDA events around every launch, PLEX_CTX_TIMING) for several bucket sizes,
plus torch's own copy kernel on the same bytes as a reference.

    PLEX_PACK_VARIANT=<v> python tools/kbench.py --model qwen2.5-0.5b --buckets 256,1024
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_20863_b200 as P  # noqa: E402
from plexgen import MODELS, manifest  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-0.5b")
    ap.add_argument("--buckets", default="256,1024")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ballast-gb", type=int, default=0, help="occupy this much HBM first (experiment)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    ballast = torch.empty(a.ballast_gb << 30, dtype=torch.uint8, device="cuda") if a.ballast_gb else None
    out = {"ballast_gb": a.ballast_gb, "variant": os.environ.get("PLEX_PACK_VARIANT", "0"), "model": a.model}
    for bmb in [int(x) for x in a.buckets.split(",")]:
        mgr = P.StateManager(device=0, bucket_bytes=bmb << 20, n_slots=2, timing=True, duplex=False,
                             bootstrap=False)
        plan = mgr.plan(manifest(a.model), head_dim=MODELS[a.model].head_dim, tp=1, dp=1)
        job = P.Job(mgr, plan, seed=0).alloc().init_synthetic()
        arena = mgr.arena(plan)
        job.suspend(release=False)
        job.resume()
        job.sync(arena)
        mgr.reset_stats()
        for _ in range(a.reps):
            job.suspend(release=False)
            job.resume()
            job.sync(arena)
        st = mgr.stats()
        res = {}
        for k in ("pack", "unpack", "push", "d2h", "h2d"):
            v = st[k]
            if v["launches"]:
                res[k] = {"GBs": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1),
                          "us_per_launch": round(1e3 * v["ms"] / v["launches"], 2),
                          "MB_per_launch": round(v["bytes"] / v["launches"] / 1e6, 2)}
        tr = [(k, round(ms * 1e3, 1), round(b / (ms * 1e-3) / 1e9)) for k, ms, b in mgr.trace()
              if k in ("pack", "unpack")]
        res["per_launch_us_GBs"] = tr[:64]
        out[f"bucket_{bmb}MiB"] = res
        del job, arena, plan
        mgr.close()
        torch.cuda.empty_cache()
    # reference: torch copy of a 1 GiB buffer (read + write bytes)
    x = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        y.copy_(x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        y.copy_(x)
    e1.record()
    e1.synchronize()
    out["torch_copy_GBs"] = round(2 * x.numel() * 10 / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
