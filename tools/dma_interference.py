#!/usr/bin/env python
"""Does copy-engine traffic slow an HBM-bound kernel?  The fused cast+push of
the weight sync (no copies of its own) timed per launch (PLEX_CTX_TIMING) with
the copy engines idle, then with a background loop of pinned D2H and/or H2D
copies on other streams -- the situation the pack/unpack kernels are always in
inside a switch.

    python tools/dma_interference.py [--model qwen2.5-3b]
"""
import argparse
import json
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_20863_b200 as P  # noqa: E402
from plexgen import MODELS, manifest  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-3b")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    mgr = P.StateManager(device=0, bucket_bytes=64 << 20, timing=True, bootstrap=False)
    plan = mgr.plan(manifest(a.model), head_dim=MODELS[a.model].head_dim, tp=1, dp=1)
    job = P.Job(mgr, plan, seed=0, slab=False).alloc(kinds=(1,)).init_synthetic()
    arena = mgr.arena(plan)
    n = 2 << 30
    hb = torch.empty(n, dtype=torch.uint8).pin_memory()
    db = torch.empty(n, dtype=torch.uint8, device="cuda")
    hb2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    db2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    out = {"model": a.model}
    for mode in ("idle", "d2h", "h2d", "both", "idle_again"):
        stop = threading.Event()
        streams = []

        def loop(kind):
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                while not stop.is_set():
                    if kind == "d2h":
                        hb.copy_(db, non_blocking=True)
                    else:
                        db2.copy_(hb2, non_blocking=True)
                    s.synchronize()

        ths = []
        if mode in ("d2h", "both"):
            ths.append(threading.Thread(target=loop, args=("d2h",)))
        if mode in ("h2d", "both"):
            ths.append(threading.Thread(target=loop, args=("h2d",)))
        for t in ths:
            t.start()
        torch.cuda.synchronize()
        job.sync(arena)                                  # warm
        mgr.reset_stats()
        for _ in range(a.reps):
            job.sync(arena)
        st = mgr.stats()["push"]
        stop.set()
        for t in ths:
            t.join()
        out[mode] = {"push_GBs": round(st["bytes"] / (st["ms"] * 1e-3) / 1e9, 1),
                     "ms_per_launch": round(st["ms"] / max(1, st["launches"]), 3)}
    print(json.dumps(out), flush=True)
    mgr.close()


if __name__ == "__main__":
    main()
