#!/usr/bin/env python
"""Kernel / copy-engine timeline of one context switch (CUDA events recorded
by the library around every pack/unpack launch and every bucket D2H/H2D copy,
PLEX_CTX_TIMING): the evidence that the copy engines run back to back at the
host-link rate, that the two directions of a duplex switch overlap, and that
the pack/unpack kernels hide under the copies.

    python tools/timeline.py --model qwen2.5-1.5b --bucket-mb 512 [--sequential]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_20863_b200 as P  # noqa: E402
from plexgen import manifest  # noqa: E402


def busy(iv):
    """Total length of the union of intervals."""
    tot, end = 0.0, -1e30
    for a, b in sorted(iv):
        if b <= end:
            continue
        tot += b - max(a, end)
        end = b
    return tot


def overlap(x, y):
    return busy(x) + busy(y) - busy(x + y)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-1.5b")
    ap.add_argument("--bucket-mb", type=int, default=512)
    ap.add_argument("--sequential", action="store_true", help="offload then onload instead of the duplex switch")
    ap.add_argument("--swap", action="store_true", help="in-place swap (one device copy, one slab): bench N=1 mode")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    mgr = P.StateManager(device=0, bucket_bytes=a.bucket_mb << 20, n_slots=2, timing=True, bootstrap=False)
    if a.swap:
        plan = mgr.plan(manifest(a.model))
        jobs = [P.Job(mgr, plan, seed=0, slab=False).alloc(), P.Job(mgr, plan, seed=1)]
        jobs[1].shards = jobs[0].shards
        jobs[1].init_synthetic()
        jobs[1].suspend(release=False)
        jobs[1].shards = type(jobs[0].shards)()
        jobs[0].init_synthetic()
        for _ in range(2):
            jobs[0].swap_with(jobs[1])
            jobs[1].swap_with(jobs[0])
    else:
        plans = [mgr.plan(manifest(a.model)) for _ in range(2)]
        jobs = [P.Job(mgr, pl, seed=s).alloc().init_synthetic() for pl, s in zip(plans, (0, 1))]
        jobs[1].suspend()
        for _ in range(2):                               # warm up both directions
            jobs[0].switch_to(jobs[1])
            jobs[1].switch_to(jobs[0])
    torch.cuda.synchronize()
    mgr.reset_stats()
    if a.swap:
        jobs[0].swap_with(jobs[1])
    elif a.sequential:
        jobs[0].suspend()
        jobs[1].resume()
    else:
        jobs[0].switch_to(jobs[1])
    recs = mgr.timeline()
    t0 = min(r["start_ms"] for r in recs if r["call"] == 0)
    lanes = {}
    for r in recs:
        # every call's records are relative to its own first launch; lay calls end to end
        lanes.setdefault(r["kind"], []).append(r)
    if a.sequential:                                     # call 1 starts after call 0 ends
        end0 = max(r["start_ms"] + r["ms"] for r in recs if r["call"] == 0)
        for r in recs:
            if r["call"] == 1:
                r["start_ms"] += end0
    iv = {k: [(r["start_ms"] - t0, r["start_ms"] - t0 + r["ms"]) for r in v] for k, v in lanes.items()}
    span = max(b for v in iv.values() for _, b in v)
    summ = {"model": a.model, "mode": "swap" if a.swap else "sequential" if a.sequential else "duplex",
            "bucket_MiB": a.bucket_mb,
            "span_ms": round(span, 2)}
    for k, v in iv.items():
        byts = sum(r["bytes"] for r in lanes[k])
        summ[k] = {"n": len(v), "busy_ms": round(busy(v), 2), "GBs_while_busy": round(byts / busy(v) / 1e6, 1),
                   "busy_frac_of_span": round(busy(v) / span, 3)}
    if "d2h" in iv and "h2d" in iv:
        summ["d2h_h2d_overlap_ms"] = round(overlap(iv["d2h"], iv["h2d"]), 2)
        # one direction alone at the ends: before the first D2H starts / after the last H2D ends
        summ["head_ms_before_first_d2h"] = round(min(x for x, _ in iv["d2h"]), 2)
        summ["tail_ms_after_last_h2d"] = round(span - max(y for _, y in iv["h2d"]), 2)
        summ["swap_pieces_env"] = os.environ.get("PLEX_SWAP_PIECES", "default")
    kern = iv.get("pack", []) + iv.get("unpack", [])
    copies = iv.get("d2h", []) + iv.get("h2d", [])
    if kern and copies:
        summ["kernel_ms_hidden_under_copies"] = round(overlap(kern, copies), 2)
        summ["kernel_ms_total"] = round(busy(kern), 2)
    # text gantt: one row per lane, 100 columns over the span
    rows = []
    for k in ("pack", "d2h", "h2d", "unpack", "derive"):
        if k not in iv:
            continue
        line = [" "] * 100
        for s_, e_ in iv[k]:
            for col in range(int(s_ / span * 100), min(100, int(e_ / span * 100) + 1)):
                line[col] = "#"
        rows.append(f"{k:>7} |{''.join(line)}|")
    text = json.dumps(summ) + "\n" + "\n".join(rows) + "\n" + json.dumps(
        [{**r, "start_ms": round(r["start_ms"] - t0, 3)} for r in recs]) + "\n"
    print(text, flush=True)
    if a.out:
        with open(a.out, "a") as f:
            f.write(text)
    mgr.close()


if __name__ == "__main__":
    main()
