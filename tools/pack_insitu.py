#!/usr/bin/env python
"""Where does the K1/K2 in-situ gap come from?

In the N=1 bench the pack / unpack kernels run at ~0.93 of the measured HBM
copy while the same kernel isolated under ncu runs at ~1.02.  This tool
launches the exact bucket kernels of the bench's 7B FSDP-1 plan through
plex_diag_pack (one launch per 2 GiB bucket, no copies, no verification) and
times every launch with CUDA events on the launching stream, under:

  b2b       launches back to back, nothing else on the GPU
  b2b+dma   the same while both copy engines stream 2 GiB pinned copies
            (D2H and H2D at once, as during the in-place swap)
  gap       a ~5 ms spin gap between launches (the bench's kernels wait
            ~45 ms for their copies), nothing else
  gap+dma   gaps and both copy engines busy: the bench's situation

for each kernel build (variant 0 = default, 1 = L2::evict_first on the bulk
copies), pack and unpack.  torch's own 2 GiB copy is timed in b2b and b2b+dma
as the reference.  One JSON line per (variant, direction, mode).

    python tools/pack_insitu.py --model qwen2.5-7b --out gpurun_out/pack_insitu.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_20863_b200 as P  # noqa: E402
from paper_2605_20863_b200.state import diag_pack_variant  # noqa: E402
from plexgen import MODELS, manifest  # noqa: E402


def bucket_payload(plan, bucket_bytes):
    """Per bucket: data bytes, bf16 (PARAM) data bytes, number of segments touching it."""
    nb = plan.rank_info(0).n_buckets
    pay, bf16, nseg = [0] * nb, [0] * nb, [0] * nb
    for s in plan.segments(0):
        lo, hi = s.slab_offset, s.slab_offset + s.nbytes
        while lo < hi:
            b = lo // bucket_bytes
            e = min(hi, (b + 1) * bucket_bytes)
            pay[b] += e - lo
            if s.kind == 0:
                bf16[b] += e - lo
            nseg[b] += 1
            lo = e
    return pay, bf16, nseg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-7b")
    ap.add_argument("--bucket-mb", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--gap-ms", type=float, default=5.0)
    ap.add_argument("--variants", default="0,1")
    ap.add_argument("--out", default="")
    ap.add_argument("--shift-sweep", action="store_true", help="staging-offset sweep (gap mode) only")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    B = a.bucket_mb << 20
    mgr = P.StateManager(device=0, bucket_bytes=B, n_slots=2, bootstrap=False)           # 8 GiB staging
    plan = mgr.plan(manifest(a.model), head_dim=MODELS[a.model].head_dim, tp=1, dp=1)
    job = P.Job(mgr, plan, seed=1, slab=False).alloc().init_synthetic()
    pay, bf16, nseg = bucket_payload(plan, B)
    full = [k for k in range(len(pay)) if pay[k] > 0.9 * B]          # the full buckets (ragged tail excluded)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = float(peaks["hbm_gbs"])
    # background copy engines: 2 GiB pinned <-> device, both directions
    CB = 2 << 30
    h_src = torch.empty(CB, dtype=torch.uint8, pin_memory=True)
    h_dst = torch.empty(CB, dtype=torch.uint8, pin_memory=True)
    d_a = torch.empty(CB, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(CB, dtype=torch.uint8, device="cuda")
    s_k, s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    cyc_per_ms = peaks.get("sm_max_mhz", 1965.0) * 1e3
    torch.cuda.synchronize()

    def dma(n):
        with torch.cuda.stream(s_up):
            for _ in range(n):
                d_a.copy_(h_src, non_blocking=True)
        with torch.cuda.stream(s_dn):
            for _ in range(n):
                h_dst.copy_(d_b, non_blocking=True)

    def run(pack: bool, mode: str):
        ev = []
        n_launch = len(full) * a.reps
        mgr.diag_pack(plan, job.shards, full[0], pack, s_k)              # pointer table, untimed
        torch.cuda.synchronize()
        if "dma" in mode:
            per = (a.gap_ms if "gap" in mode else 0.75) * n_launch + 50.0
            dma(int(per / 40.0) + 2)                                     # ~40 ms per 2 GiB copy
        with torch.cuda.stream(s_k):
            if "dma" in mode:
                torch.cuda._sleep(int(5 * cyc_per_ms))                   # copies under way first
            for _ in range(a.reps):
                for k in full:
                    if "gap" in mode:
                        torch.cuda._sleep(int(a.gap_ms * cyc_per_ms))
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s_k)
                    mgr.diag_pack(plan, job.shards, k, pack, s_k, upload=False)
                    e1.record(s_k)
                    ev.append((e0, e1, 2 * pay[k], k))
        torch.cuda.synchronize()
        ms = [x.elapsed_time(y) for x, y, _, _ in ev]
        byt = sum(b for _, _, b, _ in ev)
        t = sum(ms)
        per_b = {}
        for (_, _, b, k), m in zip(ev, ms):
            per_b.setdefault(k, []).append(m)
        buckets = [{"bucket": k, "us": round(1e3 * sum(v) / len(v), 1),
                    "frac": round(2 * pay[k] / (sum(v) / len(v) * 1e-3) / 1e9 / hbm, 4),
                    "bf16_share": round(bf16[k] / pay[k], 3), "segments": nseg[k]} for k, v in sorted(per_b.items())]
        return {"launches": len(ms), "avg_us": round(1e3 * t / len(ms), 1), "GBs": round(byt / (t * 1e-3) / 1e9, 1),
                "frac": round(byt / (t * 1e-3) / 1e9 / hbm, 4), "min_us": round(1e3 * min(ms), 1),
                "max_us": round(1e3 * max(ms), 1), "per_bucket": buckets}

    def torch_copy(mode: str):
        n = 8
        if "dma" in mode:
            dma(4)
        x, y = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda"), torch.empty(1 << 30, dtype=torch.bfloat16,
                                                                                    device="cuda")
        ev = []
        with torch.cuda.stream(s_k):
            if "dma" in mode:
                torch.cuda._sleep(int(5 * cyc_per_ms))
            for _ in range(n):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s_k)
                y.copy_(x)
                e1.record(s_k)
                ev.append((e0, e1))
        torch.cuda.synchronize()
        ms = [a_.elapsed_time(b_) for a_, b_ in ev]
        del x, y
        return {"avg_us": round(1e3 * sum(ms) / n, 1), "GBs": round(4 * 2 ** 30 / (sum(ms) / n * 1e-3) / 1e9, 1)}

    out = []
    if a.shift_sweep:
        # staging-offset sweep in gap mode: single-tensor buckets vs normal ones, and torch's
        # copy of the same tensor bytes into the same staging addresses
        single = [k for k in full if nseg[k] <= 5]
        normal = [k for k in full if nseg[k] > 20][:2]
        stg = mgr.staging
        emb = job.shards[("model.embed_tokens.weight", 1)].view(torch.uint8).reshape(-1)[:B]
        for off in [0, 64 << 10, 256 << 10, 1 << 20, (2 << 20) + (64 << 10), (6 << 20) + (192 << 10),
                    (33 << 20) + (320 << 10), (1 << 30) + (2 << 20), 2 << 30, (3 << 30) + (4 << 10)]:
            res = {}
            for k in single + normal:
                mgr.diag_pack(plan, job.shards, k, True, s_k, staging_offset=off)
                torch.cuda.synchronize()
                ts = []
                with torch.cuda.stream(s_k):
                    for _ in range(3):
                        torch.cuda._sleep(int(a.gap_ms * cyc_per_ms))
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(s_k)
                        mgr.diag_pack(plan, job.shards, k, True, s_k, upload=False, staging_offset=off)
                        e1.record(s_k)
                        ts.append((e0, e1))
                torch.cuda.synchronize()
                res[k] = round(1e3 * sum(x.elapsed_time(y) for x, y in ts) / 3, 1)
            ts = []
            with torch.cuda.stream(s_k):
                for _ in range(3):
                    torch.cuda._sleep(int(a.gap_ms * cyc_per_ms))
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s_k)
                    stg[off:off + B].copy_(emb)
                    e1.record(s_k)
                    ts.append((e0, e1))
            torch.cuda.synchronize()
            r = {"tool": "pack_insitu", "sweep": "staging_offset", "offset": off,
                 "pack_us": {str(k): v for k, v in res.items()},
                 "segments": {str(k): nseg[k] for k in res},
                 "torch_copy_embed_to_staging_us": round(1e3 * sum(x.elapsed_time(y) for x, y in ts) / 3, 1),
                 "addr_delta_embed_minus_staging": int(emb.data_ptr()) - int(stg.data_ptr()) - off}
            print(json.dumps(r), flush=True)
            out.append(r)
        if a.out:
            with open(a.out, "a") as f:
                for r in out:
                    f.write(json.dumps(r) + "\n")
        mgr.close()
        return
    for v in [int(x) for x in a.variants.split(",")]:
        diag_pack_variant(v)
        run(True, "b2b")                                                # warm-up
        for pack in (True, False):
            for mode in ("b2b", "b2b+dma", "gap", "gap+dma"):
                r = {"tool": "pack_insitu", "model": a.model, "bucket_mb": a.bucket_mb, "variant": v,
                     "kernel": "pack" if pack else "unpack", "mode": mode, "hbm_peak_gbs": hbm, **run(pack, mode)}
                print(json.dumps(r), flush=True)
                out.append(r)
    diag_pack_variant(0)
    for mode in ("b2b", "b2b+dma"):
        r = {"tool": "pack_insitu", "kernel": "torch_copy_2GiB", "mode": mode, **torch_copy(mode)}
        print(json.dumps(r), flush=True)
        out.append(r)
    if a.out:
        with open(a.out, "a") as f:
            for r in out:
                f.write(json.dumps(r) + "\n")
    mgr.close()


if __name__ == "__main__":
    main()
