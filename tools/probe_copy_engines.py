#!/usr/bin/env python
"""Host-link probe: pinned D2H / H2D throughput with 1 or 2 streams per
direction, one direction or both at once (does a second copy stream per
direction buy bandwidth?)."""
import json

import torch


def run(n_d2h, n_h2d, size=2 << 30, reps=3):
    torch.cuda.set_device(0)
    hs = [torch.empty(size, dtype=torch.uint8).pin_memory() for _ in range(n_d2h + n_h2d)]
    ds = [torch.empty(size, dtype=torch.uint8, device="cuda") for _ in range(n_d2h + n_h2d)]
    ss = [torch.cuda.Stream() for _ in range(n_d2h + n_h2d)]
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record()
        ends = [torch.cuda.Event(enable_timing=True) for _ in ss]
        for i, s in enumerate(ss):
            s.wait_event(t0)
            with torch.cuda.stream(s):
                if i < n_d2h:
                    hs[i].copy_(ds[i], non_blocking=True)
                else:
                    ds[i].copy_(hs[i], non_blocking=True)
                ends[i].record(s)
        torch.cuda.synchronize()
        # per direction: its bytes over the span from the common start to its last copy's end
        span_d = max([t0.elapsed_time(e) for e in ends[:n_d2h]] or [0])
        span_h = max([t0.elapsed_time(e) for e in ends[n_d2h:]] or [0])
        d2h = n_d2h * size / (span_d * 1e-3) / 1e9 if n_d2h else 0.0
        h2d = n_h2d * size / (span_h * 1e-3) / 1e9 if n_h2d else 0.0
        if best is None or d2h + h2d > best[0] + best[1]:
            best = (d2h, h2d)
    return {"d2h_streams": n_d2h, "h2d_streams": n_h2d, "d2h_GBs": round(best[0], 1), "h2d_GBs": round(best[1], 1)}


if __name__ == "__main__":
    for cfg in ((1, 0), (2, 0), (0, 1), (0, 2), (1, 1), (2, 2), (1, 2), (2, 1)):
        print(json.dumps(run(*cfg)), flush=True)
