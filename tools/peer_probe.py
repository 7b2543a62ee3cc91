#!/usr/bin/env python
"""NVLink copy-engine probe from ONE process over N GPUs (peer access): the
denominators the push kernel's NVLink fraction is read against.

  pair        one GPU -> one peer, one direction (the "measured peer copy")
  bidir       one pair, both directions at once
  all2all     every GPU sends an equal share to every other GPU at once (each
              GPU's egress and ingress both busy: the sync's traffic pattern)

cudaMemcpyPeerAsync on one stream per (source, destination) pair, CUDA events
on the source GPU; rate = bytes leaving one GPU / the span of its copies.

    python tools/peer_probe.py --gpus 4 --gb 4 --out gpurun_out/peer_probe.jsonl
"""
import argparse
import json

import torch
from cuda.bindings import runtime as rt


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != rt.cudaError_t.cudaSuccess:
        raise SystemExit(f"CUDA error {err}")
    return r[1:] if isinstance(r, tuple) and len(r) > 1 else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=4)
    ap.add_argument("--gb", type=float, default=4.0, help="bytes each GPU sends per pattern, GB")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    N = a.gpus
    assert torch.cuda.device_count() >= N
    for r in range(N):
        ck(rt.cudaSetDevice(r))
        for g in range(N):
            if g != r:
                e = rt.cudaDeviceEnablePeerAccess(g, 0)[0]
                if e not in (rt.cudaError_t.cudaSuccess, rt.cudaError_t.cudaErrorPeerAccessAlreadyEnabled):
                    raise SystemExit(f"peer access {r}->{g}: {e}")
    B = int(a.gb * 1e9) // (N - 1) // 256 * 256            # bytes per (src, dst) pair
    src = [torch.empty((N - 1) * B, dtype=torch.uint8, device=f"cuda:{r}") for r in range(N)]
    dst = [torch.empty((N - 1) * B, dtype=torch.uint8, device=f"cuda:{r}") for r in range(N)]
    streams, evs = {}, {}
    for r in range(N):
        ck(rt.cudaSetDevice(r))
        for g in range(N):
            if g != r:
                streams[(r, g)] = ck(rt.cudaStreamCreateWithFlags(rt.cudaStreamNonBlocking))[0]
                evs[(r, g)] = (ck(rt.cudaEventCreate())[0], ck(rt.cudaEventCreate())[0])

    def slot(r, g):                                          # unique per destination
        return (r - g - 1) % N

    def run(pairs, nbytes):
        for r in range(N):
            ck(rt.cudaSetDevice(r))
            ck(rt.cudaDeviceSynchronize())
        for (r, g) in pairs:
            ck(rt.cudaSetDevice(r))
            s = streams[(r, g)]
            e0, e1 = evs[(r, g)]
            k = slot(r, g)
            ck(rt.cudaEventRecord(e0, s))
            ck(rt.cudaMemcpyPeerAsync(dst[g].data_ptr() + k * B, g, src[r].data_ptr() + k * B, r, nbytes, s))
            ck(rt.cudaEventRecord(e1, s))
        for r in range(N):
            ck(rt.cudaSetDevice(r))
            ck(rt.cudaDeviceSynchronize())
        ms = 0.0
        by_src = {}
        for (r, g) in pairs:
            by_src.setdefault(r, []).append(evs[(r, g)])
        for r, lst in by_src.items():
            ref = lst[0][0]
            t0 = min(ck(rt.cudaEventElapsedTime(ref, e0))[0] for e0, _ in lst)
            t1 = max(ck(rt.cudaEventElapsedTime(ref, e1))[0] for _, e1 in lst)
            ms = max(ms, t1 - t0)
        return ms

    out = []
    patterns = (("pair", [(0, 1)], B, B),
                ("bidir", [(0, 1), (1, 0)], B, B),
                ("all2all", [(r, g) for r in range(N) for g in range(N) if g != r], B, (N - 1) * B))
    for name, pairs, nb, per_gpu in patterns:
        ms = [run(pairs, nb) for _ in range(a.reps + 2)][2:]
        best = min(ms)
        line = {"probe": "peer_copy", "pattern": name, "n_gpus": N, "bytes_per_gpu_per_direction": per_gpu,
                "ms_best": round(best, 3), "ms_median": round(sorted(ms)[len(ms) // 2], 3),
                "GBs_per_gpu_per_direction_best": round(per_gpu / (best * 1e-3) / 1e9, 1),
                "GBs_per_gpu_per_direction_median": round(per_gpu / (sorted(ms)[len(ms) // 2] * 1e-3) / 1e9, 1)}
        print(json.dumps(line), flush=True)
        out.append(line)
    if a.out:
        with open(a.out, "a") as f:
            for l_ in out:
                f.write(json.dumps(l_) + "\n")


if __name__ == "__main__":
    main()
