#!/usr/bin/env python
"""Benchmark of the B200 state-transition hot path (BASELINE.json metric:
"state-switch latency (ms) and GB/s vs HBM/host-link/NVLink peak").

One STEP = one pass of the whole hot path on the GPU group
shared by two synthetic Qwen2.5-7B-shaped jobs A and B: the context switch of
PAPER.md:555 (resident A -> incoming B = [OFFLOAD A, ONLOAD B]) followed by the
train->rollout weight sync of B; the next step switches back.
    suspend A (a3 gather-pack + a4 D2H into A's pinned slab)
    resume  B (a6 H2D + a7 scatter-unpack + checksum verify)   -- concurrent with
              the suspend (NEXT-1): duplex when both jobs fit in HBM, else the
              in-place swap through one device copy and one pinned slab
    sync    B (a8 fp32->bf16 RNE + a9-a11 reshard into the rollout layout)
Workload at N GPUs: FSDP-N shards -> rollout TP-min(2,N) x DP-N/TP (configs[1]
is N=8: FSDP-8 -> TP-2 x DP-4).  ``value`` = state bytes moved through the
switch by all ranks per second (sum over ranks of S_out + S_in, ÷ the
max-over-ranks step time); ``ms_per_step`` is the switch + sync latency.

    python bench.py [--gpus N --steps K --warmup W]            # our CUDA path
    python bench.py --impl reference ...                        # the CPU oracle
    torchrun --nproc-per-node N bench.py --gpus N ...           # N > 1
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "state-switch latency (ms) and GB/s vs HBM/host-link/NVLink peak at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="plex", choices=["plex", "reference"])
    ap.add_argument("--model", default="qwen2.5-7b")
    ap.add_argument("--tp", type=int, default=0, help="rollout TP (default min(2, N))")
    ap.add_argument("--ep", type=int, default=1)
    ap.add_argument("--rank-map", default="auto", choices=["tp", "dp", "auto"],
                    help="rollout rank placement (R10): g = dp*TP+tp, g = tp*DP+dp, or the lighter ledger")
    ap.add_argument("--bucket-mb", type=int, default=2048)
    ap.add_argument("--slots", type=int, default=2)
    ap.add_argument("--no-hugepage", dest="hugepage", action="store_false",
                    help="pin slabs with cudaHostAlloc instead of mmap(MADV_HUGEPAGE) + cudaHostRegister")
    ap.add_argument("--no-duplex", action="store_true", help="sequential offload then onload")
    ap.add_argument("--single-job", action="store_true", help="step = suspend + resume + sync of one job")
    ap.add_argument("--swap", action="store_true", help="in-place swap switch even when two device copies fit")
    ap.add_argument("--no-balance", action="store_true", help="no NVLink-carried buckets (host-link balancing)")
    ap.add_argument("--e2e-steps", type=int, default=-1, help="end-to-end steps (default = steps)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-derived-variant", action="store_true",
                    help="skip the labelled N=1 derived-param (elision) sub-measurement")
    ap.add_argument("--cpu-ranks", type=int, default=8,
                    help="simulated ranks of the per-rank CPU-oracle setting (0 = skip)")
    ap.add_argument("--cpu-sample-layers", type=int, default=2)
    ap.add_argument("--sync-nccl", action="store_true", help="NCCL send/recv sync transport (baseline)")
    ap.add_argument("--out", default="")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md: clocks DURING the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None
        self.lines = []

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(self.index)],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None

    def _read(self):
        for ln in self.p.stdout:
            self.lines.append(ln.strip())

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# CPU oracle baseline (bounded sample of the same workload)
# ---------------------------------------------------------------------------
def cpu_oracle_prepare(model: str, world: int, tp: int, ep: int, layers: int):
    """Inputs of the CPU baseline: the first ``layers`` decoder layers (+ final
    norm) of rank 0's FSDP-``world`` shard (4 kinds) and every rank's master
    rows of those tensors.  Returns a callable that runs one timed sample:
    the oracle's o4 pack, o5 parse, and o6/o7 gather->RNE->reshard."""
    import numpy as np

    from oracle import plex_oracle as O
    from plexgen import gen_range, manifest

    man = [(k, s) for k, s in manifest(model)
           if any(k.startswith(f"model.layers.{l}.") for l in range(layers)) or k == "model.norm.weight"]
    dp = world // tp
    shards, ms = {}, {}
    for k, s in man:
        re_ = int(np.prod(s[1:])) if len(s) > 1 else 1
        parts = []
        for r in range(world):
            a, b = O.fsdp_rows(s[0], world, r)
            parts.append(gen_range(0, k, 1, a * re_, (b - a) * re_).reshape((b - a,) + tuple(s[1:])))
        ms[k] = parts
        a, b = O.fsdp_rows(s[0], world, 0)
        for kd in range(4):
            shards[(k, kd)] = parts[0] if kd == 1 else \
                gen_range(0, k, kd, a * re_, (b - a) * re_).reshape((b - a,) + tuple(s[1:]))
    S = sum(x.nbytes for x in shards.values())

    def one():
        t0 = time.perf_counter()
        segs, size = O.slab_layout(man, world, 0)
        slab = O.pack_slab(segs, size, shards)
        O.parse_slab(slab, segs, dict(man))
        O.weight_sync(ms, tp, dp, ep)
        dt = time.perf_counter() - t0
        return S / dt / 1e9, dt

    sample = (f"{model} layers[0:{layers}]+norm, rank-0 FSDP-{world} shard ({S / 1e9:.3f} GB state): "
              f"o4 pack + o5 parse + o6/o7 gather-RNE-reshard to TP-{tp}xDP-{dp} (all ranks' outputs)")
    return one, sample


def cpu_oracle_sample(model: str, world: int, tp: int, ep: int, layers: int):
    one, sample = cpu_oracle_prepare(model, world, tp, ep, layers)
    v, dt = one()
    return v, dt, sample


def box_info() -> dict:
    """The host the oracle runs on: lscpu model / sockets /
    cores, the CPUs this process may use, host memory."""
    out = {"affinity_cpus": len(os.sched_getaffinity(0)), "logical_cpus": os.cpu_count()}
    try:
        txt = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        want = {"Model name": "model", "Socket(s)": "sockets", "Core(s) per socket": "cores_per_socket",
                "Thread(s) per core": "threads_per_core", "NUMA node(s)": "numa_nodes"}
        for ln in txt.splitlines():
            k, _, v = ln.partition(":")
            if k.strip() in want:
                v = v.strip()
                out[want[k.strip()]] = int(v) if v.isdigit() else v
        if "sockets" in out and "cores_per_socket" in out:
            out["physical_cores"] = out["sockets"] * out["cores_per_socket"]
    except Exception as e:                                  # lscpu missing: say so
        out["lscpu"] = f"unavailable ({type(e).__name__})"
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal:"):
                out["mem_total_gb"] = round(int(ln.split()[1]) * 1024 / 1e9, 1)
    except OSError:
        pass
    return out


def _hwm_gb() -> float:
    """This process's own resident high-water mark (VmHWM; getrusage's ru_maxrss
    would report the bench parent's peak in a spawned child)."""
    try:
        for ln in open("/proc/self/status"):
            if ln.startswith("VmHWM:"):
                return round(int(ln.split()[1]) * 1024 / 1e9, 2)
    except OSError:
        pass
    return -1.0


def _oracle_single_worker(args):
    """The single-process setting in its own process (its own memory high-water mark)."""
    model, world, tp, ep, layers = args
    v, dt, sample = cpu_oracle_sample(model, world, tp, ep, layers)
    return v, dt, sample, _hwm_gb()


def _oracle_rank_worker(args):
    """One simulated rank of the per-rank CPU setting (runs in its own process):
    rank r's o4 pack + o5 parse of its FSDP-W shard of the sample, and o6/o7
    gather -> RNE -> slice/fuse of its own rollout tensors (g = r).  Inputs are
    generated before the common start barrier; the timed part is the oracle as it stands."""
    model, W, tp, ep, layers, r, barrier = args
    import numpy as np

    from oracle import plex_oracle as O
    from plexgen import gen_range, manifest
    man = [(k, s) for k, s in manifest(model)
           if any(k.startswith(f"model.layers.{l}.") for l in range(layers)) or k == "model.norm.weight"]
    dp = W // tp
    shards, ms = {}, {}
    for k, s in man:
        re_ = int(np.prod(s[1:])) if len(s) > 1 else 1
        parts = []
        for q in range(W):
            a, b = O.fsdp_rows(s[0], W, q)
            parts.append(gen_range(0, k, 1, a * re_, (b - a) * re_).reshape((b - a,) + tuple(s[1:])))
        ms[k] = parts
        a, b = O.fsdp_rows(s[0], W, r)
        for kd in range(4):
            shards[(k, kd)] = parts[r] if kd == 1 else \
                gen_range(0, k, kd, a * re_, (b - a) * re_).reshape((b - a,) + tuple(s[1:]))
    S = sum(x.nbytes for x in shards.values())
    barrier.wait()                                           # every rank starts together
    t0 = time.perf_counter()
    segs, size = O.slab_layout(man, W, r)
    slab = O.pack_slab(segs, size, shards)
    O.parse_slab(slab, segs, dict(man))
    from collections import OrderedDict
    full = OrderedDict((k, O.rne_bf16(O.gather(v))) for k, v in ms.items())
    O.rollout_tensors(full, tp, dp, ep, r)
    dt = time.perf_counter() - t0
    return S, dt, _hwm_gb()


def cpu_oracle_ranks(model: str, W: int, tp: int, ep: int, layers: int) -> dict:
    """SURVEY §8(d) D5 second setting: one process per simulated rank (W cores),
    all starting together; value = all ranks' state bytes / the slowest rank."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m, ctx.Pool(W) as pool:
        bar = m.Barrier(W)
        res = pool.map(_oracle_rank_worker, [(model, W, tp, ep, layers, r, bar) for r in range(W)], chunksize=1)
    S = sum(r[0] for r in res)
    dt = max(r[1] for r in res)
    dp = W // tp
    return {"value": round(S / dt / 1e9, 4), "unit": "GB/s", "cores": W, "kind": "oracle",
            "sample": (f"{model} layers[0:{layers}]+norm, FSDP-{W} -> TP-{tp}xDP-{dp} (configs[1] layout), one "
                       f"process per simulated rank: o4 pack + o5 parse of its shard ({S / W / 1e9:.3f} GB) + "
                       f"o6/o7 gather-RNE-reshard of its own rollout tensors"),
            "seconds_max_rank": round(dt, 2), "max_rss_gb_per_rank": max(r[2] for r in res)}


def cpu_baseline(a, world: int, tp: int) -> dict:
    """cpu_baseline of the bench line: the oracle, as it stands, on the box's host
    cores -- single process (headline, as the reference arm) plus the per-rank setting."""
    import multiprocessing as mp
    with mp.get_context("spawn").Pool(1) as pool:
        v, dt, sample, hwm = pool.apply(_oracle_single_worker, ((a.model, world, tp, a.ep, a.cpu_sample_layers),))
    out = {"value": round(v, 4), "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample,
           "seconds": round(dt, 2), "max_rss_gb": hwm, "box": box_info()}
    if a.cpu_ranks > 1:
        try:
            out["per_rank"] = cpu_oracle_ranks(a.model, a.cpu_ranks, min(2, a.cpu_ranks), a.ep, 1)
        except Exception as e:                               # never lose the bench line over the baseline
            out["per_rank"] = {"error": f"{type(e).__name__}: {e}"}
    return out


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = a.gpus
    tp = a.tp or min(2, world)
    one, sample = cpu_oracle_prepare(a.model, world, tp, a.ep, a.cpu_sample_layers)
    for _ in range(a.warmup):
        one()
    vals, secs = [], []
    for _ in range(a.steps):
        v, dt = one()
        vals.append(v)
        secs.append(dt)
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GB/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(1e3 * statistics.median(secs), 2),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (counter-based generator, DESIGN.md §3)",
            "config": {"workload": (f"two {a.model}-shaped jobs (bf16 param + fp32 master/m/v each) FSDP-{world} -> "
                                    f"rollout TP-{tp}xDP-{world // tp}; step = context switch + weight sync -- the "
                                    f"CPU oracle runs a bounded sample of it (see cpu_baseline.sample)"),
                       "model_shape": a.model, "impl_note": "CPU oracle (NumPy), no GPU"},
            "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample,
                             "box": box_info()},
            "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our CUDA path
# ---------------------------------------------------------------------------
def run_plex(a):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    import paper_2605_20863_b200 as P
    from paper_2605_20863_b200 import _lib as L
    from plexgen import MODELS, manifest

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allmin(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return float(t.item())

    def allsum(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t)
        return float(t.item())

    tp = a.tp or min(2, world)
    dp = world // tp
    shape = MODELS[a.model]
    bucket = a.bucket_mb << 20
    t_setup = time.perf_counter()
    mgr = P.StateManager(device=local, rank=rank, world=world, bucket_bytes=bucket, n_slots=a.slots, timing=True,
                         sync_nccl=a.sync_nccl)
    # host-link roofline BW_host(k = world): pinned copy of 4 GiB, all ranks at once
    probe = 4 << 30
    h = torch.empty(probe, dtype=torch.uint8).pin_memory()
    dbuf = torch.empty(probe, dtype=torch.uint8, device=f"cuda:{local}")
    bw = {}
    for direction in ("d2h", "h2d"):
        best = 0.0
        for _ in range(3):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            (h.copy_(dbuf, non_blocking=True) if direction == "d2h" else dbuf.copy_(h, non_blocking=True))
            e1.record()
            e1.synchronize()
            best = max(best, probe / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        bw[direction] = best
    # ... and both directions at once (what a duplex / swap switch can get per direction)
    h2 = torch.empty(probe, dtype=torch.uint8).pin_memory()
    dbuf2 = torch.empty(probe, dtype=torch.uint8, device=f"cuda:{local}")
    s_d, s_h = torch.cuda.Stream(local), torch.cuda.Stream(local)
    bw2 = {"d2h": 0.0, "h2d": 0.0}
    for _ in range(3):
        barrier()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        cur_s = torch.cuda.current_stream(local)
        s_d.wait_stream(cur_s)
        s_h.wait_stream(cur_s)
        with torch.cuda.stream(s_d):
            ev[0].record(s_d)
            h.copy_(dbuf, non_blocking=True)
            ev[1].record(s_d)
        with torch.cuda.stream(s_h):
            ev[2].record(s_h)
            dbuf2.copy_(h2, non_blocking=True)
            ev[3].record(s_h)
        torch.cuda.synchronize(local)
        bw2["d2h"] = max(bw2["d2h"], probe / (ev[0].elapsed_time(ev[1]) * 1e-3) / 1e9)
        bw2["h2d"] = max(bw2["h2d"], probe / (ev[2].elapsed_time(ev[3]) * 1e-3) / 1e9)
    del h, dbuf, h2, dbuf2
    torch.cuda.empty_cache()

    # NEXT-1 host-link balancing: every rank's rate for one offload + one onload
    # byte, all-gathered; the planner hands whole buckets from slow-link ranks
    # to fast-link ranks over NVLink when that shortens the slowest rank
    weights = None
    if world > 1 and not a.no_balance:
        # a duplex switch takes max(S/d2h, S/h2d) at the both-directions rates;
        # a sequential one S/d2h + S/h2d at the one-direction rates
        w_local = (1.0 / (1.0 / bw["d2h"] + 1.0 / bw["h2d"]) if a.no_duplex
                   else min(bw2["d2h"], bw2["h2d"]))
        wt = torch.tensor([w_local], dtype=torch.float64, device=f"cuda:{local}")
        allw = [torch.zeros_like(wt) for _ in range(world)]
        dist.all_gather(allw, wt)
        weights = [float(x.item()) for x in allw]

    t0 = time.perf_counter()
    rank_map = {"tp": 0, "dp": 1, "auto": 2}[a.rank_map]
    plans = [mgr.plan(manifest(a.model), head_dim=shape.head_dim, tp=tp, dp=dp, ep=a.ep, rank_map=rank_map,
                      link_weights=weights) for _ in range(2)]
    for pl in plans:
        mgr.enable_carry(pl)
    n_carried = len(plans[0].carry())
    plan_s = (time.perf_counter() - t0) / 2
    plan = plans[0]
    info = plan.rank_info(rank)
    # two jobs of the same shape (seeds 1, 2): B starts suspended, A resident --
    # one resident job per GPU group (R17).  duplex: both jobs keep their own
    # device tensors and slabs and the switch runs offload A || onload B
    # (plex_state_switch).  swap: when two device copies do not fit in HBM (N=1:
    # 2 x 106.6 GB), A and B share ONE set of device tensors and ONE slab and the
    # switch is the in-place plex_state_swap -- both host-link directions still
    # run at once.  sequential (--no-duplex): offload A, then onload B.
    free0, _ = torch.cuda.mem_get_info(local)
    fits2 = 2 * info.payload_bytes + info.dst_arena_bytes + (6 << 30) < free0
    if a.single_job:
        mode = "single"
    elif a.swap or not allmin(1.0 if fits2 else 0.0) > 0.5:
        mode = "swap"
    else:
        mode = "sequential" if a.no_duplex else "duplex"
    job_b = None
    if mode in ("duplex", "sequential"):
        try:
            job_b = P.Job(mgr, plans[1], seed=2, hugepage=a.hugepage).alloc().init_synthetic()
            job_b.suspend()
            job_a = P.Job(mgr, plans[0], seed=1, hugepage=a.hugepage).alloc().init_synthetic()
            ok = 1.0
        except P.PlexError as e:
            if e.code != P._lib.E_TIER_FULL:
                raise
            ok = 0.0
        if not allmin(ok) > 0.5:                      # two slabs exceed the pinnable host memory
            job_b = job_a = None
            torch.cuda.empty_cache()
            mode = "swap"
    if mode == "swap" and n_carried:                  # the in-place swap does not carry buckets
        plans = [mgr.plan(manifest(a.model), head_dim=shape.head_dim, tp=tp, dp=dp, ep=a.ep, rank_map=rank_map)
                 for _ in range(2)]
        plan, n_carried = plans[0], 0
        info = plan.rank_info(rank)
    if mode == "swap":
        job_a = P.Job(mgr, plans[0], seed=1, slab=False).alloc()
        job_b = P.Job(mgr, plans[0], seed=2, hugepage=a.hugepage)
        job_b.shards = job_a.shards                   # B's state: generated in place, offloaded
        job_b.init_synthetic()
        job_b.suspend(release=False)
        job_b.shards = type(job_a.shards)()
        job_a.init_synthetic()                        # A resident in the same tensors
    if mode == "single":
        job_a = P.Job(mgr, plans[0], seed=1, hugepage=a.hugepage).alloc().init_synthetic()
    two_jobs = mode != "single"
    duplex = mode in ("duplex", "swap")
    jobs = [job_a, job_b] if two_jobs else [job_a, job_a]
    group = None
    if two_jobs:
        # the GPU group's residency authority (plex_group) decides and
        # executes every switch: swap for jobs sharing one device copy, duplex when
        # both fit, sequential under an HBM budget of one job (--no-duplex)
        budget = None
        if mode == "sequential":
            budget = sum(v.numel() * v.element_size() for v in job_a.slab_shards().values())
        group = P.Group(mgr, hbm_budget=budget)
        shared = 0 if mode == "swap" else None
        group.add(job_a, resident=True, storage=shared)
        group.add(job_b, storage=shared)
    arena = mgr.arena(plan)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup

    phase_ev = []
    cur = {"i": 0}
    modes_seen = set()

    def step(record=False):
        """PAPER.md:555 transition: resident A -> incoming B = [OFFLOAD A, ONLOAD B], then SYNC B."""
        i = cur["i"]
        out, inc = jobs[i], jobs[1 - i]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if record else None
        if ev:
            ev[0].record()
        if group is not None:
            res = group.transition(inc)                  # the library decides [OFFLOAD A, ONLOAD B] and runs it
            modes_seen.add(res["mode"])
        else:
            out.suspend(release=False)
            inc.resume()
        if ev:
            ev[1].record()
        if group is not None:
            group.transition(inc, sync=arena)            # resident: [SYNC B]
        else:
            inc.sync(arena)
        if ev:
            ev[2].record()
            phase_ev.append(ev)
        cur["i"] = 1 - i

    for _ in range(a.warmup):
        step()
    mgr.reset_stats()
    clocks = Clocks(local)
    barrier()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record()
    for _ in range(a.steps):
        step(record=True)
    e1.record()
    barrier()
    clk = clocks.stop()
    local_ph = {n: sum(ev[i].elapsed_time(ev[i + 1]) for ev in phase_ev) / a.steps
                for i, n in enumerate(("switch", "sync"))}
    phases = {n: allmax(v) for n, v in local_ph.items()}
    phases_min = {n: allmin(v) for n, v in local_ph.items()}
    ms_local = e0.elapsed_time(e1) / a.steps
    ms = allmax(ms_local)
    st = mgr.stats()

    # end-to-end through the public API (Job.switch_to / suspend+resume, Job.sync),
    # host clock: every step H2D-copies the incoming job's state (the step's input)
    # from pinned host memory and D2H-copies the outgoing job's state (its result),
    # with release / re-acquire of device storage.
    e2e_steps = a.steps if a.e2e_steps < 0 else a.e2e_steps
    e2e = None
    if e2e_steps > 0:
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            step()
        torch.cuda.synchronize()
        barrier()
        e2e_s = allmax((time.perf_counter() - t0) / e2e_steps)
        e2e = {"s": e2e_s, "h2d": info.slab_bytes, "d2h": info.slab_bytes + 16 * info.n_segments}

    executor_desc = (("plex_group_transition (library residency map decides every switch; modes "
                      f"seen: {sorted(modes_seen)})") if group is not None else "direct calls")

    # ---- diagnostic (N>1, outside the timed region): the fused push split into its
    # local (HBM-only) and remote (NVLink) items, timed as two launches so that each
    # gets its own roofline fraction (PLEX_CTX_SPLIT_PUSH)
    split = None
    if world > 1 and not a.sync_nccl and two_jobs:
        inc = jobs[cur["i"]]                            # the resident job after the last step
        mgr.set_split_push(True)
        for _ in range(2):
            group.transition(inc, sync=arena)
        mgr.reset_stats()
        n_sp = max(3, min(a.steps, 10))
        for _ in range(n_sp):
            barrier()
            group.transition(inc, sync=arena)
        mgr.set_split_push(False)
        sst = mgr.stats()
        pk_hbm, pk_kind = load_peaks()
        t_l = allmax(sst["push_local"]["ms"] / n_sp)
        t_r = allmax(sst["push_remote"]["ms"] / n_sp)
        nvb = allmax(float(max(info.send_bytes, info.recv_bytes)))
        loc_gbs = (sst["push_local"]["bytes"] / n_sp) / (max(t_l, 1e-9) * 1e-3) / 1e9
        rem_gbs = nvb / (max(t_r, 1e-9) * 1e-3) / 1e9
        split = {"local": {"bound": "hbm", "achieved": round(loc_gbs, 1), "peak": pk_hbm, "unit": "GB/s",
                           "frac": round(loc_gbs / pk_hbm, 4), "ms": round(t_l, 3),
                           "note": "local push items alone (split launch, diagnostic after the timed region)"},
                 "remote": {"bound": "nvlink", "achieved": round(rem_gbs, 1), "peak": 770.0, "unit": "GB/s",
                            "frac": round(rem_gbs / 770.0, 4), "frac_of_nominal": round(rem_gbs / 900.0, 4),
                            "bytes_max_rank": nvb, "ms": round(t_r, 3),
                            "peak_kind": "measured peer copy 770 GB/s/dir (B200_PROFILING.md); nominal 900",
                            "note": ("remote push items alone (split launch, diagnostic after the timed region): "
                                     "max over ranks of max(send, recv) / max over ranks of the launch time")}}

    # ---- labelled variant (N=1): the realistic post-optimizer-step state -------------
    # param == RNE(master) (what a mixed-precision step leaves), so
    # NEXT-2 elision derives the bf16 params on resume instead of moving them
    # through the host link.  Same workload and step; the headline above keeps the
    # conservative independent-param state (reading D2').
    variant = None
    if world == 1 and mode == "swap" and not a.no_derived_variant:
        import gc
        group.close()
        del group, jobs, job_a, job_b
        group = job_a = job_b = jobs = None
        gc.collect()
        torch.cuda.empty_cache()
        plan_el = mgr.plan(manifest(a.model), head_dim=shape.head_dim, tp=tp, dp=dp, ep=a.ep, rank_map=rank_map,
                           elide_param=True)
        va = P.Job(mgr, plan_el, seed=1, slab=False).alloc()
        vb = P.Job(mgr, plan_el, seed=2, hugepage=a.hugepage)
        vb.shards = va.shards
        vb.init_synthetic(derived_param=True)
        vb.suspend(release=False)
        vb.shards = type(va.shards)()
        va.init_synthetic(derived_param=True)
        vgroup = P.Group(mgr)
        vgroup.add(va, resident=True, storage=0)
        vgroup.add(vb, storage=0)
        vjobs, vcur = [va, vb], {"i": 0}

        def vstep():
            inc = vjobs[1 - vcur["i"]]
            vgroup.transition(inc)
            vgroup.transition(inc, sync=arena)
            vcur["i"] = 1 - vcur["i"]

        vsteps, vwarm = max(1, min(a.steps, 10)), max(3, min(a.warmup, 3))
        for _ in range(vwarm):
            vstep()
        mgr.reset_stats()
        barrier()
        v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        v0.record()
        for _ in range(vsteps):
            vstep()
        v1.record()
        barrier()
        vms = allmax(v0.elapsed_time(v1) / vsteps)
        vst = mgr.stats()
        vinfo = plan_el.rank_info(rank)
        variant = {"label": "derived_param (param == RNE(master)): NEXT-2 elision active",
                   "value": round(2 * vinfo.payload_bytes / (vms * 1e-3) / 1e9, 3), "unit": "GB/s",
                   "ms_per_step": round(vms, 2), "steps": vsteps, "warmup": vwarm,
                   "elided": bool(vjobs[1 - vcur["i"]].slab.elided),     # the slab holder: the suspended job
                   "host_link_bytes_per_step": int((vst["d2h"]["bytes"] + vst["h2d"]["bytes"]) / vsteps),
                   "state_bytes_switched_per_step": int(2 * vinfo.payload_bytes),
                   "derive_ms_per_step": round(vst["derive"]["ms"] / vsteps, 3),
                   "note": ("value = state bytes switched (both jobs' full 4-kind state) / step time; the bf16 "
                            "params (1/7 of the bytes) are re-derived on the device, not moved")}
        vgroup.close()
        del vgroup, vjobs, va, vb
        gc.collect()
        torch.cuda.empty_cache()

    S_total = allsum(float(2 * info.payload_bytes))      # offloaded + onloaded state per switch
    value = S_total / (ms * 1e-3) / 1e9
    peak_hbm, peak_kind = load_peaks()

    # roofline of the dominant kernel (largest total device time among ours)
    kern = {k: st[k] for k in ("pack", "unpack", "push", "rpack", "runpack") if st[k]["launches"]}
    dom = max(kern, key=lambda k: kern[k]["ms"])
    d = kern[dom]
    per_launch_bytes = d["bytes"] / d["launches"]
    avg_ms = d["ms"] / d["launches"]
    achieved = per_launch_bytes / (avg_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        traffic = tj.get(dom, {}).get("dram_bytes_per_launch")

    def frac(x, p):
        return round(x / p, 4) if p else None

    d2h, h2d = st["d2h"], st["h2d"]
    rl = {}
    for k, v in kern.items():
        if v["ms"] > 0:
            gbs = v["bytes"] / (v["ms"] * 1e-3) / 1e9
            rl[k] = {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak_hbm, "unit": "GB/s",
                     "frac": frac(gbs, peak_hbm), "launches_per_step": v["launches"] / a.steps,
                     "ms_per_step": round(v["ms"] / a.steps, 3)}
    bw_ref = bw2 if duplex else bw                      # duplex / swap: both directions share the link
    for k, v, ref in (("d2h", d2h, bw_ref["d2h"]), ("h2d", h2d, bw_ref["h2d"])):
        gbs = v["bytes"] / (v["ms"] * 1e-3) / 1e9 if v["ms"] > 0 else 0.0
        lo, hi = allmin(gbs), allmax(gbs)
        ref_lo = allmin(ref)
        if v["ms"] > 0:
            rl["host_" + k] = {"bound": "host_link", "achieved": round(gbs, 2), "peak": round(ref, 2),
                               "unit": "GB/s", "frac": frac(gbs, ref),
                               "achieved_min_max_over_ranks": [round(lo, 2), round(hi, 2)],
                               "peak_min_over_ranks": round(ref_lo, 2),
                               "peak_kind": (f"measured pinned copy, {world} GPU(s) concurrently, "
                                             + ("both directions at once" if duplex else "one direction")
                                             + " (this rank)"),
                               "peak_one_direction": round(bw[k], 2)}
    if world > 1:
        # The fused cast+push kernel moves local casts through HBM and remote ones
        # over NVLink at once: its roofline is the slower of the two resources
        # (B200_PROFILING.md: fused compute+collective kernels).  Per rank
        # T_hbm = (fp32 read + local bf16 writes + incoming bf16 writes) / HBM peak,
        # T_nvl = max(send, recv) / 770 GB/s measured peer copy; bound = max over
        # ranks of max(T_hbm, T_nvl); frac = bound / measured push time (max over ranks).
        nv = allmax(float(max(info.send_bytes, info.recv_bytes)))
        hbm_b = float(info.src_read_bytes + info.local_bytes + info.recv_bytes)
        t_hbm = allmax(hbm_b / (peak_hbm * 1e9) * 1e3)
        t_nvl = allmax(float(max(info.send_bytes, info.recv_bytes)) / 770e9 * 1e3)
        if not st["nccl"]["launches"]:
            # the single-resource "push" row (all 6 B/element over HBM) does not
            # describe a kernel that also stores over NVLink: push_fused replaces it
            rl.pop("push", None)
            t_push = allmax(st["push"]["ms"] / a.steps)
            bound = "nvlink" if t_nvl >= t_hbm else "hbm"
            rl["push_fused"] = {"bound": bound, "lower_bound_ms": round(max(t_hbm, t_nvl), 3),
                                "t_hbm_ms": round(t_hbm, 3), "t_nvlink_ms": round(t_nvl, 3),
                                "achieved_ms": round(t_push, 3), "frac": frac(max(t_hbm, t_nvl), t_push),
                                "nvlink_bytes_max_rank": nv, "hbm_bytes_this_rank": hbm_b,
                                "peak_kind": f"HBM {peak_hbm} GB/s ({peak_kind}); NVLink 770 GB/s measured peer copy "
                                             "(900 nominal)"}
        else:
            t_x = allmax(st["nccl"]["ms"] / a.steps)
            gbs = nv / (t_x * 1e-3) / 1e9
            rl["nvlink"] = {"bound": "nvlink", "achieved": round(gbs, 1), "peak": 770.0, "unit": "GB/s",
                            "frac": frac(gbs, 770.0), "frac_of_nominal": frac(gbs, 900.0),
                            "bytes_max_rank": nv, "ms": round(t_x, 3), "over": "NCCL exchange rounds",
                            "peak_kind": "measured peer copy 770 GB/s/dir (B200_PROFILING.md); nominal 900"}
        if split is not None:
            rl["push_local"] = split["local"]
            rl["nvlink"] = split["remote"]

        if st["nccl"]["launches"]:
            rl["nccl_exchange"] = {"ms_per_step": round(st["nccl"]["ms"] / a.steps, 3),
                                   "rounds_per_step": st["nccl"]["launches"] / a.steps}
    # our kernel launches in the timed region: pack + unpack + push (+NCCL-path K4/K5) + 1 verify per onload
    launches = sum(v["launches"] for v in kern.values()) + a.steps
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(ms, 2), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "dtype_note": "state moved as raw bits (bf16 + fp32); the only arithmetic is the fp32->bf16 RNE cast in 32-bit integer ops",
            "data": "synthetic (counter-based generator, DESIGN.md §3); random-init Qwen2.5-7B-shaped state",
            "config": {"workload": (f"two {a.model}-shaped jobs (bf16 param + fp32 master/m/v each) FSDP-{world} -> "
                                    f"rollout TP-{tp}xDP-{dp}; step = context switch A->B (full suspend of A + full "
                                    f"resume of B, " + {"duplex": "duplex: offload || onload",
                                                        "swap": "in-place swap: offload || onload through one "
                                                                "device copy and one pinned slab",
                                                        "sequential": "sequential"}[mode] + ") + "
                                    f"weight sync of B") if two_jobs else
                                   (f"one {a.model}-shaped job (bf16 param + fp32 master/m/v) FSDP-{world} -> rollout "
                                    f"TP-{tp}xDP-{dp}; step = full suspend + full resume + weight sync (two jobs' "
                                    f"slabs exceed the host's pinnable memory)"),
                       "jobs": 2 if two_jobs else 1,
                       "host_link_weights_GBs": [round(x, 2) for x in weights] if weights else None,
                       "carried_buckets_per_job": n_carried,
                       "model_shape": a.model, "state_bytes_per_rank_per_job": info.payload_bytes,
                       "bytes_switched_per_step": int(S_total), "duplex": duplex, "switch_mode": mode,
                       "bucket_bytes": bucket, "staging_slots": a.slots,
                       "l2": "inputs (state) larger than L2 (126 MB); no flush needed",
                       "plan_ms": round(plan_s * 1e3, 1), "setup_s": round(setup_s, 1),
                       "sync_transport": "nccl" if a.sync_nccl else "nvlink-push",
                       "executor": executor_desc,
                       "rank_map": ["tp_fast (g = dp*TP + tp)", "dp_fast (g = tp*DP + dp)"][plan.stats().rank_map]},
            "roofline": {"kernel": dom, "bound": "hbm", "achieved": round(achieved, 1), "peak": peak_hbm,
                         "unit": "GB/s", "frac": frac(achieved, peak_hbm), "traffic": traffic,
                         "algorithmic_bytes_per_launch": int(per_launch_bytes), "avg_launch_ms": round(avg_ms, 4),
                         "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"},
            "rooflines": rl,
            "phases_ms": {k: round(v, 3) for k, v in phases.items()},
            "phases_ms_min_over_ranks": {k: round(v, 3) for k, v in phases_min.items()},
            "clocks": clk,
            "gpu_launches": int(launches),
        }
        if e2e:
            line["e2e"] = {"value": round(S_total / e2e["s"] / 1e9, 3), "unit": "GB/s",
                           "ms_per_step": round(e2e["s"] * 1e3, 2), "h2d_bytes_per_step": e2e["h2d"],
                           "d2h_bytes_per_step": e2e["d2h"],
                           "api": {"swap": "Group.transition(B) (in-place swap) -> Group.transition(B, sync=arena) "
                                           "(host clock)",
                                   "duplex": "Group.transition(B) (duplex, storage release/acquire) -> "
                                             "Group.transition(B, sync=arena) (host clock)",
                                   "sequential": "Group.transition(B) (sequential under a one-job HBM budget, "
                                                 "storage release/acquire) -> Group.transition(B, sync=arena) "
                                                 "(host clock)",
                                   "single": "Job.suspend + Job.resume -> Job.sync (host clock)"}[mode]}
        if variant is not None:
            line["derived_param"] = variant
        if not a.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(a, world, tp)
        print(json.dumps(line), flush=True)
        if a.out:
            with open(a.out, "w") as f:
                json.dump(line, f, indent=1)
    barrier()
    del jobs, job_a, job_b, arena, group
    mgr.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_plex(a)


if __name__ == "__main__":
    main()
