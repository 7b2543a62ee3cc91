#!/usr/bin/env python
"""Measurements of the other BASELINE.json configs.

bench.py times the headline workload; this script times the rest, one JSON
line per run (rank 0), device-timed with CUDA events on the caller stream and
max over ranks:

  duplex     two jobs of --model: step = switch A->B (offload A || onload B,
             NEXT-1) + sync B, alternating; reports the switch latency against
             the sequential C_setup = T_offload + T_load (Eq. 3)
  optim      configs[2]: optimizer kinds only (master/m/v) of rank r's FSDP-8
             shard of --model (default Qwen2.5-32B), offload + onload with k =
             WORLD_SIZE GPUs at once (each process is rank r of the 8-rank plan)
  moe        configs[3]: Qwen3-30B-A3B, FSDP-N -> attention TP-2 x DP + experts
             EP-N weight sync, plus per-expert KEY_MAJOR pack/offload/onload of
             --units expert units
  multiplex  configs[4]: 4 jobs (0.5B/1.5B/3B/7B, seeds 0..3) time-slicing
             the group, R rounds round-robin; each visit = transition ops of
             PAPER.md:555 (offload resident, onload incoming) + mutation + sync

    torchrun --nproc-per-node N tools/scenarios.py --scenario duplex --gpus N
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2605_20863_b200 as P  # noqa: E402
from paper_2605_20863_b200 import _lib as L  # noqa: E402
from plexgen import MODELS, manifest  # noqa: E402

from bench import Clocks  # noqa: E402


class Ctx:
    def __init__(self, gpus: int):
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        assert self.world == gpus, (gpus, self.world)
        torch.cuda.set_device(self.local)
        if self.world > 1:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{self.local}"))

    def barrier(self):
        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(self, x: float) -> float:
        if self.world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{self.local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allmin(self, x: float) -> float:
        if self.world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{self.local}")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return float(t.item())

    def allsum(self, x: float) -> float:
        if self.world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{self.local}")
        dist.all_reduce(t)
        return float(t.item())

    def emit(self, line: dict, out: str):
        if self.rank == 0:
            print(json.dumps(line), flush=True)
            if out:
                with open(out, "a") as f:
                    f.write(json.dumps(line) + "\n")


def timed(c: Ctx, fn, steps: int, warmup: int, min_s: float = 1.5):
    """CUDA-event time per call (max over ranks) and the clocks sampled during
    it.  Short calls (a 7 ms sync) are repeated until the timed region lasts
    >= min_s, so nvidia-smi (200 ms period) records the clocks under load."""
    for _ in range(warmup):
        fn()
    if min_s > 0 and steps > 0:
        c.barrier()
        t0 = time.perf_counter()
        fn()
        c.barrier()
        dt = time.perf_counter() - t0
        steps = int(c.allmax(float(max(steps, min(2000, int(min_s / max(dt, 1e-5)) + 1)))))
    clocks = Clocks(c.local)
    c.barrier()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    c.barrier()
    clk = clocks.stop()
    clk["timed_calls"] = steps
    return c.allmax(e0.elapsed_time(e1) / max(1, steps)), clk


def scen_duplex(a, c: Ctx):
    shape = MODELS[a.model]
    tp = a.tp or min(2, c.world)
    mgr = P.StateManager(device=c.local, rank=c.rank, world=c.world, bucket_bytes=a.bucket_mb << 20, timing=True)
    plans = [mgr.plan(manifest(a.model), head_dim=shape.head_dim, tp=tp, dp=c.world // tp, rank_map=L.RANKMAP_AUTO)
             for _ in range(2)]
    jobs = [P.Job(mgr, pl, seed=s).alloc().init_synthetic() for pl, s in zip(plans, (1, 2))]
    arena = mgr.arena(plans[0])
    jobs[1].suspend()
    state = {"cur": 0}

    def seq_step():                                  # sequential C_setup = T_off + T_load
        i = state["cur"]
        jobs[i].suspend()
        jobs[1 - i].resume()
        jobs[1 - i].sync(arena)
        state["cur"] = 1 - i

    def duplex_step():
        i = state["cur"]
        jobs[i].switch_to(jobs[1 - i])
        jobs[1 - i].sync(arena)
        state["cur"] = 1 - i

    ms_seq, _ = timed(c, seq_step, a.steps, a.warmup)
    ms_dup, clk = timed(c, duplex_step, a.steps, a.warmup)
    S = plans[0].rank_info(c.rank).payload_bytes
    tot = c.allsum(2.0 * S)
    c.emit({"scenario": "duplex", "model": a.model, "n_gpus": c.world, "layout": f"FSDP-{c.world}->TP-{tp}",
            "state_bytes_per_rank_per_job": S,
            "sequential_switch_ms": round(ms_seq, 2), "duplex_switch_ms": round(ms_dup, 2),
            "speedup": round(ms_seq / ms_dup, 3),
            "host_link_GBs_aggregate": round(tot / (ms_dup * 1e-3) / 1e9, 2), "clocks": clk,
            "note": "step = context switch (offload A, onload B) + sync B; both jobs fully resident on device "
                    "during the switch"}, a.out)


def scen_elide(a, c: Ctx):
    """NEXT-2: the bench step (switch + sync) with bf16 params = RNE(master) (what a
    mixed-precision optimizer step leaves) and PLEX_PLAN_ELIDE_PARAM: the param
    buckets are checked on the device and re-derived on resume instead of moved.
    Duplex switch when two device copies fit, else the in-place swap (bench N=1)."""
    shape = MODELS[a.model]
    tp = a.tp or min(2, c.world)
    mgr = P.StateManager(device=c.local, rank=c.rank, world=c.world, bucket_bytes=a.bucket_mb << 20, timing=True)
    out = {}
    for elide in (False, True):
        plans = [mgr.plan(manifest(a.model), head_dim=shape.head_dim, tp=tp, dp=c.world // tp, elide_param=elide)
                 for _ in range(2)]
        info = plans[0].rank_info(c.rank)
        free, _ = torch.cuda.mem_get_info(c.local)
        swap = c.allmin(1.0 if 2 * info.payload_bytes + info.dst_arena_bytes + (6 << 30) < free else 0.0) < 0.5
        if swap:
            jobs = [P.Job(mgr, plans[0], seed=1, slab=False).alloc(), P.Job(mgr, plans[0], seed=2)]
            jobs[1].shards = jobs[0].shards
            jobs[1].init_synthetic(derived_param=True)
            jobs[1].suspend(release=False)
            jobs[1].shards = type(jobs[0].shards)()
            jobs[0].init_synthetic(derived_param=True)
        else:
            jobs = [P.Job(mgr, pl, seed=s).alloc().init_synthetic(derived_param=True) for pl, s in zip(plans, (1, 2))]
            jobs[1].suspend()
        arena = mgr.arena(plans[0])
        state = {"cur": 0}

        def step():
            i = state["cur"]
            (jobs[i].swap_with if swap else jobs[i].switch_to)(jobs[1 - i])
            jobs[1 - i].sync(arena)
            state["cur"] = 1 - i

        ms, clk = timed(c, step, a.steps, a.warmup)
        out["elided" if elide else "full"] = {"switch_plus_sync_ms": round(ms, 2), "mode": "swap" if swap else "duplex",
                                              "slab_elided": bool(jobs[1 - state["cur"]].slab.elided),
                                              "elide_bytes_per_rank": info.elide_bytes}
        del jobs, arena, plans
        torch.cuda.empty_cache()
    c.emit({"scenario": "elide", "model": a.model, "n_gpus": c.world, "layout": f"FSDP-{c.world}->TP-{tp}",
            **out, "speedup": round(out["full"]["switch_plus_sync_ms"] / out["elided"]["switch_plus_sync_ms"], 3)},
           a.out)


def scen_hrrs(a, c: Ctx):
    """NEXT-4: drain one queue of RLVR requests from 4 jobs time-slicing the
    GPU group, FCFS vs HRRS (Alg. 1 / Eq. 3-4) ordering.  Context switches and
    weight syncs are real, decided and executed by the group's residency
    authority (plex_group_transition); a request's compute phase is modeled
    as a host-side wait of its Table-2 duration scaled by
    --time-scale.  HRRS gets C_setup = T_offload + T_load as measured by the
    library on the first switches (Setup.from_stats)."""
    import random

    from paper_2605_20863_b200.scheduler import Req, Setup, priority
    models = ["qwen2.5-0.5b", "qwen2.5-1.5b", "qwen2.5-3b", "qwen2.5-7b"]
    mgr = P.StateManager(device=c.local, rank=c.rank, world=c.world, bucket_bytes=a.bucket_mb << 20, timing=True)
    plans, jobs, arenas = [], [], []
    for j, mo in enumerate(models):
        tp = 1 if mo == "qwen2.5-0.5b" or c.world == 1 else 2
        pl = mgr.plan(manifest(mo), head_dim=MODELS[mo].head_dim, tp=tp, dp=c.world // tp, rank_map=L.RANKMAP_AUTO)
        plans.append(pl)
        jb = P.Job(mgr, pl, seed=j).alloc().init_synthetic()
        jb.suspend()
        jobs.append(jb)
        arenas.append(mgr.arena(pl))
    # Table 2 phases (s): compute_log_prob, update_actor, sync_weight of the 7B job;
    # smaller jobs scale with parameter count
    base = {"log_prob": 9.66, "update": 38.08, "sync": 9.76}
    psize = [plans[j].stats().total_params / plans[3].stats().total_params for j in range(4)]
    rng = random.Random(0)
    reqs = []
    for j in range(4):
        for cyc in range(a.rounds):
            for k, (kind, sec) in enumerate(base.items()):
                reqs.append(Req(j, rng.uniform(0, 1.0) + cyc + 0.01 * k, sec * psize[j] * a.time_scale, name=kind))
    reqs.sort(key=lambda r: r.arrival)

    def run(policy: str, setup: Setup):
        group = P.Group(mgr)              # the residency authority executes every switch the order causes
        for jb in jobs:                   # every job starts HOST-resident
            group.add(jb)
        resident = None
        t0 = time.perf_counter()
        pending = list(reqs)
        switches = 0
        waits = []
        while pending:
            now = time.perf_counter() - t0 + 1.0          # every request has arrived by t = 1
            if policy == "fcfs":
                pick = 0
            else:
                cur = Req(resident, 0.0, 1e-9, remaining=1e-9) if resident is not None else None
                pick = max(range(len(pending)), key=lambda i: priority(pending[i], now, cur, setup))
            if c.world > 1:                               # every rank must run the same request
                obj = [pick]
                dist.broadcast_object_list(obj, src=0)
                pick = obj[0]
            r = pending[pick]
            pending.remove(r)
            waits.append(now - r.arrival)
            # the group compares the request's job with its resident
            # job and prepends [OFFLOAD, ONLOAD] itself when they differ
            res = group.transition(jobs[r.job], sync=arenas[r.job] if r.name == "sync" else None)
            if res["mode"] not in ("none",):
                switches += 1
            resident = r.job
            torch.cuda.synchronize()
            time.sleep(r.exec_time)                       # the request's own compute phase (modeled)
        group.close()                                     # park the resident job for the next run
        jobs[resident].suspend()
        return time.perf_counter() - t0, switches, sum(waits) / len(waits)

    mgr.reset_stats()
    t_fcfs, n_fcfs, w_fcfs = run("fcfs", Setup(0.0, 0.0))
    st = mgr.stats()
    setup = Setup.from_stats(st, n_fcfs, n_fcfs, duplex=True,
                             job_bytes={j: plans[j].rank_info(c.rank).payload_bytes for j in range(4)})
    t_hrrs, n_hrrs, w_hrrs = run("hrrs", setup)
    c.emit({"scenario": "hrrs", "jobs": models, "n_gpus": c.world, "requests": len(reqs),
            "time_scale": a.time_scale,
            "measured_host_link_GBs": {"d2h": round(setup.bw_out / 1e9, 2), "h2d": round(setup.bw_in / 1e9, 2)},
            "fcfs": {"makespan_s": round(c.allmax(t_fcfs), 3), "switches": n_fcfs, "mean_wait_s": round(w_fcfs, 3)},
            "hrrs": {"makespan_s": round(c.allmax(t_hrrs), 3), "switches": n_hrrs, "mean_wait_s": round(w_hrrs, 3)}},
           a.out)


def scen_overlap(a, c: Ctx):
    """NEXT-1 off-critical-path switching: 4 jobs visit the
    group round-robin; each visit = switch in + weight sync + the job's compute
    phase (modeled as a host wait of its Table-2 update_actor time x
    --time-scale).  'blocking': duplex switch at the visit boundary.
    'overlap': while job j computes, the previous job drains and the next one
    is prefetched, so the boundary only waits for what is left."""
    models = ["qwen2.5-0.5b", "qwen2.5-1.5b", "qwen2.5-3b", "qwen2.5-7b"]
    mgr = P.StateManager(device=c.local, rank=c.rank, world=c.world, bucket_bytes=a.bucket_mb << 20, timing=True)
    plans, jobs, arenas = [], [], []
    for j, mo in enumerate(models):
        tp = 1 if mo == "qwen2.5-0.5b" or c.world == 1 else 2
        pl = mgr.plan(manifest(mo), head_dim=MODELS[mo].head_dim, tp=tp, dp=c.world // tp, rank_map=L.RANKMAP_AUTO)
        plans.append(pl)
        jb = P.Job(mgr, pl, seed=j).alloc().init_synthetic()
        jb.suspend()
        jobs.append(jb)
        arenas.append(mgr.arena(pl))
    psize = [plans[j].stats().total_params / plans[3].stats().total_params for j in range(4)]
    compute = [38.08 * psize[j] * a.time_scale for j in range(4)]      # update_actor
    schedule = list(range(4)) * a.rounds

    def blocking():
        boundary = 0.0
        resident = None
        for j in schedule:
            t = time.perf_counter()
            if resident is None:
                jobs[j].resume()
            else:
                jobs[resident].switch_to(jobs[j])
            jobs[j].sync(arenas[j])
            torch.cuda.synchronize()
            boundary += time.perf_counter() - t
            time.sleep(compute[j])
            resident = j
        jobs[resident].suspend()
        return boundary

    def overlapped():
        boundary = 0.0
        jobs[schedule[0]].resume()
        for v, j in enumerate(schedule):
            p = schedule[v - 1] if v > 0 else None
            t = time.perf_counter()
            if v > 0:
                jobs[j].wait_prefetch()                   # started during p's compute
            jobs[j].sync(arenas[j])
            torch.cuda.synchronize()
            boundary += time.perf_counter() - t
            if p is not None:
                jobs[p].drain()                           # off the critical path, during j's compute
            if v + 1 < len(schedule):
                jobs[schedule[v + 1]].prefetch()          # ditto for the next job
            time.sleep(compute[j])
            if p is not None:
                t = time.perf_counter()
                jobs[p].wait_drain()                      # normally long done
                boundary += time.perf_counter() - t
        jobs[schedule[-1]].suspend()
        return boundary

    t_block = blocking()
    t_over = overlapped()
    c.emit({"scenario": "overlap", "jobs": models, "n_gpus": c.world, "visits": len(schedule),
            "time_scale": a.time_scale, "compute_s_per_visit": [round(x, 3) for x in compute],
            "blocking_boundary_s_total": round(c.allmax(t_block), 3),
            "overlapped_boundary_s_total": round(c.allmax(t_over), 3),
            "note": "boundary = time the group is not running the active job's compute (switch + sync)"}, a.out)


def scen_nvme(a, c: Ctx):
    """NEXT-4 cold tier: spill a suspended job's slab to local storage with
    O_DIRECT and fill it back; the next resume verifies it."""
    model = a.model or "qwen2.5-1.5b"
    mgr = P.StateManager(device=c.local, rank=c.rank, world=c.world, bucket_bytes=a.bucket_mb << 20)
    plan = mgr.plan(manifest(model))
    job = P.Job(mgr, plan, seed=5).alloc().init_synthetic()
    job.suspend()
    path = os.path.join(a.spill_dir, f"plex_slab_r{c.rank}.bin")
    n = plan.rank_info(c.rank).slab_bytes
    c.barrier()
    t0 = time.perf_counter()
    job.slab.spill(path, threads=a.io_threads)
    t1 = time.perf_counter()
    job.slab.fill(path, threads=a.io_threads)
    t2 = time.perf_counter()
    job.resume()                                   # checksum-verified
    os.remove(path)
    # NEXT-3 checkpoint materialisation: written in the background while the
    # job computes (here: while it is resumed), restored into a fresh slab
    job.suspend(release=False)
    ck = os.path.join(a.spill_dir, f"plex_ckpt_r{c.rank}.safetensors")
    c.barrier()
    t3 = time.perf_counter()
    th = job.slab.checkpoint(ck, threads=a.io_threads, background=True)
    job.resume()
    t4 = time.perf_counter()
    th.join()
    t5 = time.perf_counter()
    assert not th.errors
    slab2 = P.Slab(plan, c.rank)
    t6 = time.perf_counter()
    slab2.restore(ck, threads=a.io_threads)
    t7 = time.perf_counter()
    job.slab = slab2
    job.resume()                                   # verified against the file's checksums
    os.remove(ck)
    c.emit({"scenario": "nvme", "model": model, "n_gpus": c.world, "slab_bytes_per_rank": n,
            "spill_GBs_per_rank": round(n / (c.allmax(t1 - t0)) / 1e9, 2),
            "fill_GBs_per_rank": round(n / (c.allmax(t2 - t1)) / 1e9, 2),
            "checkpoint_GBs_per_rank": round(n / (c.allmax(t5 - t3)) / 1e9, 2),
            "resume_during_checkpoint_ms": round(1e3 * c.allmax(t4 - t3), 1),
            "restore_GBs_per_rank": round(n / (c.allmax(t7 - t6)) / 1e9, 2), "io_threads": a.io_threads,
            "dir": a.spill_dir}, a.out)


def scen_optim(a, c: Ctx):
    # each process = rank c.rank of an FSDP-8 plan; k = world processes copy at once
    W = 8
    shape = MODELS[a.model]
    mgr = P.StateManager(device=c.local, rank=c.rank, world=W, bucket_bytes=a.bucket_mb << 20, bootstrap=False,
                         timing=True)
    plan = mgr.plan(manifest(a.model), world=W, kind_mask=L.KINDMASK_OPTIM)
    job = P.Job(mgr, plan, seed=2).alloc(kinds=(1, 2, 3)).init_synthetic()

    def step():
        job.suspend(release=False)
        job.resume()

    ms, clk = timed(c, step, a.steps, a.warmup)
    S = plan.rank_info(c.rank).payload_bytes
    st = mgr.stats()
    d2h = st["d2h"]["bytes"] / (st["d2h"]["ms"] * 1e-3) / 1e9
    h2d = st["h2d"]["bytes"] / (st["h2d"]["ms"] * 1e-3) / 1e9
    c.emit({"scenario": "optim-offload", "model": a.model, "k_gpus": c.world, "fsdp": W,
            "optimizer_bytes_per_gpu": S, "aggregate_bytes": c.allsum(float(S)),
            "ms_offload_plus_onload": round(ms, 2),
            "per_gpu_GBs_each_way": round(2 * S / (ms * 1e-3) / 1e9, 2),
            "rank0_copy_engine_GBs": {"d2h": round(d2h, 2), "h2d": round(h2d, 2)}, "clocks": clk,
            "note": "paper's context: 19.0 s optimizer-state load for 30B (PAPER.md:604), bytes/ranks unstated"},
           a.out)
    _ = shape


def scen_m2rank(a, c: Ctx):
    """configs[1] per-GPU workload at k GPUs: each process is rank c.rank of the
    M2 plan (Qwen2.5-7B FSDP-8 -> TP-2 x DP-4, AUTO rank map) and switches the
    GPU between two such jobs through the group executor (duplex: offload A ||
    onload B, 13.33 GB each way per GPU).  k = WORLD_SIZE GPUs switch at once,
    sharing the box's host memory system as 8 ranks of a real 8-GPU box would
    share theirs.  The M2 sync is not run here (it needs all 8 ranks' peers);
    its NVLink bound from the plan's ledger is reported next to it."""
    W = 8
    model = "qwen2.5-7b"
    mgr = P.StateManager(device=c.local, rank=c.rank, world=W, bucket_bytes=a.bucket_mb << 20, bootstrap=False,
                         timing=True)
    plan = mgr.plan(manifest(model), head_dim=MODELS[model].head_dim, world=W, tp=2, dp=4, rank_map=L.RANKMAP_AUTO)
    ja = P.Job(mgr, plan, seed=1).alloc().init_synthetic()
    jb = P.Job(mgr, plan, seed=2).alloc().init_synthetic()
    jb.suspend()
    group = P.Group(mgr)
    group.add(ja, resident=True)
    group.add(jb)
    modes = {}
    cur = {"j": ja}

    def step():
        nxt = jb if cur["j"] is ja else ja
        res = group.transition(nxt)
        modes[res["mode"]] = modes.get(res["mode"], 0) + 1
        cur["j"] = nxt

    ms, clk = timed(c, step, a.steps, a.warmup, min_s=0)
    S = plan.rank_info(c.rank).payload_bytes
    st = mgr.stats()
    d2h = st["d2h"]["bytes"] / (st["d2h"]["ms"] * 1e-3) / 1e9
    h2d = st["h2d"]["bytes"] / (st["h2d"]["ms"] * 1e-3) / 1e9
    led = plan.ledger()
    nv = max(max(int(led[r].sum() - led[r, r]), int(led[:, r].sum() - led[r, r])) for r in range(W))
    c.emit({"scenario": "m2rank", "model": model, "plan": "FSDP-8 -> TP-2xDP-4 (AUTO rank map)", "k_gpus": c.world,
            "state_bytes_per_gpu": S, "switch_ms_max_rank": round(ms, 2), "modes": modes,
            "GBs_per_gpu_each_way": round(S / (ms * 1e-3) / 1e9, 2),
            "rank0_copy_engine_GBs": {"d2h": round(d2h, 2), "h2d": round(h2d, 2)},
            "m2_sync_nvlink_bound_ms": round(nv / 770e9 * 1e3, 2), "m2_sync_busiest_link_bytes": nv,
            "clocks": clk}, a.out)


def scen_moe(a, c: Ctx):
    model = "qwen3-30b-a3b"
    shape = MODELS[model]
    tp = min(2, c.world)
    mgr = P.StateManager(device=c.local, rank=c.rank, world=c.world, bucket_bytes=a.bucket_mb << 20, timing=True)
    plan = mgr.plan(manifest(model), head_dim=shape.head_dim, tp=tp, dp=c.world // tp, ep=c.world,
                    rank_map=L.RANKMAP_AUTO)
    job = P.Job(mgr, plan, seed=3, slab=False).alloc(kinds=(1,)).init_synthetic()
    arena = mgr.arena(plan)
    mgr.reset_stats()
    ms_sync, clk = timed(c, lambda: job.sync(arena), a.steps, a.warmup)
    st = mgr.stats()
    push_ms = c.allmax(st["push"]["ms"] / max(1, st["push"]["launches"]))
    info = plan.rank_info(c.rank)
    nv = c.allmax(float(max(info.send_bytes, info.recv_bytes)))
    # per-expert units: KEY_MAJOR slab of the first --units (layer, expert) units
    from plexgen.models import expert_keys
    units = [(l, e) for l in range(shape.layers) for e in range(shape.experts)][:a.units]
    keys = expert_keys(model, units)
    uplan = mgr.plan(manifest(model), slab_layout=L.SLAB_KEY_MAJOR, subset=keys)
    ujob = P.Job(mgr, uplan, seed=3)
    for k in keys:                                    # share the master shards, add the other kinds
        t = uplan.index[k]
        shp = uplan.shard_shape(c.rank, t)
        for kd in range(4):
            ujob.shards[(k, kd)] = job.shards[(k, 1)] if kd == 1 else \
                torch.empty(shp, dtype=P.state.KIND_TORCH[kd], device=f"cuda:{c.local}")
    ms_unit, _ = timed(c, lambda: (ujob.suspend(release=False), ujob.resume()), a.steps, a.warmup)
    ub = uplan.rank_info(c.rank).payload_bytes
    c.emit({"scenario": "moe", "model": model, "n_gpus": c.world, "layout": f"attn TP-{tp}xDP-{c.world // tp}, EP-{c.world}",
            "sync_ms": round(ms_sync, 3), "push_kernel_ms": round(push_ms, 3), "nvlink_bytes_max_rank": nv,
            "nvlink_GBs_push_kernel": round(nv / (push_ms * 1e-3) / 1e9, 1) if c.world > 1 else None,
            "rank_map": plan.stats().rank_map,
            "units": a.units, "unit_bytes_per_gpu": ub // max(1, a.units),
            "unit_offload_onload_ms": round(ms_unit, 3), "clocks": clk}, a.out)


def scen_sync(a, c: Ctx):
    """Weight sync alone for any dense config (e.g. configs[2]: Qwen2.5-32B
    FSDP-N -> TP-4 x DP; at 4 GPUs FSDP-4 -> TP-4), masters only on the device,
    both transports."""
    model = a.model or "qwen2.5-32b"
    shape = MODELS[model]
    tp = a.tp or min(4, c.world)
    out = {}
    runs = [("push", 64 << 10), ("nccl", 64 << 10)]
    if a.tiles:
        runs = [("push", int(t)) for t in a.tiles.split(",")]
    for transport, tile in runs:
        mgr = P.StateManager(device=c.local, rank=c.rank, world=c.world, bucket_bytes=256 << 20, timing=True,
                             sync_nccl=transport == "nccl", duplex=False)
        plan = mgr.plan(manifest(model), head_dim=shape.head_dim, tp=tp, dp=c.world // tp, rank_map=L.RANKMAP_AUTO,
                        tile_bytes=tile)
        job = P.Job(mgr, plan, seed=2, slab=False).alloc(kinds=(1,)).init_synthetic()
        arena = mgr.arena(plan)
        mgr.reset_stats()
        ms, clk = timed(c, lambda: job.sync(arena), a.steps, a.warmup)
        st = mgr.stats()
        info = plan.rank_info(c.rank)
        nv = c.allmax(float(max(info.send_bytes, info.recv_bytes)))
        # data-moving time: the push kernel, or (NCCL) the whole call -- the
        # per-round exchange events include waiting for peers' K4 rounds
        t_x = c.allmax(st["push"]["ms"] / max(1, st["push"]["launches"])) if transport == "push" else ms
        out[transport if not a.tiles else f"push_tile_{tile >> 10}KiB"] = {"sync_ms": round(ms, 3), "data_ms": round(t_x, 3),
                          "nvlink_GBs": round(nv / (t_x * 1e-3) / 1e9, 1) if c.world > 1 and t_x > 0 else None}
        del job, arena, plan
        mgr.close()
        torch.cuda.empty_cache()
    c.emit({"scenario": "sync", "model": model, "n_gpus": c.world, "layout": f"FSDP-{c.world}->TP-{tp}xDP-{c.world // tp}",
            "nvlink_bytes_max_rank": nv, **out, "clocks": clk}, a.out)


def scen_multiplex(a, c: Ctx):
    """configs[4]: 4 jobs shaped 0.5B / 1.5B / 3B / 7B
    (seeds 0..3) time-slice the GPU group round-robin for --rounds rounds
    (default 5: 20 visits, 19 switches).  Every visit goes through the
    library's residency authority (plex_group_transition: it decides the
    ops and picks duplex / sequential from what fits), then one
    simulated training step (synth_mutate) and the weight sync through the
    group.  Full-size parity of the same trace: tests/test_gpu_fullsize_configs.py
    ::test_m5_multiplex_trace_fullsize."""
    from paper_2605_20863_b200.state import synth_mutate
    models = ["qwen2.5-0.5b", "qwen2.5-1.5b", "qwen2.5-3b", "qwen2.5-7b"]
    mgr = P.StateManager(device=c.local, rank=c.rank, world=c.world, bucket_bytes=a.bucket_mb << 20, timing=True)
    group = P.Group(mgr)
    plans, jobs, arenas = [], [], []
    for j, mo in enumerate(models):
        tp = 1 if mo == "qwen2.5-0.5b" or c.world == 1 else 2
        pl = mgr.plan(manifest(mo), head_dim=MODELS[mo].head_dim, tp=tp, dp=c.world // tp)
        plans.append(pl)
        jb = P.Job(mgr, pl, seed=j).alloc().init_synthetic()
        jb.suspend()
        group.add(jb)
        jobs.append(jb)
        arenas.append(mgr.arena(pl))
    schedule = list(range(4)) * a.rounds
    steps = [0] * 4
    modes: dict = {}
    ms_switch = []

    def mutate(j):
        for t, (key, shape) in enumerate(plans[j].manifest):
            a0, _ = plans[j].shard_rows(c.rank, t)
            re_ = int(np.prod(shape[1:])) if len(shape) > 1 else 1
            for kd in range(4):
                synth_mutate(jobs[j].shards[(key, kd)], kd, j, steps[j], key, a0 * re_)
        steps[j] += 1

    def run_trace():
        for j in schedule:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            res = group.transition(jobs[j])                       # the library decides and executes
            e1.record()
            modes[res["mode"]] = modes.get(res["mode"], 0) + 1
            mutate(j)                                             # simulated training step
            group.transition(jobs[j], sync=arenas[j])             # [SYNC j]
            torch.cuda.synchronize()
            ms_switch.append(e0.elapsed_time(e1))

    ms, clk = timed(c, run_trace, 1, 0, min_s=0)
    c.emit({"scenario": "multiplex", "jobs": models, "n_gpus": c.world, "rounds": a.rounds,
            "visits": len(schedule), "switches": len(schedule) - 1, "executor": "plex_group_transition",
            "modes": modes, "trace_ms": round(ms, 1), "ms_per_visit": round(ms / len(schedule), 1),
            "switch_ms_max_rank_sum": round(c.allmax(float(sum(ms_switch))), 1),
            "state_gb_per_rank": [round(pl.rank_info(c.rank).payload_bytes / 1e9, 2) for pl in plans],
            "clocks": clk}, a.out)


def scen_zero2(a, c: Ctx):
    """NEXT-2 canonical dedup under ZeRO-2: the bf16 params are
    replicated on every rank.  naive = every rank offloads/onloads its full
    replica plus its optimizer shards; dedup = every rank moves only its FSDP
    rows of the replica (replica_param plan) and resume restores the rest with
    the NVLink all-gather (plex_param_allgather).  Step = suspend + resume."""
    man = manifest(a.model)
    B = a.bucket_mb << 20
    mgr = P.StateManager(device=c.local, rank=c.rank, world=c.world, bucket_bytes=B, timing=True, duplex=False)
    out = {}
    # dedup
    plan = mgr.plan(man, replica_param=True)
    job = P.Job(mgr, plan, seed=5).alloc().init_synthetic()
    ref = {k: P.checksum(v).cpu() for k, v in job.shards.items() if k[1] == 0}
    mgr.reset_stats()
    ms, clk = timed(c, lambda: (job.suspend(), job.resume()), a.steps, a.warmup)
    st = mgr.stats()
    ok = all(torch.equal(P.checksum(v).cpu(), ref[k]) for k, v in job.shards.items() if k[1] == 0)
    info = plan.rank_info(c.rank)
    n = a.steps + a.warmup
    out["dedup"] = {"suspend_resume_ms": round(ms, 1), "host_bytes_per_rank_each_way": info.slab_bytes,
                    "gather_ms_per_step": round(st["gather"]["ms"] / max(1, n), 2),
                    "gather_send_bytes": info.gather_send_bytes, "replicas_restored_bit_exact": bool(c.allmin(ok))}
    del job, plan
    torch.cuda.empty_cache()
    # naive: full replica through the host link on every rank
    mgr1 = P.StateManager(device=c.local, rank=0, world=1, bucket_bytes=B, bootstrap=False, duplex=False)
    plan_p = mgr1.plan(man, kind_mask=1 << L.KIND_PARAM)
    plan_o = mgr.plan(man, kind_mask=L.KINDMASK_OPTIM)
    jp = P.Job(mgr1, plan_p, seed=5, rank=0).alloc(kinds=(0,)).init_synthetic()
    jo = P.Job(mgr, plan_o, seed=5).alloc(kinds=(1, 2, 3)).init_synthetic()

    def naive():
        jp.suspend()
        jo.suspend()
        jp.resume()
        jo.resume()

    ms2, _ = timed(c, naive, a.steps, a.warmup)
    out["naive"] = {"suspend_resume_ms": round(ms2, 1),
                    "host_bytes_per_rank_each_way": plan_p.rank_info(0).slab_bytes + plan_o.rank_info(c.rank).slab_bytes}
    del jp, jo
    mgr1.close()
    c.emit({"scenario": "zero2", "model": a.model, "n_gpus": c.world, **out,
            "host_bytes_ratio": round(out["naive"]["host_bytes_per_rank_each_way"] /
                                      out["dedup"]["host_bytes_per_rank_each_way"], 3),
            "speedup": round(ms2 / ms, 3), "clocks": clk}, a.out)


def scen_carry(a, c: Ctx):
    """NEXT-1 host-link balancing transports: the 7B duplex switch with rank 0's
    link declared at half speed (so its last buckets are carried by the other
    ranks), carried over peer memory (default: the carrier's copy engine reads /
    writes the owner's slot over NVLink) vs NCCL send/recv through the
    carrier's staging, and without carrying.  Bit-exact restores checked by
    checksums."""
    man = manifest(a.model)
    shape = MODELS[a.model]
    tp = a.tp or min(2, c.world)
    out = {}
    for name, kw, weights in (("no_carry", {}, None),
                              ("peer_memory", {}, [0.5] + [1.0] * (c.world - 1)),
                              ("nccl", {"carry_nccl": True}, [0.5] + [1.0] * (c.world - 1))):
        mgr = P.StateManager(device=c.local, rank=c.rank, world=c.world, bucket_bytes=a.bucket_mb << 20,
                             timing=True, **kw)
        plans = [mgr.plan(man, head_dim=shape.head_dim, tp=tp, dp=c.world // tp, link_weights=weights)
                 for _ in range(2)]
        for pl in plans:
            mgr.enable_carry(pl)
        jobs = [P.Job(mgr, pl, seed=s).alloc().init_synthetic() for pl, s in zip(plans, (1, 2))]
        ref = [{k: P.checksum(v).cpu() for k, v in j.shards.items()} for j in jobs]
        jobs[1].suspend()
        state = {"cur": 0}

        def step():
            i = state["cur"]
            jobs[i].switch_to(jobs[1 - i])
            state["cur"] = 1 - i

        ms, clk = timed(c, step, a.steps, a.warmup)
        cur = jobs[state["cur"]]
        ok = all(torch.equal(P.checksum(v).cpu(), ref[state["cur"]][k]) for k, v in cur.shards.items())
        out[name] = {"switch_ms": round(ms, 1), "carried_buckets_per_job": len(plans[0].carry()),
                     "bit_exact": bool(c.allmin(1.0 if ok else 0.0) > 0.5)}
        del jobs, plans
        mgr.close()
        torch.cuda.empty_cache()
    c.emit({"scenario": "carry", "model": a.model, "n_gpus": c.world, **out}, a.out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenario", required=True, choices=["duplex", "elide", "optim", "moe", "multiplex", "hrrs", "overlap", "nvme", "sync", "zero2", "carry",
                             "m2rank"])
    ap.add_argument("--spill-dir", default="/tmp")
    ap.add_argument("--io-threads", type=int, default=8)
    ap.add_argument("--time-scale", type=float, default=0.005)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--model", default="")
    ap.add_argument("--tp", type=int, default=0)
    ap.add_argument("--bucket-mb", type=int, default=2048)
    ap.add_argument("--units", type=int, default=64)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--duplex", action="store_true")
    ap.add_argument("--tiles", default="", help="sync scenario: push-kernel tile sizes (bytes) to compare")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    c = Ctx(a.gpus)
    if not a.model:
        a.model = {"duplex": "qwen2.5-7b", "elide": "qwen2.5-7b", "optim": "qwen2.5-32b", "zero2": "qwen2.5-7b", "carry": "qwen2.5-7b"}.get(a.scenario, "")
    {"duplex": scen_duplex, "elide": scen_elide, "optim": scen_optim, "moe": scen_moe,
     "multiplex": scen_multiplex, "hrrs": scen_hrrs, "m2rank": scen_m2rank, "overlap": scen_overlap, "nvme": scen_nvme,
     "sync": scen_sync, "zero2": scen_zero2, "carry": scen_carry}[a.scenario](a, c)
    c.barrier()
    if c.world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
