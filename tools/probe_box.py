"""Probe a GPU box: topology, host memory, pinned-copy bandwidth (1..k GPUs concurrently).

Infra script (not product): measures the host-link roofline BW_host(k, dir) of
SURVEY.md §8(d) D3 with torch pinned buffers and cudaMemcpyAsync via Tensor.copy_.
"""
import json, os, subprocess, sys, threading, time
import torch

def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)

out = {}
out["topo"] = sh("nvidia-smi topo -m")
out["free"] = sh("free -g")
out["ulimit_l"] = sh("ulimit -l")
out["lscpu"] = sh("lscpu | head -30")
out["numa"] = sh("cat /sys/devices/system/node/online; ls /sys/devices/system/node")
out["affinity"] = len(os.sched_getaffinity(0))
out["meminfo"] = sh("grep -i -E 'huge|MemTotal|MemAvail' /proc/meminfo")
out["smi"] = sh("nvidia-smi --query-gpu=index,name,pci.bus_id,memory.total,clocks.max.sm,pcie.link.gen.max,pcie.link.width.max --format=csv")
ng = torch.cuda.device_count()
out["ngpu"] = ng
GB = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nbytes = GB << 30
bufs = []
for d in range(ng):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    g = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{d}")
    bufs.append((h, g))

def run(devs, direction, reps=3):
    res = {}
    barrier = threading.Barrier(len(devs))
    def w(d):
        torch.cuda.set_device(d)
        h, g = bufs[d]
        s = torch.cuda.Stream(d)
        best = 0.0
        for _ in range(reps):
            barrier.wait()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                if direction == "d2h":
                    h.copy_(g, non_blocking=True)
                else:
                    g.copy_(h, non_blocking=True)
                e1.record(s)
            e1.synchronize()
            best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        res[d] = best
    ts = [threading.Thread(target=w, args=(d,)) for d in devs]
    [t.start() for t in ts]; [t.join() for t in ts]
    return res

bw = {}
for k in [1, 2, 4, 8]:
    if k > ng:
        break
    for dr in ("d2h", "h2d"):
        r = run(list(range(k)), dr)
        bw[f"k{k}_{dr}"] = {"per_gpu": r, "min": min(r.values()), "sum": sum(r.values())}
        print(k, dr, r, flush=True)
out["pinned_bw_GBs"] = bw
# HBM copy
torch.cuda.set_device(0)
a = torch.empty(1 << 32, dtype=torch.uint8, device="cuda:0"); b = torch.empty_like(a)
for _ in range(3): b.copy_(a)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(10): b.copy_(a)
e1.record(); e1.synchronize()
out["hbm_copy_GBs"] = 2 * a.numel() * 10 / (e0.elapsed_time(e1) * 1e-3) / 1e9
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k not in ("topo", "lscpu")}, indent=1))
print(out["topo"]); print(out["lscpu"])
