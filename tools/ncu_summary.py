#!/usr/bin/env python
"""Summarise the ncu evidence of one tools/ncu_run.sh run into profiles/.

    python tools/ncu_summary.py <tag>

Reads gpurun_out/<tag>_launches.csv (per-launch gpu__time_duration, cold and
serialised) and gpurun_out/<tag>_{pack,push}.ncu-rep (--set full), writes
profiles/<tag>_ncu_summary.md and merges per-launch DRAM traffic into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
           "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__shared_mem_per_block_dynamic"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = r[i].replace(",", "")
                try:
                    f = float(v)
                except ValueError:
                    d[m] = v
                    continue
                u = units[i]
                if m.startswith("dram__bytes"):
                    f *= UNIT.get(u, 1)
                elif m == "gpu__time_duration.sum":            # always microseconds
                    f *= {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}.get(u, 1.0)
                    u = "us"
                d[m] = f
                d[m + ".unit"] = u
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[i]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[i + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] in ("nsecond", "ns") else v * 1e3 if r[ui] in ("msecond", "ms") else v
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    return agg


def main():
    tag = sys.argv[1]
    g = os.path.join(ROOT, "gpurun_out")
    lines = [f"# ncu summary — {tag}", ""]
    lp = os.path.join(g, f"{tag}_launches.csv")
    if os.path.exists(lp):
        agg = launches(lp)
        tot = sum(v[1] for v in agg.values())
        lines += ["## Launch list (`--metrics gpu__time_duration.sum --clock-control none`, cold + serialised)", "",
                  "| kernel | launches | total µs | share |", "|---|---|---|---|"]
        for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{k}` | {n} | {us:.1f} | {us / tot:.1%} |")
        lines.append("")
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for which in ("pack", "push"):
        rep = os.path.join(g, f"{tag}_{which}.ncu-rep")
        if not os.path.exists(rep):
            continue
        res = raw(rep)
        lines += [f"## `--set full` capture: {which} kernel", "", "| metric | " +
                  " | ".join(f"launch {i}" for i in range(len(res))) + " |",
                  "|---|" + "---|" * len(res)]
        for m in METRICS:
            vals = []
            for d in res:
                v = d.get(m)
                unit = "B" if m.startswith("dram__bytes") else d.get(m + ".unit", "")
                vals.append(f"{v:,.1f} {unit}".strip() if isinstance(v, float) else str(v))
            lines.append(f"| {m} | " + " | ".join(vals) + " |")
        lines.append(f"| kernel | " + " | ".join(d["kernel"][:60] for d in res) + " |")
        lines.append("")
        groups = {}
        for d in res:      # pack_kernel<1,...> = K1 pack, pack_kernel<0,...> = K2 unpack
            k = which
            if which == "pack" and "pack_kernel<0" in d["kernel"].replace("(bool)0", "0").replace(" ", ""):
                k = "unpack"
            groups.setdefault(k, []).append(d)
        for k, ds in groups.items():
            rd = [d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in ds]
            traffic[k] = {"dram_bytes_per_launch": sum(rd) / len(rd), "source": f"profiles/{tag}_ncu_summary.md (capture gpurun_out/{tag}_{which}.ncu-rep, not committed)",
                          "duration_us": sum(d.get("gpu__time_duration.sum", 0) for d in ds) / len(ds),
                          "launches": len(ds)}
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    out = os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md")
    open(out, "w").write("\n".join(lines) + "\n")
    print(out)


if __name__ == "__main__":
    main()
