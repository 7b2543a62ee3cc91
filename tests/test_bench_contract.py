"""bench.py's JSON contract, checked on CPU through the reference arm (the
CPU oracle on a bounded sample; the CUDA arm needs a GPU)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--model", "mid",
                        "--steps", "2", "--warmup", "1", "--cpu-sample-layers", "1"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["unit"] == d["unit"]
    assert d["value"] > 0


import pytest  # noqa: E402


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [[], ["--swap"]])
def test_cuda_arm_json_line(extra):
    """The CUDA arm on a small shape: every contract key, a roofline object for the
    dominant kernel, clocks sampled during the timed region, our launches counted."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--model", "mid", "--steps", "3",
                        "--warmup", "3", "--bucket-mb", "1", "--no-cpu-baseline"] + extra,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "rooflines", "clocks", "e2e",
              "gpu_launches"):
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    rl = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rl, k
    assert rl["bound"] == "hbm" and 0 < rl["frac"] < 1.5 and rl["unit"] == "GB/s"
    assert d["config"]["workload"] and d["config"]["switch_mode"] == ("swap" if extra else "duplex")
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] > 0 and "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    # every switch was decided and executed by the library's group executor (a1)
    assert "plex_group_transition" in d["config"]["executor"]
    assert d["config"]["executor"].endswith(("['swap'])", "['duplex'])"))
    if extra:                                 # the labelled derived-param (NEXT-2 elision) sub-line
        dv = d["derived_param"]
        assert dv["elided"] is True and dv["value"] > 0
        assert dv["host_link_bytes_per_step"] < dv["state_bytes_switched_per_step"]
