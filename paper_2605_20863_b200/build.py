"""Build libplex.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python paper_2605_20863_b200/build.py          # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libplex.so")
SOURCES = ["plex_plan.cpp", "plex_group.cpp", "plex_kernels.cu", "plex_runtime.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir() -> str:
    # torch's own NCCL (nvidia-nccl-cu12 wheel): link the same libnccl.so.2
    # that torch loads so one process never holds two NCCLs.
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia.nccl wheel not found")
    return list(spec.submodule_search_locations)[0]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def build(verbose: bool = False, force: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, "plex_internal.h"),
                   os.path.join(os.path.dirname(HERE), "include", "plex.h")]
    if (not force and os.path.exists(OUT)
            and os.path.getmtime(OUT) >= max(os.path.getmtime(d) for d in deps)):
        return OUT
    nccl = _nccl_dir()
    cmd = [_nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(nccl, "include"), "-I", os.path.join(os.path.dirname(HERE), "include"),
           "-o", OUT + ".tmp", *srcs,
           "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
           "-Xlinker", "-rpath=" + os.path.join(nccl, "lib"), "-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libplex.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True))
