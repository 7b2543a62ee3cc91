"""How much host memory can one process pin?  cudaHostAlloc vs mmap+cudaHostRegister
(libplex slab flags), in 16 GiB slabs until failure (infra probe)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_20863_b200 as P  # noqa: E402
from paper_2605_20863_b200 import _lib as L  # noqa: E402

torch.cuda.set_device(0)
mode = sys.argv[1] if len(sys.argv) > 1 else "alloc"
gib = int(sys.argv[2]) if len(sys.argv) > 2 else 16
man = [("x", (gib << 30 >> 12, 1024))]
slabs = []
tot = 0
t0 = time.time()
for i in range(40):
    plan = P.Plan(man, world=1, kind_mask=0x2)
    try:
        t = time.time()
        s = P.Slab(plan, 0, hugepage=(mode == "huge"))
        slabs.append((plan, s))
        tot += gib
        print(f"{mode}: slab {i} ok, total {tot} GiB, {time.time() - t:.1f}s", flush=True)
    except P.PlexError as e:
        print(f"{mode}: FAILED at total {tot} GiB + {gib}: {e}", flush=True)
        break
print(f"{mode}: pinned {tot} GiB in {time.time() - t0:.1f}s", flush=True)
