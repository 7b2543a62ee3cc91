"""The device-metadata workspace allocator (csrc/plex_heap.h, behind
plex_ctx_create's caller-owned workspace) on the host: a tiny g++ driver runs
random alloc / free sequences against a plain Python first-fit model, and the
invariants every CUDA table relies on are checked -- 256-B aligned blocks,
inside the region, never overlapping, exhaustion reported instead of an
overrun, and full coalescing once everything is freed."""
import os
import random
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = r'''
#include <cstdio>
#include "plex_heap.h"
int main() {
    plex::OffsetHeap h;
    char op;
    unsigned long long x;
    while (std::scanf(" %c %llu", &op, &x) == 2) {
        if (op == 'R') { h.reset(x); std::printf("ok\n"); }
        else if (op == 'A') { unsigned long long o = h.alloc(x); std::printf("%lld\n", o == plex::OffsetHeap::kNone ? -1LL : (long long)o); }
        else if (op == 'F') { std::printf("%d\n", h.free(x) ? 1 : 0); }
        else if (op == 'S') { std::printf("%llu %llu %zu %llu\n", (unsigned long long)h.in_use(),
                                          (unsigned long long)h.high_water(), h.free_blocks(),
                                          (unsigned long long)h.largest_free()); }
    }
    return 0;
}
'''


class Model:
    """First fit over a sorted free list with coalescing (what plex_heap.h claims to do)."""

    def __init__(self, n):
        self.n = n & ~255
        self.free = [[0, self.n]] if self.n else []
        self.used = {}
        self.in_use = self.hw = 0

    def alloc(self, n):
        need = (n + 255) & ~255
        for i, (o, s) in enumerate(self.free):
            if s >= need:
                if s == need:
                    self.free.pop(i)
                else:
                    self.free[i] = [o + need, s - need]
                self.used[o] = need
                self.in_use += need
                self.hw = max(self.hw, self.in_use)
                return o
        return -1

    def release(self, o):
        if o not in self.used:
            return 0
        s = self.used.pop(o)
        self.in_use -= s
        self.free.append([o, s])
        self.free.sort()
        merged = []
        for b in self.free:
            if merged and merged[-1][0] + merged[-1][1] == b[0]:
                merged[-1][1] += b[1]
            else:
                merged.append(b)
        self.free = merged
        return 1


@pytest.fixture(scope="module")
def driver(tmp_path_factory):
    if not shutil.which("g++"):
        pytest.skip("g++ not available")
    d = tmp_path_factory.mktemp("heap")
    src = d / "heap_driver.cpp"
    src.write_text(DRIVER)
    exe = d / "heap_driver"
    subprocess.run(["g++", "-O1", "-std=c++17", "-I", os.path.join(ROOT, "paper_2605_20863_b200", "csrc"),
                    str(src), "-o", str(exe)], check=True)
    return str(exe)


def run(exe, cmds):
    out = subprocess.run([exe], input="\n".join(cmds) + "\n", capture_output=True, text=True, check=True).stdout
    return out.split("\n")


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_heap_matches_first_fit_model(driver, seed):
    rng = random.Random(seed)
    size = rng.choice([1 << 20, (1 << 20) + 300, 64 << 10])
    m = Model(size)
    cmds, want = [f"R {size}"], ["ok"]
    live = []
    for _ in range(3000):
        if live and rng.random() < 0.45:
            o = live.pop(rng.randrange(len(live)))
            cmds.append(f"F {o}")
            want.append(str(m.release(o)))
        elif rng.random() < 0.03:
            bogus = rng.randrange(0, size) | 1                  # never a block start (odd)
            cmds.append(f"F {bogus}")
            want.append("0")
        else:
            n = rng.choice([1, 255, 256, 257, 4096, 10000, 65536, rng.randrange(1, size // 4)])
            o = m.alloc(n)
            cmds.append(f"A {n}")
            want.append(str(o))
            if o >= 0:
                live.append(o)
                # invariants of the model's answer (and thus of the driver's, compared below)
                assert o % 256 == 0 and o + n <= m.n
        if rng.random() < 0.05:
            cmds.append("S 0")
            want.append(f"{m.in_use} {m.hw} {len(m.free)} {max([s for _, s in m.free], default=0)}")
    for o in live:                                              # free everything: one block again
        cmds.append(f"F {o}")
        want.append(str(m.release(o)))
    cmds.append("S 0")
    want.append(f"0 {m.hw} 1 {m.n}")
    got = run(driver, cmds)
    assert got[:len(want)] == want


def test_heap_blocks_never_overlap_and_exhaustion_is_reported(driver):
    cmds = ["R 4096"] + ["A 1000"] * 5 + ["F 1024", "A 1024", "A 2048", "S 0"]
    got = run(driver, cmds)
    # 1000 B -> 1024-B blocks: four fit, the fifth is refused; a freed block is reused in place
    assert got[:10] == ["ok", "0", "1024", "2048", "3072", "-1", "1", "1024", "-1", "4096 4096 0 0"]
