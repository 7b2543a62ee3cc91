"""Full-size oracle evaluation fanned out over the host's cores (TEST
INFRASTRUCTURE: only the full-size GPU tests use it).

The oracle functions run as they stand (plexgen's generator, O.checksum,
O.rne_bf16, O.rollout_tensors); this module only splits the work into
tensor / segment chunks and runs them on a thread pool (NumPy releases the GIL
inside its array operations), so a 100 GB state can be regenerated and
compared byte for byte within the slow tier's budget.  Chunks of one segment
are combined with R14's additivity (pinned in tests/test_oracle_checksum.py).
"""
from __future__ import annotations

import os
from collections import OrderedDict
from concurrent.futures import ThreadPoolExecutor
from typing import Dict, List, Sequence, Tuple

import numpy as np

from oracle import plex_oracle as O
from plexgen import gen_range

CHUNK = 1 << 23                     # elements per task
M64 = (1 << 64) - 1


def workers(cap: int = 32) -> int:
    return max(1, min(cap, len(os.sched_getaffinity(0))))


def check_slab(seed: int, man, segs, host: np.ndarray, special_bits: int = 0,
               threads: int = 0) -> Tuple[np.ndarray, List[Tuple[str, int]]]:
    """Every slab byte vs the oracle's regeneration of its segment, and the
    oracle's (S1, S2) of every segment.  ``segs`` are the product plan's
    segment descriptors (tensor, kind, slab_offset, nbytes, index_base).
    Returns (checksums [n_seg, 2] uint64, [(key, kind) of segments whose bytes differ])."""
    tasks = []
    for i, s in enumerate(segs):
        es = 2 if s.kind == 0 else 4
        n = s.nbytes // es
        for o in range(0, max(n, 1), CHUNK):
            tasks.append((i, o, min(CHUNK, n - o)))

    def run(t):
        i, o, c = t
        s = segs[i]
        key = man[s.tensor][0]
        es = 2 if s.kind == 0 else 4
        if c <= 0:
            return i, 0, 0, True
        want = gen_range(seed, key, s.kind, s.index_base + o, c, special_bits if s.kind else 0)
        lo = s.slab_offset + o * es
        got = host[lo:lo + c * es].view(want.dtype)
        a, b = O.checksum(want, s.index_base + o)
        return i, a, b, bool(np.array_equal(got, want))

    cks = np.zeros((len(segs), 2), dtype=np.uint64)
    acc = [[0, 0] for _ in segs]
    bad = set()
    with ThreadPoolExecutor(threads or workers()) as ex:
        for i, a, b, ok in ex.map(run, tasks):
            acc[i][0] = (acc[i][0] + a) & M64
            acc[i][1] = (acc[i][1] + b) & M64
            if not ok:
                bad.add(i)
    for i, (a, b) in enumerate(acc):
        cks[i] = (a, b)
    return cks, sorted((man[segs[i].tensor][0], segs[i].kind) for i in bad)


def _layer_groups(man) -> List[List[Tuple[str, Tuple[int, ...]]]]:
    """Manifest split into units whose rollout tensors depend only on themselves:
    one decoder layer, or one top-level tensor (embed, norm, lm_head)."""
    out: "OrderedDict[str, list]" = OrderedDict()
    for k, s in man:
        if k.startswith("model.layers."):
            g = ".".join(k.split(".")[:3])
        else:
            g = k
        out.setdefault(g, []).append((k, s))
    return list(out.values())


def rollout_checksums(seed: int, man, tp: int, dp: int, ep: int, rank_map: int, head_dim: int,
                      special_bits: int = 0, threads: int = 0) -> Dict[Tuple[int, str], Tuple[int, int]]:
    """(S1, S2) of every rollout tensor of every destination rank g, from the
    oracle's c1.3 definition: gather (the full master, regenerated) -> RNE ->
    slice_g / fuse_g (O.rollout_tensors), one decoder layer per task."""
    W = tp * dp

    def run(group):
        full = OrderedDict()
        for k, s in group:
            n = 1
            for d in s:
                n *= d
            full[k] = O.rne_bf16(gen_range(seed, k, 1, 0, n, special_bits)).reshape(s)
        res = {}
        for g in range(W):
            for name, x in O.rollout_tensors(full, tp, dp, ep, g, rank_map, head_dim).items():
                res[(g, name)] = O.checksum(x, 0)
        return res

    out: Dict[Tuple[int, str], Tuple[int, int]] = {}
    with ThreadPoolExecutor(threads or workers(16)) as ex:
        for r in ex.map(run, _layer_groups(man)):
            out.update(r)
    return out


def tensor_bits(seed: int, key: str, kind: int, index_base: int, count: int, special_bits: int = 0) -> np.ndarray:
    return gen_range(seed, key, kind, index_base, count, special_bits if kind else 0)


def sample_keys(man: Sequence[Tuple[str, Tuple[int, ...]]], n: int, seed: int = 0) -> List[str]:
    """n random manifest keys plus the largest tensor."""
    rng = np.random.default_rng(seed)
    keys = [k for k, _ in man]
    pick = set(rng.choice(len(keys), size=min(n, len(keys)), replace=False).tolist())
    sizes = [int(np.prod(s)) for _, s in man]
    pick.add(int(np.argmax(sizes)))
    return [keys[i] for i in sorted(pick)]


def tensor_checksums(seed: int, man, kinds=(0, 1, 2, 3), special_bits: int = 0,
                     threads: int = 0) -> Dict[Tuple[str, int], Tuple[int, int]]:
    """The oracle's (S1, S2) of every logical (key, kind) tensor of the initial
    synthetic state, chunked (R14 additivity) over the host's cores."""
    tasks = []
    for k, s in man:
        n = 1
        for d in s:
            n *= d
        for kd in kinds:
            for o in range(0, max(n, 1), CHUNK):
                tasks.append((k, kd, o, min(CHUNK, n - o)))

    def run(t):
        k, kd, o, c = t
        if c <= 0:
            return k, kd, 0, 0
        a, b = O.checksum(gen_range(seed, k, kd, o, c, special_bits if kd else 0), o)
        return k, kd, a, b

    out: Dict[Tuple[str, int], List[int]] = {}
    with ThreadPoolExecutor(threads or workers()) as ex:
        for k, kd, a, b in ex.map(run, tasks):
            acc = out.setdefault((k, kd), [0, 0])
            acc[0] = (acc[0] + a) & M64
            acc[1] = (acc[1] + b) & M64
    return {kk: (v[0], v[1]) for kk, v in out.items()}
