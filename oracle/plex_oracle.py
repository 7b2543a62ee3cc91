"""CPU oracle for the PlexRL state-transition hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product (``paper_2605_20863_b200``) never imports it and shares
no code with it; the only common dependency is the input module ``plexgen``
(shape fixtures + counter-based value generator, no method arithmetic).

Plain, slow, obviously-correct NumPy.  Every function cites the passage of
/root/reference/PAPER.md (or the DESIGN.md reading, "R<n>", where the paper is
silent) it follows.  Element values are handled as raw bit patterns
(uint16 for bf16, uint32 for fp32) so that every comparison is bit-exact.

Pins (tests/test_oracle_*.py, marked ``not gpu``) tie each function to
something other than itself; see DESIGN.md §4.  Timing is "parity unpinned":
the paper prints no comparable number (R13).
"""
from __future__ import annotations

from collections import OrderedDict
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

KIND_PARAM, KIND_MASTER, KIND_EXP_AVG, KIND_EXP_AVG_SQ = 0, 1, 2, 3
ALL_KINDS = (0, 1, 2, 3)
OPTIM_KINDS = (1, 2, 3)
ELEM_BYTES = {0: 2, 1: 4, 2: 4, 3: 4}
ELEM_DTYPE = {0: np.uint16, 1: np.uint32, 2: np.uint32, 3: np.uint32}
SEG_ALIGN = 256                       # R4: 256-B segment alignment, zero padding
KIND_MAJOR, KEY_MAJOR = 0, 1          # R4 slab layouts
TP_FAST, DP_FAST = 0, 1               # R10 rank maps


# ---------------------------------------------------------------------------
# a8 / o6 — fp32 -> bf16 round-to-nearest-even (north_star; paper silent: R8)
# ---------------------------------------------------------------------------
def rne_bf16(u32: np.ndarray) -> np.ndarray:
    """R8: r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16; any NaN -> 0x7FC0.

    The paper only says weights are materialised "into the format expected by
    serving instances" (§4.5); the north_star fixes RNE.
    """
    u = np.asarray(u32, dtype=np.uint32).astype(np.uint64)
    r = ((u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16))
    out = (r & np.uint64(0xFFFF)).astype(np.uint16)
    is_nan = ((u & np.uint64(0x7F800000)) == np.uint64(0x7F800000)) & ((u & np.uint64(0x7FFFFF)) != 0)
    out[is_nan] = np.uint16(0x7FC0)
    return out


# ---------------------------------------------------------------------------
# o3 — FSDP-N dim-0 shards (north_star "FSDP shards"; paper: PAPER.md:524; R2)
# ---------------------------------------------------------------------------
def fsdp_rows(d0: int, world: int, rank: int) -> Tuple[int, int]:
    """R2: rank r owns rows [min(d0, r*c), min(d0, (r+1)*c)), c = ceil(d0/N)."""
    c = -(-d0 // world)
    return min(d0, rank * c), min(d0, (rank + 1) * c)


def row_elems(shape: Tuple[int, ...]) -> int:
    n = 1
    for s in shape[1:]:
        n *= s
    return n


def shard(full: np.ndarray, world: int, rank: int) -> np.ndarray:
    r0, r1 = fsdp_rows(full.shape[0], world, rank)
    return full[r0:r1]


def gather(shards: Sequence[np.ndarray]) -> np.ndarray:
    """All-gather of FSDP shards = concatenation along dim 0 (c1.3, 'gather')."""
    return np.concatenate(list(shards), axis=0)


# ---------------------------------------------------------------------------
# R14 — per-tensor checksum (north_star "per-tensor checksums")
# ---------------------------------------------------------------------------
def checksum(bits: np.ndarray, index_base: int = 0) -> Tuple[int, int]:
    """S1 = sum b_i, S2 = sum (i+1) b_i  (mod 2^64), i = logical flat index."""
    b = np.ascontiguousarray(bits).reshape(-1).astype(np.uint64)
    i1 = np.arange(index_base + 1, index_base + 1 + b.size, dtype=np.uint64)
    with np.errstate(over="ignore"):
        s1 = int(np.sum(b, dtype=np.uint64))
        s2 = int(np.sum(i1 * b, dtype=np.uint64))
    return s1, s2


# ---------------------------------------------------------------------------
# a2 / a3 / o4 — canonical slab layout ("indexing offloaded
# tensors by logical keys"; order/alignment: R4)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Segment:
    key: str
    tensor: int         # index in the manifest
    kind: int
    offset: int         # byte offset in the slab (256-B aligned)
    nbytes: int
    row0: int
    row1: int
    index_base: int     # logical flat index of the segment's first element


def _align(x: int, a: int = SEG_ALIGN) -> int:
    return (x + a - 1) // a * a


def slab_layout(manifest: Sequence[Tuple[str, Tuple[int, ...]]], world: int, rank: int,
                layout: int = KIND_MAJOR, kinds: Sequence[int] = ALL_KINDS,
                keys: Optional[Sequence[str]] = None) -> Tuple[List[Segment], int]:
    """Segments of one rank's slab in canonical order, and the slab size.

    KIND_MAJOR: for kind: for key.  KEY_MAJOR: for key: for kind.  Each segment
    starts at the next 256-B boundary; the slab size is the end rounded up to
    256 B; every byte not covered by a segment is zero.
    """
    keyset = None if keys is None else set(keys)
    sel = [(t, k, s) for t, (k, s) in enumerate(manifest) if keyset is None or k in keyset]
    kinds = [k for k in ALL_KINDS if k in set(kinds)]
    order = ([(kd, t, k, s) for kd in kinds for (t, k, s) in sel] if layout == KIND_MAJOR
             else [(kd, t, k, s) for (t, k, s) in sel for kd in kinds])
    segs: List[Segment] = []
    cur = 0
    for kd, t, k, s in order:
        r0, r1 = fsdp_rows(s[0], world, rank)
        re = row_elems(s)
        nb = (r1 - r0) * re * ELEM_BYTES[kd]
        off = _align(cur)
        segs.append(Segment(k, t, kd, off, nb, r0, r1, r0 * re))
        cur = off + nb
    return segs, _align(cur)


def pack_slab(segs: Sequence[Segment], size: int,
              shards: Dict[Tuple[str, int], np.ndarray]) -> np.ndarray:
    """o4: the expected slab bytes.  ``shards[(key, kind)]`` = this rank's rows."""
    slab = np.zeros(size, dtype=np.uint8)
    for sg in segs:
        b = np.ascontiguousarray(shards[(sg.key, sg.kind)]).reshape(-1).view(np.uint8)
        assert b.size == sg.nbytes, (sg, b.size)
        slab[sg.offset:sg.offset + sg.nbytes] = b
    return slab


def parse_slab(slab: np.ndarray, segs: Sequence[Segment],
               shapes: Dict[str, Tuple[int, ...]]) -> Dict[Tuple[str, int], np.ndarray]:
    """o5: inverse of pack_slab (onload(offload(S)) == S)."""
    out = {}
    for sg in segs:
        s = shapes[sg.key]
        shp = (sg.row1 - sg.row0,) + tuple(s[1:])
        raw = slab[sg.offset:sg.offset + sg.nbytes].copy()
        out[(sg.key, sg.kind)] = raw.view(ELEM_DTYPE[sg.kind]).reshape(shp)
    return out


def segment_checksums(segs: Sequence[Segment],
                      shards: Dict[Tuple[str, int], np.ndarray]) -> List[Tuple[int, int]]:
    return [checksum(shards[(sg.key, sg.kind)], sg.index_base) for sg in segs]


# ---------------------------------------------------------------------------
# NEXT-2 — canonical dedup of replicated state ("deduplicating
# replicated state"; ZeRO-2 training with DP-replicated weights, PAPER.md:587;
# reading R18: the replicated bf16 params are stored once per group, rank r
# keeping its FSDP rows, and restored by gathering every rank's rows)
# ---------------------------------------------------------------------------
def dedup_param_shards(replicas: Sequence["OrderedDict[str, np.ndarray]"], rank: int) -> "OrderedDict[str, np.ndarray]":
    """What rank `rank` stores of the replicated params: its FSDP rows (R2) of
    its replica.  Replicas must be identical -- the dedup is only defined then."""
    world = len(replicas)
    out = OrderedDict()
    for key, x in replicas[rank].items():
        for other in replicas:
            assert np.array_equal(other[key], x), f"replicas of {key} differ"
        out[key] = shard(x, world, rank)
    return out


def restore_replicas(stored: Sequence["OrderedDict[str, np.ndarray]"]) -> List["OrderedDict[str, np.ndarray]"]:
    """Inverse of dedup_param_shards: every rank gets the concatenation of all
    ranks' stored rows (an all-gather along dim 0)."""
    full = OrderedDict((key, gather([st[key] for st in stored])) for key in stored[0])
    return [OrderedDict((k, v.copy()) for k, v in full.items()) for _ in stored]


def param_arena_layout(manifest: Sequence[Tuple[str, Tuple[int, ...]]]) -> Tuple[List[int], int]:
    """Byte offset of every manifest tensor's full bf16 replica in a rank's param
    arena (manifest order, each at the next 256-B boundary, R4's alignment) and
    the arena size."""
    offs, cur = [], 0
    for _, s in manifest:
        off = _align(cur)
        offs.append(off)
        cur = off + int(np.prod(s)) * ELEM_BYTES[KIND_PARAM]
    return offs, _align(cur)


# ---------------------------------------------------------------------------
# NEXT-3 — checkpoint materialisation from offloaded state (PAPER.md:510
# "checkpointing ... materialization", :513 background checkpoint
# materialization; format reading R19: one safetensors tensor per slab segment)
# ---------------------------------------------------------------------------
CKPT_KIND = {KIND_PARAM: "param", KIND_MASTER: "master", KIND_EXP_AVG: "exp_avg", KIND_EXP_AVG_SQ: "exp_avg_sq"}


def checkpoint_name(key: str, kind: int) -> str:
    return key if kind == KIND_PARAM else f"optimizer.{CKPT_KIND[kind]}.{key}"


def checkpoint_tensors(segs: Sequence[Segment],
                       shards: Dict[Tuple[str, int], np.ndarray]) -> "OrderedDict[str, np.ndarray]":
    """The tensors a rank's checkpoint holds, in slab order: each segment's shard
    (this rank's FSDP rows, R2) under its checkpoint name."""
    return OrderedDict((checkpoint_name(sg.key, sg.kind), shards[(sg.key, sg.kind)]) for sg in segs)


def checkpoint_metadata(world: int, rank: int, cks: Sequence[Tuple[int, int]]) -> Dict[str, str]:
    return {"format": "pt", "plex.layout": "fsdp-dim0", "plex.world": str(world), "plex.rank": str(rank),
            "plex.checksums": ",".join(f"{v:016x}" for pair in cks for v in pair)}


# ---------------------------------------------------------------------------
# o7 — rollout layout ("each rollout rank fetches only the tensor
# slices required by its target parallel layout"; layout: R3)
# ---------------------------------------------------------------------------
def rank_coords(g: int, tp: int, dp: int, rank_map: int = TP_FAST) -> Tuple[int, int]:
    """R10: default g = dp*TP + tp.  Returns (tp_rank, dp_rank)."""
    if rank_map == TP_FAST:
        return g % tp, g // tp
    return g // dp, g % dp


def _split_rows(x: np.ndarray, parts: int, i: int) -> np.ndarray:
    n = x.shape[0] // parts
    return x[i * n:(i + 1) * n]


def _split_cols(x: np.ndarray, parts: int, i: int) -> np.ndarray:
    n = x.shape[1] // parts
    return x[:, i * n:(i + 1) * n]


class LayoutError(ValueError):
    """Shape not divisible by the destination layout (E_LAYOUT)."""


def rollout_tensors(full_bf16: "OrderedDict[str, np.ndarray]", tp: int, dp: int, ep: int,
                    g: int, rank_map: int = TP_FAST,
                    head_dim: Optional[int] = None) -> "OrderedDict[str, np.ndarray]":
    """Rank g's rollout tensors from the full cast tensors (c1.3: slice_g, fuse_g).

    R3 (Megatron/vLLM convention): column-parallel q/k/v (+bias) fused per rank
    as qkv = cat(q_tp, k_tp, v_tp); gate/up fused as gate_up = cat(gate_tp,
    up_tp); row-parallel o_proj/down_proj (dim-1 split); vocab-parallel
    embed/lm_head (dim-0 split); norms and the MoE router replicated; experts
    EP-contiguous: expert e on EP rank floor(e / (E/EP)), EP rank = g % EP,
    w13 = stack_e cat(gate_e, up_e) [E/EP, 2I, H], w2 = stack_e down_e.
    With ``head_dim`` given, q/k/v must split at head granularity
    (heads % TP == 0; kv-head replication is not supported -> LayoutError).
    """
    t, _ = rank_coords(g, tp, dp, rank_map)
    epr = g % ep
    out: "OrderedDict[str, np.ndarray]" = OrderedDict()

    def need(x: np.ndarray, parts: int, what: str) -> None:
        if x.shape[0 if what == "rows" else 1] % parts:
            raise LayoutError(what)

    keys = list(full_bf16.keys())
    done = set()
    for k in keys:
        if k in done:
            continue
        x = full_bf16[k]
        if k.endswith("embed_tokens.weight") or k == "lm_head.weight":
            need(x, tp, "rows")
            out[k] = _split_rows(x, tp, t)
        elif ".self_attn.q_proj." in k:
            suf = k.rsplit(".", 1)[1]                       # weight | bias
            pre = k.split(".self_attn.")[0] + ".self_attn."
            q, kk, v = (full_bf16[pre + n + "_proj." + suf] for n in ("q", "k", "v"))
            for y in (q, kk, v):
                need(y, tp * (head_dim or 1), "rows")
            out[pre + "qkv_proj." + suf] = np.concatenate(
                [_split_rows(q, tp, t), _split_rows(kk, tp, t), _split_rows(v, tp, t)], axis=0)
            done.update(pre + n + "_proj." + suf for n in ("q", "k", "v"))
        elif ".self_attn.o_proj." in k:
            need(x, tp, "cols")
            out[k] = _split_cols(x, tp, t)
        elif ".mlp.gate_proj." in k and ".experts." not in k:
            pre = k.split(".mlp.")[0] + ".mlp."
            gt, up = full_bf16[pre + "gate_proj.weight"], full_bf16[pre + "up_proj.weight"]
            need(gt, tp, "rows")
            need(up, tp, "rows")
            out[pre + "gate_up_proj.weight"] = np.concatenate(
                [_split_rows(gt, tp, t), _split_rows(up, tp, t)], axis=0)
            done.update([pre + "gate_proj.weight", pre + "up_proj.weight"])
        elif ".mlp.down_proj." in k and ".experts." not in k:
            need(x, tp, "cols")
            out[k] = _split_cols(x, tp, t)
        elif ".mlp.experts." in k:
            pre = k.split(".mlp.experts.")[0] + ".mlp.experts."
            E = 0
            while (pre + f"{E}.gate_proj.weight") in full_bf16:
                E += 1
            if E % ep:
                raise LayoutError("experts")
            per = E // ep
            mine = range(epr * per, (epr + 1) * per)
            out[pre + "w13_weight"] = np.stack([
                np.concatenate([full_bf16[pre + f"{e}.gate_proj.weight"],
                                full_bf16[pre + f"{e}.up_proj.weight"]], axis=0) for e in mine])
            out[pre + "w2_weight"] = np.stack([full_bf16[pre + f"{e}.down_proj.weight"] for e in mine])
            for e in range(E):
                done.update(pre + f"{e}.{n}_proj.weight" for n in ("gate", "up", "down"))
        else:
            # norms (input/post-attention/final, q_norm, k_norm) and router
            out[k] = x
    return out


def weight_sync(master_shards: Dict[str, Sequence[np.ndarray]], tp: int, dp: int, ep: int,
                rank_map: int = TP_FAST,
                head_dim: Optional[int] = None) -> List["OrderedDict[str, np.ndarray]"]:
    """c1.3: sync(master)[g][t] = fuse_g(slice_g(RNE(concat_r shard_r(master_t)))).

    ``master_shards[key]`` = the W FSDP shards (uint32 bits), in manifest order.
    Returns the rollout tensors of every destination rank g < TP*DP.
    """
    full = OrderedDict((k, rne_bf16(gather(v))) for k, v in master_shards.items())
    return [rollout_tensors(full, tp, dp, ep, g, rank_map, head_dim) for g in range(tp * dp)]


def inverse_sync(rollout: List["OrderedDict[str, np.ndarray]"],
                 manifest: Sequence[Tuple[str, Tuple[int, ...]]], tp: int, dp: int, ep: int,
                 rank_map: int = TP_FAST) -> "OrderedDict[str, np.ndarray]":
    """o8: un-fuse, concatenate TP slices along the split dim, un-stack experts.

    Asserts every DP replica (and every EP replica group) holds identical bytes.
    Returns the full bf16 tensors by manifest key.
    """
    shapes = OrderedDict(manifest)
    n_experts = _experts_per_layer(manifest)
    W = tp * dp
    by_tp: Dict[int, List[int]] = {}
    for g in range(W):
        t, _ = rank_coords(g, tp, dp, rank_map)
        by_tp.setdefault(t, []).append(g)
    # DP replicas of the same tp rank must agree on all non-expert tensors.
    for t, gs in by_tp.items():
        for g in gs[1:]:
            for name, x in rollout[gs[0]].items():
                if ".mlp.experts." in name:
                    continue
                assert np.array_equal(x, rollout[g][name]), ("dp replica mismatch", name, g)
    out: "OrderedDict[str, np.ndarray]" = OrderedDict()
    for k, s in shapes.items():
        if k.endswith("embed_tokens.weight") or k == "lm_head.weight":
            out[k] = np.concatenate([rollout[by_tp[t][0]][k] for t in range(tp)], axis=0)
        elif ".self_attn." in k and any(f".{n}_proj." in k for n in "qkv"):
            pre, rest = k.split(".self_attn.")
            n, suf = rest.split("_proj.")
            fused_name = pre + ".self_attn.qkv_proj." + suf
            sizes = [shapes[pre + f".self_attn.{m}_proj.{suf}"][0] // tp for m in "qkv"]
            j = "qkv".index(n)
            lo = sum(sizes[:j])
            out[k] = np.concatenate([rollout[by_tp[t][0]][fused_name][lo:lo + sizes[j]]
                                     for t in range(tp)], axis=0)
        elif ".self_attn.o_proj." in k or (".mlp.down_proj." in k and ".experts." not in k):
            out[k] = np.concatenate([rollout[by_tp[t][0]][k] for t in range(tp)], axis=1)
        elif (".mlp.gate_proj." in k or ".mlp.up_proj." in k) and ".experts." not in k:
            pre = k.split(".mlp.")[0] + ".mlp."
            half = shapes[pre + "gate_proj.weight"][0] // tp
            j = 0 if ".gate_proj." in k else 1
            out[k] = np.concatenate([rollout[by_tp[t][0]][pre + "gate_up_proj.weight"][j * half:(j + 1) * half]
                                     for t in range(tp)], axis=0)
        elif ".mlp.experts." in k:
            pre, rest = k.split(".mlp.experts.")
            e, nm = rest.split(".", 1)
            e = int(e)
            E = n_experts[pre]
            per = E // ep
            epr, j = e // per, e % per
            owners = [g for g in range(W) if g % ep == epr]
            I = shapes[pre + f".mlp.experts.{e}.gate_proj.weight"][0]
            vals = []
            for g in owners:
                if nm.startswith("gate"):
                    vals.append(rollout[g][pre + ".mlp.experts.w13_weight"][j][:I])
                elif nm.startswith("up"):
                    vals.append(rollout[g][pre + ".mlp.experts.w13_weight"][j][I:])
                else:
                    vals.append(rollout[g][pre + ".mlp.experts.w2_weight"][j])
            for v in vals[1:]:
                assert np.array_equal(vals[0], v), ("ep replica mismatch", k)
            out[k] = vals[0]
        else:
            out[k] = rollout[0][k]
            for g in range(1, W):
                assert np.array_equal(out[k], rollout[g][k]), ("replicated mismatch", k, g)
    return out


# ---------------------------------------------------------------------------
# o9 — zero-redundancy ledger ("without redundant transfer")
# ---------------------------------------------------------------------------
def _experts_per_layer(manifest: Sequence[Tuple[str, Tuple[int, ...]]]) -> Dict[str, int]:
    n: Dict[str, int] = {}
    for k, _ in manifest:
        if ".mlp.experts." in k and k.endswith("gate_proj.weight"):
            pre = k.split(".mlp.experts.")[0]
            n[pre] = n.get(pre, 0) + 1
    return n


def needed_rows(manifest: Sequence[Tuple[str, Tuple[int, ...]]], tp: int, dp: int, ep: int,
                g: int, rank_map: int = TP_FAST) -> Dict[str, Tuple[int, int, int, int]]:
    """Rectangle (r0, r1, c0, c1) of each source tensor that rank g needs (R3),
    in units of rows/cols of the 2-D view [d0, prod(shape[1:])]."""
    t, _ = rank_coords(g, tp, dp, rank_map)
    epr = g % ep
    need: Dict[str, Tuple[int, int, int, int]] = {}
    n_experts = _experts_per_layer(manifest)
    for k, s in manifest:
        d0, d1 = s[0], row_elems(s)
        if (k.endswith("embed_tokens.weight") or k == "lm_head.weight"
                or ".self_attn.q_proj." in k or ".self_attn.k_proj." in k or ".self_attn.v_proj." in k
                or ((".mlp.gate_proj." in k or ".mlp.up_proj." in k) and ".experts." not in k)):
            n = d0 // tp
            need[k] = (t * n, (t + 1) * n, 0, d1)
        elif ".self_attn.o_proj." in k or (".mlp.down_proj." in k and ".experts." not in k):
            n = d1 // tp
            need[k] = (0, d0, t * n, (t + 1) * n)
        elif ".mlp.experts." in k:
            pre, rest = k.split(".mlp.experts.")
            e = int(rest.split(".", 1)[0])
            E = n_experts[pre]
            if e // (E // ep) == epr:
                need[k] = (0, d0, 0, d1)
        else:
            need[k] = (0, d0, 0, d1)
    return need


def ledger(manifest: Sequence[Tuple[str, Tuple[int, ...]]], world: int, tp: int, dp: int,
           ep: int, rank_map: int = TP_FAST) -> np.ndarray:
    """bytes[src r, dst g] of bf16 that FSDP-``world`` rank r must send to rollout
    rank g (diagonal = bytes g already holds locally).  Each needed element is
    owned by exactly one source rank, so nothing is sent twice."""
    W = tp * dp
    assert W == world, "source and destination share one GPU group"
    L = np.zeros((world, W), dtype=np.int64)
    shapes = dict(manifest)
    for g in range(W):
        for k, (r0, r1, c0, c1) in needed_rows(manifest, tp, dp, ep, g, rank_map).items():
            d0 = shapes[k][0]
            for r in range(world):
                a, b = fsdp_rows(d0, world, r)
                rows = max(0, min(b, r1) - max(a, r0))
                L[r, g] += rows * (c1 - c0) * 2
    return L


# ---------------------------------------------------------------------------
# a1 — transition decision (PAPER.md:555 _handle_job_transition)
# ---------------------------------------------------------------------------
OP_OFFLOAD, OP_ONLOAD, OP_SYNC = 1, 2, 3


def transition_ops(resident: Optional[int], incoming: int, with_sync: bool = False) -> List[Tuple[int, int]]:
    """If the incoming op's job differs from the resident one, prepend offload
    (resident) and load (incoming).  A->A = [], None->B = [load B]."""
    ops: List[Tuple[int, int]] = []
    if resident != incoming:
        if resident is not None:
            ops.append((OP_OFFLOAD, resident))
        ops.append((OP_ONLOAD, incoming))
    if with_sync:
        ops.append((OP_SYNC, incoming))
    return ops


# ---------------------------------------------------------------------------
# o10 — multiplex replay (PAPER.md:555 automatic context switching; R17 one
# resident job per GPU group; BASELINE.json configs[4])
# ---------------------------------------------------------------------------
def multiplex_replay(jobs: Sequence[dict], schedule: Sequence[int], world: int,
                     mutate, layout: int = KIND_MAJOR) -> Tuple[list, list]:
    """Replay visits: for each visit to job j, run transition_ops(resident, j)
    through per-rank slabs (offload = pack_slab, onload = parse_slab), then one
    simulated training step (``mutate(job, step, key, kind, bits, index_base)``
    returns the new shard bits) and a weight sync of j.

    ``jobs[j]`` = {"manifest", "shards": [per-rank {(key, kind): bits}], "tp",
    "dp", "ep"}; ``shards`` is the job's initial state, which starts in its
    slabs (every job begins HOST-resident, none on the GPU group).
    Returns (per-visit [(ops, rollout)], final per-job per-rank shards).
    """
    shapes = [dict(j["manifest"]) for j in jobs]
    layouts = [[slab_layout(j["manifest"], world, r, layout) for r in range(world)] for j in jobs]
    slabs = [[pack_slab(*layouts[i][r], jobs[i]["shards"][r]) for r in range(world)]
             for i in range(len(jobs))]
    device: Optional[list] = None
    resident: Optional[int] = None
    steps = [0] * len(jobs)
    visits = []
    for j in schedule:
        ops = transition_ops(resident, j)
        for op, job in ops:
            if op == OP_OFFLOAD:
                slabs[job] = [pack_slab(*layouts[job][r], device[r]) for r in range(world)]
                device = None
            elif op == OP_ONLOAD:
                device = [parse_slab(slabs[job][r], layouts[job][r][0], shapes[job]) for r in range(world)]
        resident = j
        for r in range(world):
            for (key, kind), bits in list(device[r].items()):
                r0 = fsdp_rows(shapes[j][key][0], world, r)[0]
                device[r][(key, kind)] = mutate(j, steps[j], key, kind, bits, r0 * row_elems(shapes[j][key]))
        steps[j] += 1
        ms = OrderedDict((k, [device[r][(k, KIND_MASTER)] for r in range(world)]) for k, _ in jobs[j]["manifest"])
        visits.append((ops, weight_sync(ms, jobs[j]["tp"], jobs[j]["dp"], jobs[j]["ep"])))
    final = []
    for i in range(len(jobs)):
        if i == resident:
            final.append(device)
        else:
            final.append([parse_slab(slabs[i][r], layouts[i][r][0], shapes[i]) for r in range(world)])
    return visits, final


# ---------------------------------------------------------------------------
# NEXT-4 — HRRS runtime ordering (Alg. 1; Eq. 3-4, :468-480)
# ---------------------------------------------------------------------------
@dataclass
class Request:
    job: int
    arrival: float
    exec_time: float            # E_i
    remaining: float = 0.0      # for the running request


def hrrs_score(req: Request, t_now: float, running: Optional[Request], t_load: float, t_offload: float) -> float:
    """Eq. 3: S_i = E_i + 1_switch(i, curr) (T_offload + T_load); Eq. 4:
    P_i = (W_i + S_i) / S_i.  The running request uses its remaining time
    (Alg. 1 line 4).  1_switch = 1 iff the request's job differs from the
    running request's job (reading H1: Alg. 1 line 7 charges every
    non-running request; Eq. 3 only switching ones -- we follow Eq. 3)."""
    t_wait = t_now - req.arrival
    if running is not None and req is running:
        t_req = req.remaining
    else:
        switch = running is None or req.job != running.job
        t_req = req.exec_time + (t_load + t_offload if switch else 0.0)
    return (t_wait + t_req) / t_req


def hrrs_schedule(t_now: float, new: Request, running: Optional[Request], scheduled: Sequence[Request],
                  t_load: float, t_offload: float) -> List[Tuple[Request, float, float]]:
    """Alg. 1: score Omega = {new} + {running} + scheduled, sort by score
    descending (stable), then lay the timeline out from t_now, inserting a
    setup gap of T_offload + T_load before a request whose job differs from
    the job resident at that point (reading H2: Alg. 1 lines 12-14 insert it
    once, before the first non-running request; Eq. 3's indicator and
    PAPER.md:555 imply one per job change).  Returns [(request, start, end)]."""
    omega = [new] + ([running] if running is not None else []) + list(scheduled)
    scores = [hrrs_score(r, t_now, running, t_load, t_offload) for r in omega]
    order = sorted(range(len(omega)), key=lambda i: -scores[i])
    t_cursor = t_now
    resident = running.job if running is not None else None
    out = []
    for i in order:
        r = omega[i]
        if r.job != resident:
            t_cursor += t_offload + t_load if resident is not None else t_load
            resident = r.job
        t_req = r.remaining if (running is not None and r is running) else r.exec_time
        out.append((r, t_cursor, t_cursor + t_req))
        t_cursor += t_req
    return out
