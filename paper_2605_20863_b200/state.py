"""Python API of the B200 state-transition path (thin: marshalling only).

    mgr  = StateManager(device=0)                    # one per rank process
    plan = mgr.plan(manifest, head_dim=128, tp=2, dp=4)
    job  = Job(mgr, plan, seed=1).alloc().init_synthetic()
    job.suspend(); job.resume(); job.sync(arena)

Everything that touches a byte of state runs in libplex.so (CUDA kernels,
copy engines, NCCL); this module only builds argument arrays, owns PyTorch
device memory and streams, and bootstraps the NCCL id over torch.distributed.
"""
from __future__ import annotations

import ctypes as C
import re
from collections import OrderedDict
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib as L
from ._lib import PlexError, check, lib, ptr_array

KIND_TORCH = {0: torch.bfloat16, 1: torch.float32, 2: torch.float32, 3: torch.float32}

_LAYER = re.compile(r"^(model\.layers\.\d+\.)")


class Plan:
    """Immutable transition plan (plex_transition_plan)."""

    def __init__(self, manifest, head_dim: int = 1, world: int = 1, tp: int = 0, dp: int = 0, ep: int = 1,
                 rank_map: int = L.RANKMAP_TP_FAST, slab_layout: int = L.SLAB_KIND_MAJOR,
                 kind_mask: int = L.KINDMASK_ALL, subset: Optional[Sequence[str]] = None,
                 bucket_bytes: int = 2 << 30, tile_bytes: int = 64 << 10,
                 resident_job: int = -1, incoming_job: int = -1, op: int = L.OP_NONE, elide_param: bool = False,
                 link_weights: Optional[Sequence[float]] = None, replica_param: bool = False):
        self.manifest = list(manifest)
        self.index = {k: i for i, (k, _) in enumerate(self.manifest)}
        # keys and shapes only: the library derives every tensor's rollout role,
        # fusion group and split unit from its key (PLEX_ROLE_AUTO, reading R3)
        self._keys = [k.encode() for k, _ in self.manifest]
        arr = (L.TensorDesc * len(self.manifest))()
        for i, (key, shape) in enumerate(self.manifest):
            d1 = int(np.prod(shape[1:])) if len(shape) > 1 else 1
            arr[i] = L.TensorDesc(self._keys[i], int(shape[0]), d1, len(shape), L.ROLE_AUTO, 0, 0, -1, 1)
        self._arr = arr
        sub = None
        n_sub = 0
        if subset is not None:
            idx = [self.index[k] for k in subset]
            sub = (C.c_int32 * max(1, len(idx)))(*idx)
            n_sub = len(idx)
        self._sub = sub
        self._lw = None
        if link_weights is not None:
            self._lw = (C.c_float * world)(*[float(x) for x in link_weights])
        req = L.PlanReq(len(self.manifest), arr, world, tp, dp, ep, rank_map, slab_layout, kind_mask, n_sub, sub,
                        bucket_bytes, tile_bytes, resident_job, incoming_job, op,
                        (L.PLAN_ELIDE_PARAM if elide_param else 0) | (L.PLAN_REPLICA_PARAM if replica_param else 0),
                        self._lw, head_dim)
        h = C.c_void_p()
        check(lib.plex_transition_plan(C.byref(req), C.byref(h)))
        self.h = h
        self.world, self.tp, self.dp, self.ep = world, tp, dp, ep
        self.kind_mask = kind_mask
        self.bucket_bytes = bucket_bytes
        self.subset = None if subset is None else frozenset(subset)
        self.replica_param = replica_param

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value and lib is not None:
            lib.plex_plan_destroy(h)
            self.h = None

    # ---- queries ----------------------------------------------------------
    def stats(self) -> L.PlanStats:
        s = L.PlanStats()
        check(lib.plex_plan_query(self.h, C.byref(s)))
        return s

    def ops(self) -> List[Tuple[int, int]]:
        s = self.stats()
        return [(s.ops[i], s.op_jobs[i]) for i in range(s.n_ops)]

    def rank_info(self, rank: int) -> L.RankInfo:
        r = L.RankInfo()
        check(lib.plex_plan_rank_info(self.h, rank, C.byref(r)))
        return r

    def segments(self, rank: int) -> List[L.SegDesc]:
        n = self.rank_info(rank).n_segments
        out = []
        for i in range(n):
            s = L.SegDesc()
            check(lib.plex_plan_segment(self.h, rank, i, C.byref(s)))
            out.append(s)
        return out

    def shard_rows(self, rank: int, t: int) -> Tuple[int, int]:
        a, b = C.c_int64(), C.c_int64()
        check(lib.plex_plan_shard_rows(self.h, rank, t, C.byref(a), C.byref(b)))
        return a.value, b.value

    def shard_shape(self, rank: int, t: int) -> Tuple[int, ...]:
        a, b = self.shard_rows(rank, t)
        shape = self.manifest[t][1]
        return (b - a,) + tuple(shape[1:])

    def shard_numels(self, rank: int) -> List[int]:
        """numel of every tensor's FSDP shard on `rank` (cached)."""
        cache = self.__dict__.setdefault("_numels", {})
        if rank not in cache:
            cache[rank] = [int(np.prod(self.shard_shape(rank, t))) for t in range(len(self.manifest))]
        return cache[rank]

    def group(self, g: int) -> Tuple[str, int, int]:
        """(rollout tensor name, role, experts stacked) of destination group g,
        as the library's planner classified it (plex_plan_group)."""
        cache = self.__dict__.setdefault("_groups", {})
        if g not in cache:
            buf = C.create_string_buffer(512)
            n, role, ne = C.c_int32(), C.c_int32(), C.c_int32()
            check(lib.plex_plan_group(self.h, g, buf, 512, C.byref(n), C.byref(role), C.byref(ne)))
            if n.value >= 512:
                buf = C.create_string_buffer(n.value + 1)
                check(lib.plex_plan_group(self.h, g, buf, n.value + 1, None, None, None))
            cache[g] = (buf.value.decode(), role.value, ne.value)
        return cache[g]

    def dst_tensors(self, rank: int) -> List[Tuple[str, int, Tuple[int, ...]]]:
        """(rollout name, arena byte offset, shape) of rank's destination tensors."""
        n = self.rank_info(rank).n_dst_tensors
        out = []
        for i in range(n):
            d = L.DstDesc()
            check(lib.plex_plan_dst_tensor(self.h, rank, i, C.byref(d)))
            name, role, n_exp = self.group(d.group)
            shape: Tuple[int, ...] = (d.rows, d.cols)
            if role == L.ROLE_EXPERT:
                per = n_exp // self.ep
                shape = (per, d.rows // per, d.cols)
            elif len(self.manifest[d.first_tensor][1]) == 1:
                shape = (d.rows,)
            out.append((name, d.arena_offset, shape))
        return out

    def carry(self) -> List[L.CarryDesc]:
        """Carried buckets (NEXT-1 host-link balancing), in the plan's global order."""
        n = C.c_int32()
        check(lib.plex_plan_n_carry(self.h, C.byref(n)))
        out = []
        for i in range(n.value):
            d = L.CarryDesc()
            check(lib.plex_plan_carry(self.h, i, C.byref(d)))
            out.append(d)
        return out

    # ---- NEXT-2 replicated params (ZeRO-2) ------------------------------------------
    @property
    def param_arena_bytes(self) -> int:
        n = C.c_uint64()
        check(lib.plex_plan_param_arena(self.h, -1, None, C.byref(n)))
        return n.value

    def param_offsets(self) -> List[int]:
        cache = self.__dict__.setdefault("_param_off", [])
        if not cache:
            for t in range(len(self.manifest)):
                o = C.c_uint64()
                check(lib.plex_plan_param_arena(self.h, t, C.byref(o), None))
                cache.append(o.value)
        return cache

    def param_views(self, arena: torch.Tensor) -> "OrderedDict[str, torch.Tensor]":
        """Full replicated bf16 param of every manifest tensor, viewed in a param arena."""
        out = OrderedDict()
        for (key, shape), off in zip(self.manifest, self.param_offsets()):
            n = int(np.prod(shape))
            out[key] = arena[off:off + 2 * n].view(torch.bfloat16).view(shape)
        return out

    def ledger(self) -> np.ndarray:
        n = self.world * self.world
        buf = (C.c_uint64 * n)()
        check(lib.plex_plan_ledger(self.h, buf, n))
        return np.frombuffer(buf, dtype=np.uint64).reshape(self.world, self.world).astype(np.int64).copy()


class Slab:
    """Pinned host slab of one rank's state under a plan (plex_slab_create)."""

    def __init__(self, plan: Plan, rank: int, hugepage: bool = False):
        h = C.c_void_p()
        check(lib.plex_slab_create(plan.h, rank, L.SLAB_HUGEPAGE if hugepage else 0, C.byref(h)))
        self.h = h
        self.plan = plan
        self.rank = rank

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value and lib is not None:
            lib.plex_slab_destroy(h)
            self.h = None

    def info(self) -> Tuple[int, int, int]:
        p, n, r = C.c_void_p(), C.c_uint64(), C.c_int32()
        check(lib.plex_slab_info(self.h, C.byref(p), C.byref(n), C.byref(r)))
        return p.value or 0, n.value, r.value

    @property
    def residency(self) -> int:
        return self.info()[2]

    @property
    def elided(self) -> bool:
        """The last offload derived (did not store) the leading PARAM buckets (NEXT-2)."""
        v = C.c_int32()
        check(lib.plex_slab_elided(self.h, C.byref(v)))
        return bool(v.value)

    def host_bytes(self) -> np.ndarray:
        """Writable NumPy view of the pinned slab bytes."""
        p, n, _ = self.info()
        if n == 0 or not p:                      # empty, or spilled to the NVMe tier
            return np.zeros(0, dtype=np.uint8)
        return np.ctypeslib.as_array((C.c_uint8 * n).from_address(p))

    def spill(self, path: str, threads: int = 8) -> None:
        """NEXT-4: move the slab to the NVMe tier (O_DIRECT) and unpin it."""
        check(lib.plex_slab_spill(self.h, path.encode(), threads))

    def fill(self, path: str, threads: int = 8) -> None:
        """NEXT-4: bring a spilled slab back into pinned host memory."""
        check(lib.plex_slab_fill(self.h, path.encode(), threads))

    def checkpoint(self, path: str, threads: int = 8, background: bool = False):
        """NEXT-3: materialise the offloaded state as a safetensors checkpoint
        (PAPER.md:510, :513).  background=True starts the host-only write on a
        library-owned thread (plex_slab_checkpoint_start: the slab is marked
        read-only before this returns) and returns a handle; ``handle.join()``
        waits for it and fills ``handle.errors``."""
        if not background:
            check(lib.plex_slab_checkpoint(self.plan.h, self.h, path.encode(), threads))
            return None
        h = C.c_void_p()
        check(lib.plex_slab_checkpoint_start(self.plan.h, self.h, path.encode(), threads, C.byref(h)))
        return CheckpointHandle(h, self)

    def restore(self, path: str, threads: int = 8) -> None:
        """Fill this slab from a checkpoint of the same plan/rank (residency HOST)."""
        check(lib.plex_slab_restore(self.plan.h, self.h, path.encode(), threads))

    def carry_bytes(self) -> np.ndarray:
        """Pinned carry region (other ranks' carried buckets) as a NumPy view."""
        p, n = C.c_void_p(), C.c_uint64()
        check(lib.plex_slab_carry(self.h, C.byref(p), C.byref(n)))
        if not p.value or not n.value:
            return np.zeros(0, dtype=np.uint8)
        return np.ctypeslib.as_array((C.c_uint8 * n.value).from_address(p.value))

    def checksums(self) -> np.ndarray:
        n = 2 * self.plan.rank_info(self.rank).n_segments
        buf = (C.c_uint64 * max(1, n))()
        check(lib.plex_slab_checksums(self.h, buf, n))
        return np.frombuffer(buf, dtype=np.uint64)[:n].reshape(-1, 2).copy()


class CheckpointHandle:
    """A background checkpoint (plex_slab_checkpoint_start); join() = plex_ckpt_wait."""

    def __init__(self, h: C.c_void_p, slab: "Slab"):
        self.h, self.slab, self.errors = h, slab, []

    def join(self) -> None:
        if self.h is not None and self.h.value:
            code = lib.plex_ckpt_wait(self.h)
            self.h = None
            if code != L.OK:
                self.errors.append(PlexError(code, lib.plex_last_error().decode(errors="replace")))

    def __del__(self):
        self.join()


def bootstrap_nccl_id(rank: int) -> bytes:
    """Rank 0 draws the library communicator's 128-byte NCCL id; every rank
    receives it over the default torch.distributed group (any backend)."""
    import torch.distributed as dist
    buf = C.create_string_buffer(128)
    if rank == 0:
        check(lib.plex_nccl_unique_id(buf))
    obj = [bytes(buf.raw) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def plan_digest(plan: "Plan", rank: int) -> str:
    """Hash of everything rank-specific a plan holds (slab segments, rollout
    tensors, ledger): identical requests must give identical plans on every rank."""
    import hashlib
    h = hashlib.sha256()
    for sg in plan.segments(rank):
        h.update(bytes(sg))
    for name, off, shape in plan.dst_tensors(rank):
        h.update(f"{name}:{off}:{shape}".encode())
    h.update(plan.ledger().tobytes())
    return h.hexdigest()


def _stream_ptr(s) -> int:
    if s is None:
        return torch.cuda.current_stream().cuda_stream
    return s.cuda_stream


class StateManager:
    """One per rank process: the ctx (streams, staging, NCCL communicator)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, bucket_bytes: int = 2 << 30,
                 n_slots: int = 2, timing: bool = False, sync_nccl: bool = False, bootstrap: bool = True,
                 nccl_id: Optional[bytes] = None, duplex: bool = True, carry_nccl: bool = False,
                 workspace_bytes: int = 256 << 20):
        if not torch.cuda.is_available():
            raise RuntimeError("StateManager needs a CUDA device (no CPU fallback)")
        self.device = device
        torch.cuda.set_device(device)
        self.rank, self.world = rank, world
        self.bucket_bytes = bucket_bytes
        self.n_slots = n_slots
        self.pack_stream = torch.cuda.Stream(device)
        self.copy_stream = torch.cuda.Stream(device)
        # duplex: room for both rings of a switch (offload || onload)
        self.staging = torch.empty((2 if duplex else 1) * n_slots * bucket_bytes, dtype=torch.uint8,
                                   device=f"cuda:{device}")
        idbuf = None
        if world > 1 and bootstrap:
            if nccl_id is None:
                nccl_id = self._bootstrap_id()
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        flags = ((L.CTX_TIMING if timing else 0) | (L.CTX_SYNC_NCCL if sync_nccl else 0)
                 | (L.CTX_CARRY_NCCL if carry_nccl else 0))
        h = C.c_void_p()
        # the library's device metadata tables live here (it never calls cudaMalloc)
        self.workspace = torch.empty(workspace_bytes, dtype=torch.uint8, device=f"cuda:{device}")
        check(lib.plex_ctx_create(device, self.staging.data_ptr(), self.staging.numel(), self.workspace.data_ptr(),
                                  self.workspace.numel(), n_slots,
                                  self.pack_stream.cuda_stream, self.copy_stream.cuda_stream,
                                  idbuf, rank, world, flags, C.byref(h)))
        self.h = h

    def _bootstrap_id(self) -> bytes:
        return bootstrap_nccl_id(self.rank)

    def close(self):
        h = getattr(self, "h", None)
        if h is not None and h.value and lib is not None:
            lib.plex_ctx_destroy(h)
            self.h = None

    def __del__(self):
        self.close()

    # ---- plans / slabs --------------------------------------------------------
    def plan(self, manifest, **kw) -> Plan:
        kw.setdefault("world", self.world)
        kw.setdefault("bucket_bytes", self.bucket_bytes)
        return Plan(manifest, **kw)

    def slab(self, plan: Plan, rank: Optional[int] = None, hugepage: bool = False) -> Slab:
        return Slab(plan, self.rank if rank is None else rank, hugepage)

    # ---- the four hot-path calls --------------------------------------------------
    @staticmethod
    def _state_ptrs(plan: Plan, shards: Dict[Tuple[str, int], torch.Tensor], rank: int):
        """Pointer table [kind * n_tensors + t]; every shard is checked against the
        plan (device, contiguity, dtype width, FSDP shard numel) before the
        library touches it, so a mis-sized tensor never reaches a kernel."""
        nt = len(plan.manifest)
        ptrs = [0] * (L.NUM_KINDS * nt)
        numels = plan.shard_numels(rank)
        for (key, kind), t in shards.items():
            ti = plan.index[key]
            if not t.is_cuda:
                raise ValueError(f"shard {key}/{kind} must be a CUDA tensor")
            if not t.is_contiguous():
                raise ValueError(f"shard {key}/{kind} must be contiguous")
            if t.element_size() != (2 if kind == L.KIND_PARAM else 4):
                raise ValueError(f"shard {key}/{kind}: element size {t.element_size()} does not match the kind")
            want = numels[ti]
            if kind == L.KIND_PARAM and plan.replica_param:    # the full replicated tensor
                want = int(np.prod(plan.manifest[ti][1]))
            if t.numel() != want:
                raise ValueError(f"shard {key}/{kind}: {t.numel()} elements, plan expects {want} on rank {rank}")
            ptrs[kind * nt + ti] = t.data_ptr() if t.numel() else 0
        return ptr_array(ptrs), len(ptrs)

    def offload(self, plan: Plan, shards, slab: Slab, stream=None) -> None:
        arr, n = self._state_ptrs(plan, shards, slab.rank)
        check(lib.plex_state_offload(self.h, plan.h, arr, n, slab.h, _stream_ptr(stream)))

    def onload(self, plan: Plan, slab: Slab, shards, stream=None) -> None:
        arr, n = self._state_ptrs(plan, shards, slab.rank)
        check(lib.plex_state_onload(self.h, plan.h, slab.h, arr, n, _stream_ptr(stream)))

    def switch(self, plan_out: Plan, shards_out, slab_out: Slab, plan_in: Plan, slab_in: Slab, shards_in,
               stream=None) -> None:
        """Duplex context switch: offload one job while onloading another (NEXT-1)."""
        a, na = self._state_ptrs(plan_out, shards_out, slab_out.rank)
        b, nb = self._state_ptrs(plan_in, shards_in, slab_in.rank)
        check(lib.plex_state_switch(self.h, plan_out.h, a, na, slab_out.h, plan_in.h, slab_in.h, b, nb,
                                    _stream_ptr(stream)))

    def swap(self, plan: Plan, shards, slab: Slab, stream=None) -> None:
        """In-place context switch of two same-layout jobs: the resident state in
        `shards` goes to `slab` while the slab's state comes into `shards`."""
        arr, n = self._state_ptrs(plan, shards, slab.rank)
        check(lib.plex_state_swap(self.h, plan.h, arr, n, slab.h, _stream_ptr(stream)))

    @staticmethod
    def _check_masters(plan: Plan, masters: Sequence[torch.Tensor], rank: int) -> None:
        if len(masters) != len(plan.manifest):
            raise ValueError(f"{len(masters)} master shards, plan has {len(plan.manifest)} tensors")
        numels = plan.shard_numels(rank)
        for t, m in enumerate(masters):
            want = numels[t]
            if not m.is_contiguous() or m.element_size() != 4 or m.numel() != want:
                raise ValueError(f"master shard {plan.manifest[t][0]}: need {want} contiguous fp32 elements")

    @staticmethod
    def _check_arena(plan: Plan, arena: torch.Tensor, rank: int) -> None:
        need = plan.rank_info(rank).dst_arena_bytes
        if not arena.is_cuda or arena.numel() * arena.element_size() < need:
            raise ValueError(f"rollout arena of rank {rank} needs {need} device bytes")

    # ---- NEXT-1 async prefetch / drain --------------------------------------------
    def drain(self, plan: Plan, shards, slab: Slab, stream=None) -> None:
        """Start an offload and return; complete it with wait(OP_OFFLOAD)."""
        arr, n = self._state_ptrs(plan, shards, slab.rank)
        self._keep = getattr(self, "_keep", {})
        self._keep[L.OP_OFFLOAD] = arr
        check(lib.plex_state_drain(self.h, plan.h, arr, n, slab.h, _stream_ptr(stream)))

    def prefetch(self, plan: Plan, slab: Slab, shards, stream=None) -> None:
        """Start an onload into (already allocated) shards and return."""
        arr, n = self._state_ptrs(plan, shards, slab.rank)
        self._keep = getattr(self, "_keep", {})
        self._keep[L.OP_ONLOAD] = arr
        check(lib.plex_state_prefetch(self.h, plan.h, slab.h, arr, n, _stream_ptr(stream)))

    def wait(self, op: int, stream=None) -> None:
        check(lib.plex_state_wait(self.h, op, _stream_ptr(stream)))

    def poll(self, op: int) -> bool:
        d = C.c_int32()
        check(lib.plex_state_poll(self.h, op, C.byref(d)))
        return bool(d.value)

    def sync(self, plan: Plan, masters: Sequence[torch.Tensor], arena: torch.Tensor, stream=None) -> None:
        self._check_masters(plan, masters, self.rank)
        self._check_arena(plan, arena, self.rank)
        arr = ptr_array([m.data_ptr() if m.numel() else 0 for m in masters])
        check(lib.plex_weight_sync(self.h, plan.h, arr, len(masters), arena.data_ptr(), _stream_ptr(stream)))

    def sync_rank(self, plan: Plan, rank: int, masters: Sequence[torch.Tensor], arenas: Sequence[torch.Tensor],
                  stream=None) -> None:
        self._check_masters(plan, masters, rank)
        for g, a in enumerate(arenas):
            self._check_arena(plan, a, g)
        arr = ptr_array([m.data_ptr() if m.numel() else 0 for m in masters])
        ar = ptr_array([a.data_ptr() for a in arenas])
        check(lib.plex_weight_sync_rank(self.h, plan.h, rank, arr, len(masters), ar, len(arenas),
                                        _stream_ptr(stream)))

    def sync_from_slab(self, plan: Plan, slab: Slab, arena: torch.Tensor, stream=None) -> None:
        """NEXT-3: sync a suspended job straight from its pinned slab."""
        self._check_arena(plan, arena, self.rank)
        check(lib.plex_weight_sync_from_slab(self.h, plan.h, slab.h, arena.data_ptr(), _stream_ptr(stream)))

    def sync_rank_from_slab(self, plan: Plan, rank: int, slab: Slab, arenas: Sequence[torch.Tensor],
                            stream=None) -> None:
        for g, a in enumerate(arenas):
            self._check_arena(plan, a, g)
        ar = ptr_array([a.data_ptr() for a in arenas])
        check(lib.plex_weight_sync_rank_from_slab(self.h, plan.h, rank, slab.h, ar, len(arenas), _stream_ptr(stream)))

    # ---- NEXT-2 replicated-param restore ------------------------------------------------
    def param_arena(self, plan: Plan) -> torch.Tensor:
        return torch.empty(max(plan.param_arena_bytes, 256), dtype=torch.uint8, device=f"cuda:{self.device}")

    @staticmethod
    def _check_param_arena(plan: Plan, arena: torch.Tensor) -> None:
        if not plan.replica_param:
            raise ValueError("plan was not built with replica_param=True")
        if not arena.is_cuda or arena.numel() * arena.element_size() < plan.param_arena_bytes:
            raise ValueError(f"param arena needs {plan.param_arena_bytes} device bytes")

    def param_allgather(self, plan: Plan, arena: torch.Tensor, stream=None) -> None:
        """Collective: every rank's own param rows -> every peer's param arena (NVLink)."""
        self._check_param_arena(plan, arena)
        check(lib.plex_param_allgather(self.h, plan.h, arena.data_ptr(), _stream_ptr(stream)))

    def param_allgather_rank(self, plan: Plan, rank: int, arenas: Sequence[torch.Tensor], stream=None) -> None:
        for a in arenas:
            self._check_param_arena(plan, a)
        ar = ptr_array([a.data_ptr() for a in arenas])
        check(lib.plex_param_allgather_rank(self.h, plan.h, rank, ar, len(arenas), _stream_ptr(stream)))

    # ---- helpers ---------------------------------------------------------------------
    def arena(self, plan: Plan, rank: Optional[int] = None) -> torch.Tensor:
        n = plan.rank_info(self.rank if rank is None else rank).dst_arena_bytes
        return torch.empty(max(n, 256), dtype=torch.uint8, device=f"cuda:{self.device}")

    @staticmethod
    def rollout_views(plan: Plan, rank: int, arena: torch.Tensor) -> "OrderedDict[str, torch.Tensor]":
        out = OrderedDict()
        for name, off, shape in plan.dst_tensors(rank):
            n = int(np.prod(shape))
            out[name] = arena[off:off + 2 * n].view(torch.bfloat16).view(shape)
        return out

    def diag_pack(self, plan: Plan, shards, bucket: int, pack: bool = True, stream=None, upload: bool = True,
                  staging_offset: int = 0) -> None:
        """Diagnostic: one K1/K2 launch over one bucket, no copies (plex_diag_pack);
        upload=False reuses the pointer table the previous diag call uploaded."""
        arr, n = self._state_ptrs(plan, shards, self.rank)
        check(lib.plex_diag_pack(self.h, plan.h, arr, n, bucket, (1 if pack else 0) | (0 if upload else 2),
                                 staging_offset, _stream_ptr(stream)))

    def enable_carry(self, plan: Plan) -> None:
        """Give the ctx carry staging (4 bucket slots) if `plan` carries buckets."""
        if not plan.carry():
            return
        need = 4 * plan.bucket_bytes
        if getattr(self, "carry_staging", None) is None or self.carry_staging.numel() < need:
            self.carry_staging = torch.empty(need, dtype=torch.uint8, device=f"cuda:{self.device}")
            check(lib.plex_ctx_set_carry_staging(self.h, self.carry_staging.data_ptr(), self.carry_staging.numel()))

    def workspace_usage(self) -> Tuple[int, int]:
        """(bytes in use, high-water mark) of the device metadata workspace."""
        a, b = C.c_uint64(), C.c_uint64()
        check(lib.plex_ctx_workspace(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def stats(self) -> Dict[str, dict]:
        out = {}
        for i, nm in enumerate(L.STAT_NAMES):
            s = L.KernelStats()
            check(lib.plex_ctx_stats(self.h, i, C.byref(s)))
            out[nm] = {"launches": s.launches, "ms": s.total_ms, "bytes": s.bytes}
        return out

    def trace(self) -> List[Tuple[str, float, int]]:
        """Every timed launch since the last reset: (kind, ms, algorithmic bytes)."""
        n = C.c_int32()
        check(lib.plex_ctx_trace(self.h, None, 0, C.byref(n)))
        buf = (L.LaunchRecord * max(1, n.value))()
        check(lib.plex_ctx_trace(self.h, buf, n.value, C.byref(n)))
        return [(L.STAT_NAMES[r.which], float(r.ms), int(r.bytes)) for r in buf[:n.value]]

    def timeline(self) -> List[dict]:
        """The same records with their start times: {kind, call, start_ms, ms, bytes},
        start relative to the first timed launch of the same blocking call (a
        kernel / copy-engine timeline from CUDA events, no profiler needed)."""
        n = C.c_int32()
        check(lib.plex_ctx_trace(self.h, None, 0, C.byref(n)))
        buf = (L.LaunchRecord * max(1, n.value))()
        check(lib.plex_ctx_trace(self.h, buf, n.value, C.byref(n)))
        return [{"kind": L.STAT_NAMES[r.which], "call": int(r.call), "start_ms": float(r.start_ms),
                 "ms": float(r.ms), "bytes": int(r.bytes)} for r in buf[:n.value]]

    def reset_stats(self) -> None:
        check(lib.plex_ctx_reset_stats(self.h))

    def set_split_push(self, on: bool) -> None:
        """Diagnostic (PLEX_CTX_SPLIT_PUSH): time the sync's local and remote push
        items as two launches (stats "push_local" / "push_remote")."""
        check(lib.plex_ctx_set_flags(self.h, L.CTX_SPLIT_PUSH if on else 0, L.CTX_SPLIT_PUSH))


# ---- infrastructure (synthetic inputs, verification) ------------------------------
def synth_fill(t: torch.Tensor, kind: int, seed: int, key: str, index_base: int = 0, special_bits: int = 0,
               stream=None) -> None:
    check(lib.plex_synth_fill(t.data_ptr() if t.numel() else None, kind, seed, key.encode(), index_base,
                              t.numel(), special_bits, _stream_ptr(stream)))


def synth_mutate(t: torch.Tensor, kind: int, job_seed: int, step: int, key: str, index_base: int = 0,
                 stream=None) -> None:
    check(lib.plex_synth_mutate(t.data_ptr() if t.numel() else None, kind, job_seed, step, key.encode(),
                                index_base, t.numel(), _stream_ptr(stream)))


def checksum(t: torch.Tensor, index_base: int = 0, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """(S1, S2) of R14 as a 2-element int64 device tensor (bit pattern of uint64)."""
    if out is None:
        out = torch.zeros(2, dtype=torch.int64, device=t.device)
    check(lib.plex_checksum(t.data_ptr() if t.numel() else None, t.element_size(), index_base, t.numel(),
                            out.data_ptr(), _stream_ptr(stream)))
    return out


def diag_pack_variant(v: int) -> None:
    """Diagnostic: K1/K2 build for later launches (0 default, 1 L2::evict_first)."""
    check(lib.plex_diag_pack_variant(v))


def cast_rne(src: torch.Tensor, dst: torch.Tensor, stream=None) -> None:
    assert src.dtype == torch.float32 and dst.dtype == torch.bfloat16 and src.numel() == dst.numel()
    check(lib.plex_cast_rne(src.data_ptr(), dst.data_ptr(), src.numel(), _stream_ptr(stream)))


class Job:
    """One job's state on this rank: its FSDP shards (4 kinds), pinned slab
    and plan.  suspend/resume implement a3-a7 plus the release/re-acquire of
    a5 (device storage freed while HOST-resident)."""

    def __init__(self, mgr: StateManager, plan: Plan, seed: int = 0, rank: Optional[int] = None,
                 hugepage: bool = True, slab: bool = True):
        self.mgr, self.plan, self.seed = mgr, plan, seed
        self.rank = mgr.rank if rank is None else rank
        self.slab = Slab(plan, self.rank, hugepage) if slab else None
        self.shards: "OrderedDict[Tuple[str, int], torch.Tensor]" = OrderedDict()
        self.dev = f"cuda:{mgr.device}"
        self.param_arena: Optional[torch.Tensor] = None     # replica_param plans: full bf16 params

    def alloc(self, kinds=(0, 1, 2, 3)) -> "Job":
        replica = self.plan.replica_param and L.KIND_PARAM in kinds
        if replica:
            self.param_arena = self.mgr.param_arena(self.plan)
            views = self.plan.param_views(self.param_arena)
        for t, (key, _) in enumerate(self.plan.manifest):
            shp = self.plan.shard_shape(self.rank, t)
            for kd in kinds:
                if replica and kd == L.KIND_PARAM:
                    self.shards[(key, kd)] = views[key]
                else:
                    self.shards[(key, kd)] = torch.empty(shp, dtype=KIND_TORCH[kd], device=self.dev)
        return self

    def init_synthetic(self, special_bits: int = 0, derived_param: bool = False) -> "Job":
        """Counter-based synthetic state.  derived_param: the bf16
        params are RNE(master) -- what a mixed-precision optimizer step leaves --
        computed by this library's cast kernel instead of drawn independently."""
        by_key: Dict[str, list] = {}
        for (k2, kd), x in self.shards.items():
            by_key.setdefault(k2, []).append((kd, x))
        for t, (key, shape) in enumerate(self.plan.manifest):
            r0, _ = self.plan.shard_rows(self.rank, t)
            re_ = int(np.prod(shape[1:])) if len(shape) > 1 else 1
            for kd, x in by_key.get(key, ()):
                if not (derived_param and kd == 0):
                    full = kd == L.KIND_PARAM and self.param_arena is not None
                    synth_fill(x, kd, self.seed, key, 0 if full else r0 * re_, special_bits)
            if derived_param and (key, 0) in self.shards and (key, 1) in self.shards:
                p, m = self.shards[(key, 0)], self.shards[(key, 1)]
                if self.param_arena is not None:            # this rank's rows of the replica
                    p = p.reshape(-1)[r0 * re_:r0 * re_ + m.numel()]
                if p.numel():
                    cast_rne(m, p)
        return self

    def slab_shards(self):
        """The shards the plan's slab carries (kind mask and optional key subset)."""
        mask, sub = self.plan.kind_mask, self.plan.subset
        return OrderedDict((kk, v) for kk, v in self.shards.items()
                           if mask & (1 << kk[1]) and (sub is None or kk[0] in sub))

    def masters(self) -> List[torch.Tensor]:
        return [self.shards[(k, 1)] for k, _ in self.plan.manifest]

    def suspend(self, stream=None, release: bool = True) -> None:
        self.mgr.offload(self.plan, self.slab_shards(), self.slab, stream)
        if release:
            self.release()

    def release(self) -> None:
        """a5: give the slab-carried shards' device storage back to PyTorch."""
        for v in self.slab_shards().values():
            v.untyped_storage().resize_(0)

    def acquire(self) -> None:
        """a5: re-allocate the slab-carried shards' device storage."""
        if self.param_arena is not None:
            st = self.param_arena.untyped_storage()
            if st.nbytes() != self.param_arena.numel():
                st.resize_(self.param_arena.numel())
        for (key, kd), v in self.slab_shards().items():
            if kd == L.KIND_PARAM and self.param_arena is not None:
                continue
            need = v.numel() * v.element_size()
            if v.untyped_storage().nbytes() != need:
                v.untyped_storage().resize_(need)

    def restore_replicas(self, stream=None) -> None:
        """NEXT-2: after an onload, fill the other ranks' rows of the replicated params."""
        if self.param_arena is not None and self.plan.kind_mask & (1 << L.KIND_PARAM):
            self.mgr.param_allgather(self.plan, self.param_arena, stream)

    def resume(self, stream=None) -> None:
        self.acquire()
        self.mgr.onload(self.plan, self.slab, self.slab_shards(), stream)
        self.restore_replicas(stream)

    def prefetch(self, stream=None) -> None:
        """NEXT-1: start bringing this (HOST-resident) job back; returns at once."""
        self.acquire()
        self.mgr.prefetch(self.plan, self.slab, self.slab_shards(), stream)

    def drain(self, stream=None) -> None:
        """NEXT-1: start offloading this job; returns at once (finish with wait_drain)."""
        self.mgr.drain(self.plan, self.slab_shards(), self.slab, stream)

    def wait_prefetch(self, stream=None) -> None:
        self.mgr.wait(L.OP_ONLOAD, stream)
        self.restore_replicas(stream)

    def wait_drain(self, stream=None, release: bool = True) -> None:
        self.mgr.wait(L.OP_OFFLOAD, stream)
        if release:
            self.release()

    def switch_to(self, other: "Job", stream=None, release: bool = True) -> None:
        """PAPER.md:555 context switch self -> other with both host-link
        directions busy at once (offload self || onload other)."""
        other.acquire()
        self.mgr.switch(self.plan, self.slab_shards(), self.slab, other.plan, other.slab, other.slab_shards(),
                        stream)
        if release:
            self.release()
        other.restore_replicas(stream)

    def swap_with(self, other: "Job", stream=None) -> None:
        """PAPER.md:555 switch self -> other in place (plex_state_swap): other's
        state (HOST, in its slab, same plan layout) takes over self's device
        tensors and self's state takes over that slab.  One device copy and one
        pinned slab serve both jobs."""
        if other.slab is None or other.plan.h.value != self.plan.h.value:
            raise ValueError("swap_with needs the other job suspended in a slab of the same plan")
        self.mgr.swap(self.plan, self.slab_shards(), other.slab, stream)
        self.shards, other.shards = other.shards, self.shards
        self.slab, other.slab = other.slab, self.slab
        self.param_arena, other.param_arena = other.param_arena, self.param_arena
        other.restore_replicas(stream)

    def sync(self, arena: torch.Tensor, stream=None) -> None:
        self.mgr.sync(self.plan, self.masters(), arena, stream)


# ---- a1: transition decision and the group's residency authority ----------------------
def transition_decide(resident: Optional[int], incoming: int, sync: bool = False) -> List[Tuple[int, int]]:
    """PAPER.md:555 op list [(PLEX_OP_*, job)] from the library (plex_transition_decide)."""
    t = L.Transition()
    check(lib.plex_transition_decide(-1 if resident is None else resident, incoming,
                                     L.OP_SYNC if sync else L.OP_NONE, C.byref(t)))
    return [(t.ops[i], t.op_jobs[i]) for i in range(t.n_ops)]


class Group:
    """The GPU group's resident-job map and transition executor (plex_group_*,
    PAPER.md:555 ``group_executor_gpu_job`` / ``_handle_job_transition``).

    One per rank process (on its StateManager).  ``add`` registers jobs;
    ``transition(job, sync=...)`` makes ``job`` the resident one: the library
    decides the ops (offload the resident job, onload ``job``, optional sync),
    picks swap / duplex / sequential from what fits, and calls back here only
    to acquire or release a job's device storage (a5, PyTorch memory).
    ``hbm_budget`` (bytes, optional) caps the job-state bytes the group may
    hold on the device at once; an acquire beyond it (or a CUDA OOM) makes the
    library switch sequentially."""

    def __init__(self, mgr: StateManager, hbm_budget: Optional[int] = None):
        self.mgr = mgr
        self.hbm_budget = hbm_budget
        self.jobs: Dict[int, Job] = {}
        self._storage_of: Dict[int, Optional[int]] = {}
        import weakref
        me = weakref.ref(self)                          # no group <-> callback reference cycle

        def cb(user, jid, acquire, state, n_state):
            g = me()
            return 2 if g is None else g._storage(user, jid, acquire, state, n_state)
        self._cb = L.STORAGE_FN(cb)                     # kept alive with the group
        self._cb_error: Optional[BaseException] = None
        h = C.c_void_p()
        check(lib.plex_group_create(mgr.h, self._cb, None, C.byref(h)))
        self.h = h

    def close(self):
        """Destroy the library group; the jobs (and their device memory) are
        released from the group's bookkeeping."""
        h = getattr(self, "h", None)
        if h is not None and h.value and lib is not None:
            lib.plex_group_destroy(h)
            self.h = None
        self.jobs = {}

    def __del__(self):
        self.close()

    # ---- registration -----------------------------------------------------------------
    def _table(self, job: Job):
        return self.mgr._state_ptrs(job.plan, job.shards, job.rank)

    def add(self, job: Job, resident: bool = False, storage: Optional[int] = None) -> int:
        """Register ``job``; returns its id.  resident=True: its state is on the
        device now (at most one such job).  Jobs given the same ``storage`` id
        share one set of device tensors (in-place swaps): register the one whose
        shards are allocated first."""
        jid = len(self.jobs)
        arr, n = (None, 0)
        if job.shards and all(v.untyped_storage().nbytes() == v.numel() * v.element_size()
                              for v in job.slab_shards().values()):
            arr, n = self._table(job)
        check(lib.plex_group_add_job(self.h, jid, job.plan.h, job.slab.h if job.slab is not None else None,
                                     -1 if storage is None else storage, L.GROUP_RESIDENT if resident else 0,
                                     arr, n))
        self.jobs[jid] = job
        self._storage_of[jid] = storage
        job.group_id = jid
        return jid

    @property
    def resident(self) -> Optional[Job]:
        j = C.c_int64()
        check(lib.plex_group_resident(self.h, C.byref(j)))
        return None if j.value < 0 else self.jobs[j.value]

    # ---- a5 storage callback (runs inside plex_group_transition) ------------------------------
    def _device_bytes(self) -> int:
        n = 0
        for jb in self.jobs.values():
            for v in jb.slab_shards().values():
                n += v.untyped_storage().nbytes()
        return n

    def _storage(self, user, jid, acquire, state, n_state):
        try:
            job = self.jobs[jid]
            if acquire:
                if self.hbm_budget is not None:
                    need = sum(v.numel() * v.element_size() for v in job.slab_shards().values())
                    if self._device_bytes() + need > self.hbm_budget:
                        return 1                                       # does not fit: go sequential
                try:
                    job.acquire()
                except torch.OutOfMemoryError:
                    return 1
                arr, n = self._table(job)
                if n != n_state:
                    raise ValueError(f"pointer table of {n} entries, library expects {n_state}")
                for i in range(n):
                    state[i] = arr[i]
            else:
                job.release()
            return 0
        except BaseException as e:                                   # never let an exception cross the ABI
            self._cb_error = e
            return 2

    # ---- the transition --------------------------------------------------------------------
    def transition(self, job: Job, sync=None, stream=None) -> dict:
        """Run (op of) ``job`` on the group: [OFFLOAD resident, ONLOAD job] when
        they differ, then SYNC job when ``sync`` is given -- one
        rollout arena (collective sync) or every rank's arena (emulation).
        Returns {"ops": [(op, job id)], "mode": "swap"|"duplex"|...,
        "resident_before", "resident_after"}."""
        jid = job.group_id
        arenas, n_ar = None, 0
        if sync is not None:
            lst = list(sync) if isinstance(sync, (list, tuple)) else [sync]
            for g, a in enumerate(lst):
                StateManager._check_arena(job.plan, a, self.mgr.rank if len(lst) == 1 else g)
            arenas, n_ar = ptr_array([a.data_ptr() for a in lst]), len(lst)
        t = L.Transition()
        self._cb_error = None
        rb = C.c_int64()
        check(lib.plex_group_resident(self.h, C.byref(rb)))
        before = self.jobs.get(rb.value) if rb.value >= 0 else None
        code = lib.plex_group_transition(self.h, jid, L.OP_SYNC if sync is not None else L.OP_NONE, arenas, n_ar,
                                         _stream_ptr(stream), C.byref(t))
        if self._cb_error is not None:
            raise RuntimeError("storage callback failed") from self._cb_error
        shared = (before is not None and before is not job and self._storage_of.get(before.group_id) is not None
                  and self._storage_of.get(before.group_id) == self._storage_of.get(jid))
        if shared and (code == L.OK or code == L.E_CHECKSUM):
            # mirror the library's in-place swap: the slab now holds the outgoing
            # state; on success the tensors hold the incoming one
            before.slab, job.slab = job.slab, before.slab
            if code == L.OK:
                before.shards, job.shards = job.shards, before.shards
                before.param_arena, job.param_arena = job.param_arena, before.param_arena
        check(code)
        return {"ops": [(t.ops[i], t.op_jobs[i]) for i in range(t.n_ops)], "mode": L.SWITCH_NAMES[t.mode],
                "resident_before": t.resident_before, "resident_after": t.resident_after}
