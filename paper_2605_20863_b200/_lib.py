"""ctypes binding of libplex.so (include/plex.h).  Argument marshalling only:
every step of the path runs in the library's CUDA kernels / copy engines.

Importing this module loads the in-tree ``libplex.so`` and fails loudly if it
is missing: there is no CPU or PyTorch fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libplex.so")

OK, E_INVAL, E_LAYOUT, E_TIER_FULL, E_STATE, E_CUDA, E_NCCL, E_CHECKSUM = 0, -1, -2, -3, -4, -5, -6, -7
KIND_PARAM, KIND_MASTER, KIND_EXP_AVG, KIND_EXP_AVG_SQ = 0, 1, 2, 3
NUM_KINDS = 4
KINDMASK_ALL, KINDMASK_OPTIM = 0xF, 0xE
ROLE_REPLICATED, ROLE_COL, ROLE_ROW, ROLE_EXPERT, ROLE_AUTO = 0, 1, 2, 3, -1
SLAB_KIND_MAJOR, SLAB_KEY_MAJOR = 0, 1
RANKMAP_TP_FAST, RANKMAP_DP_FAST, RANKMAP_AUTO = 0, 1, 2
OP_NONE, OP_OFFLOAD, OP_ONLOAD, OP_SYNC = 0, 1, 2, 3
RES_DEVICE, RES_HOST, RES_DISK = 0, 1, 2
CTX_TIMING, CTX_SYNC_NCCL, CTX_CARRY_NCCL, CTX_SPLIT_PUSH = 0x1, 0x2, 0x4, 0x8
SLAB_HUGEPAGE = 0x1
STAT_PACK, STAT_UNPACK, STAT_PUSH, STAT_D2H, STAT_H2D, STAT_NCCL, STAT_RPACK, STAT_RUNPACK, STAT_DERIVE, \
    STAT_BARRIER, STAT_GATHER, STAT_PUSH_LOCAL, STAT_PUSH_REMOTE = range(13)
STAT_NAMES = ("pack", "unpack", "push", "d2h", "h2d", "nccl", "rpack", "runpack", "derive", "barrier", "gather",
              "push_local", "push_remote")
NUM_STATS = 13
PLAN_ELIDE_PARAM = 0x1
PLAN_REPLICA_PARAM = 0x2
SWITCH_NONE, SWITCH_LOAD, SWITCH_SWAP, SWITCH_DUPLEX, SWITCH_SEQUENTIAL = 0, 1, 2, 3, 4
SWITCH_NAMES = ("none", "load", "swap", "duplex", "sequential")
GROUP_RESIDENT = 0x1

EXPORTS = [
    "plex_last_error", "plex_version", "plex_transition_plan", "plex_plan_destroy", "plex_plan_query",
    "plex_plan_rank_info", "plex_plan_segment", "plex_plan_dst_tensor", "plex_plan_shard_rows", "plex_plan_ledger",
    "plex_plan_n_carry", "plex_plan_carry", "plex_ctx_set_carry_staging", "plex_slab_carry",
    "plex_nccl_unique_id", "plex_ctx_create", "plex_ctx_workspace", "plex_ctx_destroy", "plex_ctx_stats", "plex_ctx_reset_stats",
    "plex_ctx_trace", "plex_ctx_set_flags",
    "plex_slab_create", "plex_slab_destroy", "plex_slab_info", "plex_slab_elided", "plex_slab_checksums",
    "plex_slab_spill", "plex_slab_fill",
    "plex_state_offload", "plex_state_onload", "plex_state_switch", "plex_weight_sync",
    "plex_state_drain", "plex_state_prefetch", "plex_state_wait", "plex_state_poll", "plex_weight_sync_rank",
    "plex_weight_sync_from_slab", "plex_weight_sync_rank_from_slab",
    "plex_plan_param_arena", "plex_param_allgather", "plex_param_allgather_rank",
    "plex_slab_checkpoint", "plex_slab_checkpoint_start", "plex_ckpt_wait", "plex_slab_restore", "plex_state_swap",
    "plex_synth_fill", "plex_synth_mutate", "plex_checksum", "plex_cast_rne", "plex_diag_pack",
    "plex_diag_pack_variant",
    "plex_transition_decide", "plex_plan_group", "plex_group_create", "plex_group_destroy", "plex_group_add_job",
    "plex_group_resident", "plex_group_job_slab", "plex_group_transition",
]


class PlexError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"plex error {code}: {msg}")
        self.code = code


class TensorDesc(C.Structure):
    _fields_ = [("key", C.c_char_p), ("d0", C.c_int64), ("d1", C.c_int64), ("ndim", C.c_int32),
                ("role", C.c_int32), ("group", C.c_int32), ("slot", C.c_int32), ("expert", C.c_int32),
                ("unit", C.c_int32)]


class PlanReq(C.Structure):
    _fields_ = [("n_tensors", C.c_int32), ("tensors", C.POINTER(TensorDesc)), ("world", C.c_int32),
                ("tp", C.c_int32), ("dp", C.c_int32), ("ep", C.c_int32), ("rank_map", C.c_int32),
                ("slab_layout", C.c_int32), ("kind_mask", C.c_uint32), ("n_subset", C.c_int32),
                ("subset", C.POINTER(C.c_int32)), ("bucket_bytes", C.c_uint64), ("tile_bytes", C.c_uint64),
                ("resident_job", C.c_int64), ("incoming_job", C.c_int64), ("op", C.c_int32), ("flags", C.c_uint32),
                ("link_weights", C.POINTER(C.c_float)), ("head_dim", C.c_int32)]


class PlanStats(C.Structure):
    _fields_ = [("n_ops", C.c_int32), ("ops", C.c_int32 * 4), ("op_jobs", C.c_int64 * 4),
                ("n_tensors", C.c_int32), ("world", C.c_int32), ("tp", C.c_int32), ("dp", C.c_int32),
                ("ep", C.c_int32), ("total_params", C.c_uint64), ("rank_map", C.c_int32)]


class RankInfo(C.Structure):
    _fields_ = [("slab_bytes", C.c_uint64), ("payload_bytes", C.c_uint64), ("n_segments", C.c_int32),
                ("n_buckets", C.c_int32), ("n_pack_items", C.c_uint64), ("dst_arena_bytes", C.c_uint64),
                ("n_dst_tensors", C.c_int32), ("n_push_items", C.c_uint64), ("send_bytes", C.c_uint64),
                ("recv_bytes", C.c_uint64), ("local_bytes", C.c_uint64), ("src_read_bytes", C.c_uint64),
                ("elide_buckets", C.c_int32), ("elide_bytes", C.c_uint64), ("carried_out", C.c_int32),
                ("carried_in", C.c_int32), ("carry_bytes", C.c_uint64), ("n_gather_items", C.c_uint64),
                ("gather_send_bytes", C.c_uint64), ("gather_recv_bytes", C.c_uint64)]


class CarryDesc(C.Structure):
    _fields_ = [("owner", C.c_int32), ("bucket", C.c_int32), ("carrier", C.c_int32), ("slab_offset", C.c_uint64),
                ("bytes", C.c_uint64), ("carry_offset", C.c_uint64)]


class SegDesc(C.Structure):
    _fields_ = [("tensor", C.c_int32), ("kind", C.c_int32), ("slab_offset", C.c_uint64), ("nbytes", C.c_uint64),
                ("row0", C.c_int64), ("row1", C.c_int64), ("index_base", C.c_uint64)]


class DstDesc(C.Structure):
    _fields_ = [("group", C.c_int32), ("first_tensor", C.c_int32), ("arena_offset", C.c_uint64),
                ("rows", C.c_int64), ("cols", C.c_int64)]


class LaunchRecord(C.Structure):
    _fields_ = [("which", C.c_int32), ("ms", C.c_float), ("bytes", C.c_uint64), ("start_ms", C.c_float),
                ("call", C.c_int32)]


class Transition(C.Structure):
    _fields_ = [("n_ops", C.c_int32), ("ops", C.c_int32 * 4), ("op_jobs", C.c_int64 * 4), ("mode", C.c_int32),
                ("resident_before", C.c_int64), ("resident_after", C.c_int64)]


STORAGE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int64, C.c_int32, C.POINTER(C.c_void_p), C.c_int32)


class KernelStats(C.Structure):
    _fields_ = [("launches", C.c_uint64), ("total_ms", C.c_double), ("bytes", C.c_uint64)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    P, VP, I32, U32, U64, I64 = C.POINTER, C.c_void_p, C.c_int32, C.c_uint32, C.c_uint64, C.c_int64
    sig = {
        "plex_last_error": (C.c_char_p, []),
        "plex_version": (C.c_char_p, []),
        "plex_transition_plan": (C.c_int, [P(PlanReq), P(VP)]),
        "plex_plan_destroy": (C.c_int, [VP]),
        "plex_plan_query": (C.c_int, [VP, P(PlanStats)]),
        "plex_plan_rank_info": (C.c_int, [VP, I32, P(RankInfo)]),
        "plex_plan_segment": (C.c_int, [VP, I32, I32, P(SegDesc)]),
        "plex_plan_dst_tensor": (C.c_int, [VP, I32, I32, P(DstDesc)]),
        "plex_plan_shard_rows": (C.c_int, [VP, I32, I32, P(I64), P(I64)]),
        "plex_plan_ledger": (C.c_int, [VP, P(U64), I32]),
        "plex_plan_n_carry": (C.c_int, [VP, P(I32)]),
        "plex_plan_carry": (C.c_int, [VP, I32, P(CarryDesc)]),
        "plex_ctx_set_carry_staging": (C.c_int, [VP, VP, U64]),
        "plex_slab_carry": (C.c_int, [VP, P(VP), P(U64)]),
        "plex_nccl_unique_id": (C.c_int, [VP]),
        "plex_ctx_create": (C.c_int, [I32, VP, U64, VP, U64, I32, VP, VP, VP, I32, I32, U32, P(VP)]),
        "plex_ctx_workspace": (C.c_int, [VP, P(U64), P(U64)]),
        "plex_ctx_destroy": (C.c_int, [VP]),
        "plex_ctx_stats": (C.c_int, [VP, I32, P(KernelStats)]),
        "plex_ctx_reset_stats": (C.c_int, [VP]),
        "plex_ctx_set_flags": (C.c_int, [VP, U32, U32]),
        "plex_ctx_trace": (C.c_int, [VP, P(LaunchRecord), I32, P(I32)]),
        "plex_slab_create": (C.c_int, [VP, I32, U32, P(VP)]),
        "plex_slab_destroy": (C.c_int, [VP]),
        "plex_slab_info": (C.c_int, [VP, P(VP), P(U64), P(I32)]),
        "plex_slab_elided": (C.c_int, [VP, P(I32)]),
        "plex_slab_spill": (C.c_int, [VP, C.c_char_p, I32]),
        "plex_slab_fill": (C.c_int, [VP, C.c_char_p, I32]),
        "plex_slab_checksums": (C.c_int, [VP, P(U64), I32]),
        "plex_state_offload": (C.c_int, [VP, VP, P(VP), I32, VP, VP]),
        "plex_state_onload": (C.c_int, [VP, VP, VP, P(VP), I32, VP]),
        "plex_state_switch": (C.c_int, [VP, VP, P(VP), I32, VP, VP, VP, P(VP), I32, VP]),
        "plex_state_drain": (C.c_int, [VP, VP, P(VP), I32, VP, VP]),
        "plex_state_prefetch": (C.c_int, [VP, VP, VP, P(VP), I32, VP]),
        "plex_state_wait": (C.c_int, [VP, I32, VP]),
        "plex_state_poll": (C.c_int, [VP, I32, P(I32)]),
        "plex_weight_sync": (C.c_int, [VP, VP, P(VP), I32, VP, VP]),
        "plex_weight_sync_rank": (C.c_int, [VP, VP, I32, P(VP), I32, P(VP), I32, VP]),
        "plex_weight_sync_from_slab": (C.c_int, [VP, VP, VP, VP, VP]),
        "plex_weight_sync_rank_from_slab": (C.c_int, [VP, VP, I32, VP, P(VP), I32, VP]),
        "plex_state_swap": (C.c_int, [VP, VP, P(VP), I32, VP, VP]),
        "plex_slab_checkpoint": (C.c_int, [VP, VP, C.c_char_p, I32]),
        "plex_slab_checkpoint_start": (C.c_int, [VP, VP, C.c_char_p, I32, P(VP)]),
        "plex_ckpt_wait": (C.c_int, [VP]),
        "plex_slab_restore": (C.c_int, [VP, VP, C.c_char_p, I32]),
        "plex_plan_param_arena": (C.c_int, [VP, I32, P(U64), P(U64)]),
        "plex_param_allgather": (C.c_int, [VP, VP, VP, VP]),
        "plex_param_allgather_rank": (C.c_int, [VP, VP, I32, P(VP), I32, VP]),
        "plex_synth_fill": (C.c_int, [VP, I32, U64, C.c_char_p, U64, U64, I32, VP]),
        "plex_synth_mutate": (C.c_int, [VP, I32, U64, U64, C.c_char_p, U64, U64, VP]),
        "plex_checksum": (C.c_int, [VP, I32, U64, U64, VP, VP]),
        "plex_cast_rne": (C.c_int, [VP, VP, U64, VP]),
        "plex_diag_pack": (C.c_int, [VP, VP, P(VP), I32, I32, I32, U64, VP]),
        "plex_diag_pack_variant": (C.c_int, [I32]),
        "plex_transition_decide": (C.c_int, [I64, I64, I32, P(Transition)]),
        "plex_plan_group": (C.c_int, [VP, I32, C.c_char_p, I32, P(I32), P(I32), P(I32)]),
        "plex_group_create": (C.c_int, [VP, STORAGE_FN, VP, P(VP)]),
        "plex_group_destroy": (C.c_int, [VP]),
        "plex_group_add_job": (C.c_int, [VP, I64, VP, VP, I64, U32, P(VP), I32]),
        "plex_group_resident": (C.c_int, [VP, P(I64)]),
        "plex_group_job_slab": (C.c_int, [VP, I64, P(VP)]),
        "plex_group_transition": (C.c_int, [VP, I64, I32, P(VP), I32, VP, P(Transition)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def check(code: int) -> None:
    if code != OK:
        raise PlexError(code, lib.plex_last_error().decode(errors="replace"))


def ptr_array(ptrs) -> "C.Array":
    arr = (C.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p or None
    return arr
