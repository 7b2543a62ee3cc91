/*
 * plex.h — C ABI of libplex.so, the B200-native data plane of PlexRL's
 * GPU-group state transition (arXiv 2605.20863, /root/reference/PAPER.md).
 *
 * The paper's StateManager exposes "blocking state-transfer primitives":
 * "when a transfer returns, the requested state is resident and safe to use
 * on the default CUDA stream" (§5.3).  The scheduler prepends
 * "offload and load operations" when the incoming job differs from the
 * resident one (§5.2.2), and weight synchronisation
 * "materializ[es] training-visible state into the format expected by serving
 * instances" (§4.5) with "each rollout rank fetch[ing] only the
 * tensor slices required by its target parallel layout" (§5.3).
 *
 * Conventions:
 *  - Every export returns plex_status (PLEX_OK = 0, negative on error); a
 *    thread-local message is available from plex_last_error().  No C++
 *    exception crosses the ABI.
 *  - No partial mutation: a failed offload leaves the device tensors and the
 *    slab's residency untouched; a failed onload leaves the slab untouched and
 *    its residency HOST (destination contents unspecified); a failed sync
 *    leaves the sources untouched (destination unspecified).
 *  - Device memory is always the CALLER's (PyTorch's): state, rollout
 *    tensors, staging, and a device workspace handed to plex_ctx_create in
 *    which the library keeps its metadata tables (segment / work-item tables,
 *    pointer tables, checksum accumulators, handshake flags).  The library
 *    never calls cudaMalloc (NCCL internals excepted); it allocates pinned
 *    host memory (slabs, small mirrors) and events.  Streams are the
 *    caller's (cudaStream_t passed as void*).
 *  - Plans are immutable after creation and may be shared read-only.  Calls
 *    on one (job, rank) state are serialised by the caller (WPG-serial
 *    semantics).
 *  - Element values are treated as raw bits: bf16 = 2 B, fp32 = 4 B.
 */
#ifndef PLEX_H
#define PLEX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define PLEX_API __attribute__((visibility("default")))
#else
#define PLEX_API
#endif

typedef int plex_status;

#define PLEX_OK            0
#define PLEX_E_INVAL      -1  /* bad argument / shape / pointer count          */
#define PLEX_E_LAYOUT     -2  /* shape not divisible by TP / EP / head split   */
#define PLEX_E_TIER_FULL  -3  /* pinned host allocation failed / too small     */
#define PLEX_E_STATE      -4  /* residency mismatch (e.g. onload of empty slab)*/
#define PLEX_E_CUDA       -5  /* CUDA runtime error                            */
#define PLEX_E_NCCL       -6  /* NCCL error                                    */
#define PLEX_E_CHECKSUM   -7  /* onload: restored bytes fail the R14 checksum  */

/* State kinds (reading R1): bf16 params, fp32 master, Adam m, Adam v. */
#define PLEX_KIND_PARAM       0   /* bf16, 2 B */
#define PLEX_KIND_MASTER      1   /* fp32, 4 B */
#define PLEX_KIND_EXP_AVG     2   /* fp32, 4 B */
#define PLEX_KIND_EXP_AVG_SQ  3   /* fp32, 4 B */
#define PLEX_NUM_KINDS        4
#define PLEX_KINDMASK_ALL     0xFu
#define PLEX_KINDMASK_OPTIM   0xEu  /* master + m + v (config 3) */

/* Destination roles (reading R3, Megatron/vLLM tensor-parallel conventions). */
#define PLEX_ROLE_REPLICATED  0   /* whole tensor on every rollout rank            */
#define PLEX_ROLE_COL         1   /* dim-0 split by TP; pieces of one group fused  */
#define PLEX_ROLE_ROW         2   /* dim-1 split by TP                             */
#define PLEX_ROLE_EXPERT      3   /* whole tensor on EP rank floor(e / (E/EP))     */
#define PLEX_ROLE_AUTO       -1   /* the planner classifies the tensor from its key (R3):
                                     group / slot / expert / unit are then ignored   */

#define PLEX_SLAB_KIND_MAJOR  0   /* R4: for kind: for key   (default)  */
#define PLEX_SLAB_KEY_MAJOR   1   /* R4: for key: for kind   (per-expert units) */

#define PLEX_RANKMAP_TP_FAST  0   /* R10: g = dp*TP + tp (default) */
#define PLEX_RANKMAP_DP_FAST  1   /* R10: g = tp*DP + dp           */
#define PLEX_RANKMAP_AUTO     2   /* R10: whichever of the two moves fewer bytes over the
                                     busiest link (plan_stats.rank_map reports it) */

/* Transition ops. */
#define PLEX_OP_NONE     0
#define PLEX_OP_OFFLOAD  1
#define PLEX_OP_ONLOAD   2
#define PLEX_OP_SYNC     3

/* Residency of a slab's job state (PAPER.md:505-506 hierarchical residency). */
#define PLEX_RES_DEVICE  0
#define PLEX_RES_HOST    1
#define PLEX_RES_DISK    2   /* NEXT-4 cold tier */

/* Context flags. */
#define PLEX_CTX_TIMING    0x1u  /* record CUDA events around every kernel/copy */
#define PLEX_CTX_CARRY_NCCL 0x4u /* carried buckets (NEXT-1 balancing) via NCCL send/recv
                                    through the carrier's staging instead of the default
                                    peer-memory transport (baseline) */
#define PLEX_CTX_SYNC_NCCL 0x2u  /* weight sync via K4 pack + NCCL send/recv + K5
                                    unpack instead of the fused NVLink push     */
#define PLEX_CTX_SPLIT_PUSH 0x8u /* diagnostic: the fused push runs as two launches, the
                                    local (HBM-only) items then the remote (NVLink)
                                    items, timed separately (PLEX_STAT_PUSH_LOCAL /
                                    _REMOTE) so each gets its own roofline fraction */

/* Slab flags. */
#define PLEX_SLAB_HUGEPAGE 0x1u  /* mmap + MADV_HUGEPAGE + cudaHostRegister      */

typedef struct plex_plan_s* plex_plan_t;
typedef struct plex_ctx_s*  plex_ctx_t;
typedef struct plex_slab_s* plex_slab_t;
typedef struct plex_ckpt_s* plex_ckpt_t;     /* a background checkpoint */

/* One logical (unsharded) tensor of the job's manifest, in canonical order
 * (R4).  2-D view [d0, d1]; 1-D tensors have d1 = 1, ndim = 1.
 *   role   : PLEX_ROLE_*, or PLEX_ROLE_AUTO for every tensor of the manifest:
 *            the planner then derives role, group, slot, expert and unit from
 *            the Hugging Face / Qwen parameter key alone (reading R3,
 *            PAPER.md:576 "target parallel layout"):
 *              *embed_tokens.weight, lm_head.weight        COL (vocab-parallel)
 *              model.layers.N.self_attn.{q,k,v}_proj.{weight,bias}
 *                                                          COL, fused into
 *                   "model.layers.N.self_attn.qkv_proj.{weight,bias}" (slots q,k,v;
 *                   unit = plex_plan_req.head_dim)
 *              model.layers.N.self_attn.o_proj.weight      ROW
 *              model.layers.N.mlp.{gate,up}_proj.weight    COL, fused into
 *                   "model.layers.N.mlp.gate_up_proj.weight" (slots gate, up)
 *              model.layers.N.mlp.down_proj.weight         ROW
 *              model.layers.N.mlp.experts.E.{gate,up}_proj.weight
 *                   EXPERT E, stacked into "model.layers.N.mlp.experts.w13_weight"
 *              model.layers.N.mlp.experts.E.down_proj.weight
 *                   EXPERT E, stacked into "model.layers.N.mlp.experts.w2_weight"
 *              anything else (norms, q_norm/k_norm, router)  REPLICATED
 *            Group ids follow first appearance; plex_plan_group_name names
 *            them.  Mixing AUTO and explicit roles is E_INVAL.
 *   group  : destination tensor id; tensors sharing a group are fused into
 *            one rollout tensor, pieces concatenated along dim 0 in `slot`
 *            order (qkv = q|k|v, gate_up = gate|up, w13 = gate_e|up_e ...).
 *   expert : expert index e for PLEX_ROLE_EXPERT (else -1).
 *   unit   : COL split granularity in rows (head_dim for q/k/v, else 1). */
typedef struct {
    const char* key;
    int64_t d0, d1;
    int32_t ndim;
    int32_t role;
    int32_t group;
    int32_t slot;
    int32_t expert;
    int32_t unit;
} plex_tensor_desc;

/* Plan request (a1 + a2).  `world` is the GPU-group size: FSDP-world source
 * shards (R2: rank r owns rows [min(d0,r*c), min(d0,(r+1)*c)), c=ceil(d0/N))
 * and tp*dp destination ranks (tp*dp must equal world, or tp = dp = 0 for a
 * plan without sync).  `subset` (optional) restricts the slab to those tensor
 * indices; `kind_mask` to those kinds.  `bucket_bytes` is the staging bucket
 * (multiple of 256 B, default 64 MiB); `tile_bytes` the kernel work item
 * (multiple of 256 B, default 64 KiB).  resident_job / incoming_job (-1 =
 * none) and `op` drive the transition decision of PAPER.md:555. */
typedef struct {
    int32_t n_tensors;
    const plex_tensor_desc* tensors;
    int32_t world;
    int32_t tp, dp, ep;
    int32_t rank_map;
    int32_t slab_layout;
    uint32_t kind_mask;
    int32_t n_subset;
    const int32_t* subset;
    uint64_t bucket_bytes;
    uint64_t tile_bytes;
    int64_t resident_job;
    int64_t incoming_job;
    int32_t op;
    uint32_t flags;              /* PLEX_PLAN_* */
    /* NEXT-1 host-link balancing: relative host-link rate of every rank
     * (world entries, > 0; NULL = no carrying).  Ranks whose slab would take
     * longer than the group average hand whole buckets over NVLink to ranks
     * with spare host bandwidth, which keep them in a pinned carry region. */
    const float* link_weights;
    /* PLEX_ROLE_AUTO manifests: rows per attention head (q/k/v split unit);
     * 0 = 1 (no head-granularity check). */
    int32_t head_dim;
} plex_plan_req;

/* Plan flags. */
/* NEXT-2 derived-state elision (canonical non-redundant
 * offloaded state): with KIND_MAJOR slabs carrying PARAM and MASTER, offload
 * first checks on the device that every bf16 param equals RNE(master) (R8) -- true after every mixed-precision optimizer step
 * -- and if so neither packs nor copies the PARAM prefix (the remaining
 * slab moves on a bucket grid starting at the first MASTER byte); onload
 * re-derives the params from the restored master.  Checksums cover the derived params, so a failed
 * derivation is still caught (E_CHECKSUM).  Falls back to a full offload when
 * any element differs. */
#define PLEX_PLAN_ELIDE_PARAM 0x1u
/* NEXT-2 canonical dedup of replicated state ("deduplicating
 * replicated state"; ZeRO-2 training): the bf16 PARAM tensors
 * are replicated on every rank of the world (master / m / v stay FSDP-N dim-0
 * chunks).  Each rank's slab still holds only its own FSDP rows of every
 * param, so the slab bytes are those of the sharded plan and a replica is
 * moved over the host link exactly once per group (1/world of it per rank).
 * State pointers of kind PARAM are then the FULL replicated tensors (row 0);
 * offload/onload read/write this rank's rows of them, and
 * plex_param_allgather restores the other ranks' rows over NVLink.  The
 * replicated params live in one per-rank bf16 "param arena" whose layout is
 * given by plex_plan_param_arena (every tensor at a 256-B-aligned offset, in
 * manifest order). */
#define PLEX_PLAN_REPLICA_PARAM 0x2u

typedef struct {
    int32_t n_ops;               /* transition op list       */
    int32_t ops[4];              /* PLEX_OP_*                               */
    int64_t op_jobs[4];
    int32_t n_tensors;
    int32_t world, tp, dp, ep;
    uint64_t total_params;       /* sum of numel over the manifest         */
    int32_t rank_map;            /* rank map in use (AUTO resolved)         */
} plex_plan_stats;

typedef struct {
    uint64_t slab_bytes;         /* pinned slab size (256-B aligned)        */
    uint64_t payload_bytes;      /* sum of segment bytes (no padding)       */
    int32_t n_segments;
    int32_t n_buckets;
    uint64_t n_pack_items;
    uint64_t dst_arena_bytes;    /* rollout arena size for this rank        */
    int32_t n_dst_tensors;
    uint64_t n_push_items;
    uint64_t send_bytes;         /* bf16 bytes this rank pushes to peers    */
    uint64_t recv_bytes;         /* bf16 bytes peers push to this rank      */
    uint64_t local_bytes;        /* bf16 bytes cast locally (no transfer)   */
    uint64_t src_read_bytes;     /* fp32 bytes read by this rank's push     */
    int32_t elide_buckets;       /* PLEX_PLAN_ELIDE_PARAM: buckets still moved when eliding */
    uint64_t elide_bytes;        /* ... and the PARAM prefix derived instead (0 = none) */
    int32_t carried_out;         /* own buckets carried by other ranks      */
    int32_t carried_in;          /* other ranks' buckets this rank carries  */
    uint64_t carry_bytes;        /* pinned carry region this rank hosts     */
    uint64_t n_gather_items;     /* PLEX_PLAN_REPLICA_PARAM: all-gather push items */
    uint64_t gather_send_bytes;  /* ... bf16 bytes this rank stores into peers */
    uint64_t gather_recv_bytes;  /* ... bf16 bytes peers store into this rank  */
} plex_rank_info;

typedef struct {                 /* one carried bucket (global plan order)  */
    int32_t owner, bucket, carrier;
    uint64_t slab_offset;        /* in the owner's canonical slab           */
    uint64_t bytes;
    uint64_t carry_offset;       /* in the carrier's carry region           */
} plex_carry_desc;

typedef struct {
    int32_t tensor;              /* manifest index                          */
    int32_t kind;
    uint64_t slab_offset;
    uint64_t nbytes;
    int64_t row0, row1;          /* FSDP rows of the logical tensor         */
    uint64_t index_base;         /* logical flat index of first element     */
} plex_seg_desc;

typedef struct {
    int32_t group;               /* plex_tensor_desc.group                  */
    int32_t first_tensor;        /* manifest index of its first piece       */
    uint64_t arena_offset;       /* byte offset in the rank's arena (256-B) */
    int64_t rows, cols;          /* 2-D bf16 shape                          */
} plex_dst_desc;

typedef struct {
    uint64_t launches;
    double   total_ms;           /* sum of per-launch CUDA-event durations  */
    uint64_t bytes;              /* algorithmic bytes moved by those launches */
} plex_kernel_stats;

typedef struct {
    int32_t which;               /* PLEX_STAT_*                              */
    float ms;                    /* CUDA-event duration of the launch/copy   */
    uint64_t bytes;              /* algorithmic bytes                        */
    float start_ms;              /* start relative to the first timed launch of the same call */
    int32_t call;                /* index of the blocking call it belongs to (since the last reset) */
} plex_launch_record;

#define PLEX_STAT_PACK    0      /* K1 gather-pack (+checksum)  */
#define PLEX_STAT_UNPACK  1      /* K2 scatter-unpack (+verify) */
#define PLEX_STAT_PUSH    2      /* K3+K4 fused cast/reshard push over NVLink */
#define PLEX_STAT_D2H     3      /* CE1 bucket copies           */
#define PLEX_STAT_H2D     4      /* CE2 bucket copies           */
#define PLEX_STAT_NCCL    5      /* NCCL exchange (sync baseline) */
#define PLEX_STAT_RPACK   6      /* K4 reshard-pack (NCCL path) */
#define PLEX_STAT_RUNPACK 7      /* K5 reshard-unpack (NCCL path) */
#define PLEX_STAT_DERIVE  8      /* NEXT-2 param check / re-derivation */
#define PLEX_STAT_BARRIER 9      /* sync entry barrier (time spent waiting for the slowest rank) */
#define PLEX_STAT_GATHER  10     /* NEXT-2 replicated-param all-gather push */
#define PLEX_STAT_PUSH_LOCAL  11 /* PLEX_CTX_SPLIT_PUSH: local items (bytes: 4 read + 2 written per element) */
#define PLEX_STAT_PUSH_REMOTE 12 /* PLEX_CTX_SPLIT_PUSH: remote items (bytes: 2 sent over NVLink per element) */
#define PLEX_NUM_STATS    13

/* a1 transition decision and what the group executor did. */
#define PLEX_SWITCH_NONE        0   /* incoming job already resident: no transfer      */
#define PLEX_SWITCH_LOAD        1   /* nothing resident: onload only                   */
#define PLEX_SWITCH_SWAP        2   /* in-place plex_state_swap (shared device storage) */
#define PLEX_SWITCH_DUPLEX      3   /* plex_state_switch: offload || onload            */
#define PLEX_SWITCH_SEQUENTIAL  4   /* offload, release, acquire, onload               */

typedef struct {
    int32_t n_ops;               /* op list of PAPER.md:555 (PLEX_OP_*)          */
    int32_t ops[4];
    int64_t op_jobs[4];
    int32_t mode;                /* PLEX_SWITCH_* (plex_group_transition only)    */
    int64_t resident_before;     /* -1 = no job resident on the group             */
    int64_t resident_after;
} plex_transition;

/* ---- errors / version ---------------------------------------------------- */
PLEX_API const char* plex_last_error(void);
PLEX_API const char* plex_version(void);

/* ---- a1: transition decision (pure host) ----------------------------------- */
/* PAPER.md:555 (_handle_job_transition): if the incoming operation's job
 * differs from the job resident on the GPU group, prepend OFFLOAD(resident)
 * (when one is resident, i.e. resident >= 0) and ONLOAD(incoming); op ==
 * PLEX_OP_SYNC appends SYNC(incoming).  resident == incoming gives no
 * transfer.  Fills n_ops/ops/op_jobs and resident_before/after (mode = NONE).
 * plex_transition_plan and plex_group_transition use this same decision. */
PLEX_API plex_status plex_transition_decide(int64_t resident, int64_t incoming, int32_t op, plex_transition* out);

/* ---- a1 + a2: transition decision and plan (pure host, no CUDA calls) ----- */
/* Deterministic: identical requests give identical plans on every rank.
 * Errors: E_INVAL (bad request), E_LAYOUT (non-divisible destination). */
PLEX_API plex_status plex_transition_plan(const plex_plan_req* req, plex_plan_t* out);
PLEX_API plex_status plex_plan_destroy(plex_plan_t plan);
PLEX_API plex_status plex_plan_query(plex_plan_t plan, plex_plan_stats* out);
PLEX_API plex_status plex_plan_rank_info(plex_plan_t plan, int32_t rank, plex_rank_info* out);
PLEX_API plex_status plex_plan_segment(plex_plan_t plan, int32_t rank, int32_t i, plex_seg_desc* out);
PLEX_API plex_status plex_plan_dst_tensor(plex_plan_t plan, int32_t rank, int32_t i, plex_dst_desc* out);
/* Name of destination group `group` (PLEX_ROLE_AUTO plans: the fused rollout
 * tensor name, e.g. "model.layers.0.self_attn.qkv_proj.weight"; explicit-role
 * plans: the key of the group's first tensor).  Copies at most cap-1 bytes +
 * NUL into buf; *len = full length.  Also: *role / *n_experts of the group
 * (n_experts = experts stacked in an EXPERT group, else 0); any out may be NULL. */
PLEX_API plex_status plex_plan_group(plex_plan_t plan, int32_t group, char* buf, int32_t cap, int32_t* len,
                                     int32_t* role, int32_t* n_experts);
/* FSDP rows [row0, row1) of tensor t held by `rank` (R2; empty when row0 == row1). */
PLEX_API plex_status plex_plan_shard_rows(plex_plan_t plan, int32_t rank, int32_t t, int64_t* row0, int64_t* row1);
/* i-th carried bucket of the plan (0 <= i < plex_plan_n_carry). */
PLEX_API plex_status plex_plan_n_carry(plex_plan_t plan, int32_t* n);
PLEX_API plex_status plex_plan_carry(plex_plan_t plan, int32_t i, plex_carry_desc* out);
/* bytes[r * world + g]: bf16 bytes source rank r contributes to rollout rank g
 * (diagonal = local).  The zero-redundancy ledger of PAPER.md:576. */
PLEX_API plex_status plex_plan_ledger(plex_plan_t plan, uint64_t* bytes, int32_t n);
/* PLEX_PLAN_REPLICA_PARAM: byte offset of tensor t's bf16 replica in the param
 * arena (t < 0: only *arena_bytes), and the arena size.  E_INVAL for plans
 * without the flag. */
PLEX_API plex_status plex_plan_param_arena(plex_plan_t plan, int32_t t, uint64_t* offset, uint64_t* arena_bytes);

/* ---- lifecycle ------------------------------------------------------------ */
/* 128-byte NCCL unique id for bootstrapping (rank 0 calls it and broadcasts). */
PLEX_API plex_status plex_nccl_unique_id(void* out128);
/* device: CUDA ordinal.  staging: caller-owned device buffer of
 * staging_bytes >= n_slots * bucket_bytes of every plan used with this ctx.
 * workspace: caller-owned device buffer (256-B aligned, >= 1 MiB) holding the
 * library's device metadata for the ctx's lifetime: per plan used with the
 * ctx about 32 B per segment + 16 B per 64 KiB slab work item + 40 B per push
 * item + 48 B per segment of checksums (a Qwen2.5-7B FSDP-1 plan: ~45 MB, ~71 MB with elision);
 * freed when the plan is destroyed.  A call that would overflow it fails with
 * PLEX_E_TIER_FULL (nothing moved).  E_INVAL for a NULL / misaligned / too
 * small workspace.
 * pack_stream / copy_stream: caller-owned cudaStream_t (side streams).
 * nccl_id: 128 B from plex_nccl_unique_id, or NULL when world == 1 (or for a
 * ctx used only for single-process per-rank emulation).  Collective over
 * `world` ranks when nccl_id != NULL. */
PLEX_API plex_status plex_ctx_create(int32_t device, void* staging, uint64_t staging_bytes, void* workspace,
                                     uint64_t workspace_bytes, int32_t n_slots, void* pack_stream, void* copy_stream,
                                     const void* nccl_id, int32_t rank, int32_t world, uint32_t flags,
                                     plex_ctx_t* out);
/* Device workspace bytes in use now and at most since creation. */
PLEX_API plex_status plex_ctx_workspace(plex_ctx_t ctx, uint64_t* in_use, uint64_t* high_water);
PLEX_API plex_status plex_ctx_destroy(plex_ctx_t ctx);
/* NEXT-1 host-link balancing: caller-owned device buffer of >= 4 x bucket
 * bytes (256-B aligned) used to stage carried buckets (plans built with
 * link_weights).  With carried buckets, offload / onload / switch become
 * collective over the ctx's NCCL world (every rank calls them with the same
 * plan). */
PLEX_API plex_status plex_ctx_set_carry_staging(plex_ctx_t ctx, void* staging, uint64_t bytes);
PLEX_API plex_status plex_ctx_stats(plex_ctx_t ctx, int32_t which, plex_kernel_stats* out);
/* flags = (flags & ~mask) | (value & mask); only PLEX_CTX_TIMING and
 * PLEX_CTX_SPLIT_PUSH may change after creation (E_INVAL otherwise). */
PLEX_API plex_status plex_ctx_set_flags(plex_ctx_t ctx, uint32_t value, uint32_t mask);
PLEX_API plex_status plex_ctx_reset_stats(plex_ctx_t ctx);
/* Per-launch records behind plex_ctx_stats (PLEX_CTX_TIMING), oldest first,
 * since the last reset; *n = how many exist (copies min(cap, *n)). */
PLEX_API plex_status plex_ctx_trace(plex_ctx_t ctx, plex_launch_record* out, int32_t cap, int32_t* n);

/* Pinned host slab for `rank`'s state under `plan` (exact size; PAPER.md:574
 * "the host tier uses pinned memory").  Initial residency: DEVICE.
 * Errors: E_TIER_FULL if pinning fails. */
PLEX_API plex_status plex_slab_create(plex_plan_t plan, int32_t rank, uint32_t flags, plex_slab_t* out);
PLEX_API plex_status plex_slab_destroy(plex_slab_t slab);
/* host_ptr: the slab bytes (read/write, for verification and fault injection) */
PLEX_API plex_status plex_slab_info(plex_slab_t slab, void** host_ptr, uint64_t* bytes, int32_t* residency);
/* NEXT-4 cold tier (PAPER.md:505-506 GPU/host/NVMe residency; :574 "the NVMe
 * tier bypasses the page cache through direct I/O"): write a HOST-resident
 * slab's bytes to `path` with O_DIRECT using `threads` parallel writers, fsync,
 * and release its pinned memory (residency DISK).  fill re-pins, reads the
 * file back (residency HOST); onload then verifies the recorded checksums.
 * E_STATE on a wrong residency, E_INVAL if the file cannot be opened with
 * O_DIRECT, E_TIER_FULL on I/O or pinning failure (state unchanged). */
PLEX_API plex_status plex_slab_spill(plex_slab_t slab, const char* path, int32_t threads);
PLEX_API plex_status plex_slab_fill(plex_slab_t slab, const char* path, int32_t threads);
/* The pinned carry region holding other ranks' carried buckets (carry_offset
 * of plex_carry_desc), NULL / 0 if this rank carries none. */
PLEX_API plex_status plex_slab_carry(plex_slab_t slab, void** host_ptr, uint64_t* bytes);
/* *elided = 1 if the last offload elided the derived PARAM buckets. */
PLEX_API plex_status plex_slab_elided(plex_slab_t slab, int32_t* elided);
/* out[2*i], out[2*i+1] = (S1, S2) of segment i recorded at offload (R14). */
PLEX_API plex_status plex_slab_checksums(plex_slab_t slab, uint64_t* out, int32_t n);

/* ---- a3 + a4: suspend ----------------------------------------------------- */
/* src[kind * n_tensors + t] = device pointer of this rank's contiguous shard
 * of tensor t (kind in the plan's kind_mask and t in its subset; others may
 * be NULL).  Gather-packs every segment into staging buckets (fused R14
 * checksums), D2H-copies each bucket into the slab at its canonical offset,
 * double-buffered on (pack, copy) streams.  Ordered after prior work on
 * `caller_stream`; returns when the slab holds the canonical bytes (host
 * blocking).  Residency -> HOST.  Idempotent (no-op) when already HOST. */
PLEX_API plex_status plex_state_offload(plex_ctx_t ctx, plex_plan_t plan, const void* const* src, int32_t n_src,
                               plex_slab_t slab, void* caller_stream);

/* ---- a6 + a7: resume ------------------------------------------------------ */
/* dst: same indexing as offload's src, caller-(re)allocated with the plan's
 * shard shapes.  H2D-copies buckets and scatter-unpacks them, recomputing
 * the checksums; returns PLEX_E_CHECKSUM (residency stays HOST) if any
 * segment differs from what offload recorded.  Residency -> DEVICE.
 * Idempotent (no-op) when already DEVICE; E_STATE if the slab was never
 * written. */
PLEX_API plex_status plex_state_onload(plex_ctx_t ctx, plex_plan_t plan, plex_slab_t slab, void* const* dst,
                              int32_t n_dst, void* caller_stream);

/* ---- NEXT-1: scheduler-directed prefetch and asynchronous drain ------------ */
/* PAPER.md:506 ("when an upcoming context switch is predicted, StateManager
 * can proactively move state upward in the hierarchy") and :513 ("state can be
 * prefetched or drained across the memory hierarchy asynchronously", keeping
 * only operations on the active deployment on the critical path).
 * plex_state_drain = plex_state_offload and plex_state_prefetch =
 * plex_state_onload, except that they return as soon as the transfer is
 * enqueued on library-owned side streams (ordered after prior work on
 * caller_stream) so the caller keeps computing; the source (drain) / the
 * destination (prefetch) must not be touched until plex_state_wait.  One drain
 * and one prefetch may be in flight per ctx (they use the two staging halves:
 * staging >= 2 x n_slots x bucket); blocking state transfers on the ctx return
 * E_STATE meanwhile, plex_weight_sync does not.  plex_state_wait(op =
 * PLEX_OP_OFFLOAD | PLEX_OP_ONLOAD) host-blocks until that transfer is done,
 * makes caller_stream wait on it, and flips residency (prefetch: verifies the
 * R14 checksums first, E_CHECKSUM leaves the slab HOST); a no-op if nothing is
 * in flight.  plex_state_poll sets *done without blocking. */
PLEX_API plex_status plex_state_drain(plex_ctx_t ctx, plex_plan_t plan, const void* const* src, int32_t n_src,
                                      plex_slab_t slab, void* caller_stream);
PLEX_API plex_status plex_state_prefetch(plex_ctx_t ctx, plex_plan_t plan, plex_slab_t slab, void* const* dst,
                                         int32_t n_dst, void* caller_stream);
PLEX_API plex_status plex_state_wait(plex_ctx_t ctx, int32_t op, void* caller_stream);
PLEX_API plex_status plex_state_poll(plex_ctx_t ctx, int32_t op, int32_t* done);

/* ---- NEXT-1: duplex switch (offload A || onload B) ------------------------ */
/* The context switch of PAPER.md:555 (OFFLOAD resident A, ONLOAD incoming B)
 * as one call whose two halves run concurrently: A's buckets go D2H on
 * ctx's copy stream while B's come H2D on a second, library-owned copy
 * stream, so the switch costs ~max(T_offload, T_load) instead of the sum
 * C_setup = T_offload + T_load of Eq. 3.  src_out/dst_in
 * as in plex_state_offload/onload (each half skipped if already done).  Needs
 * staging >= n_slots x (bucket_out + bucket_in).  Blocking; residencies flip
 * per half on success; E_CHECKSUM if B fails verification (B stays HOST, A
 * is HOST and its slab valid). */
PLEX_API plex_status plex_state_switch(plex_ctx_t ctx, plex_plan_t plan_out, const void* const* src_out, int32_t n_src,
                                       plex_slab_t slab_out, plex_plan_t plan_in, plex_slab_t slab_in,
                                       void* const* dst_in, int32_t n_dst, void* caller_stream);

/* NEXT-1 in-place swap (PAPER.md:555 context switch, R17 one resident job):
 * the resident job's state (state pointers, plex_state_offload layout) and the
 * incoming job's state (in `slab`, HOST-resident, offloaded under the same
 * plan) trade places.  On return the tensors hold the incoming state (checksum
 * verified) and the slab holds the outgoing state with its checksums.  Both
 * host-link directions run at once through the two staging rings (like
 * plex_state_switch), but only ONE device copy and ONE pinned slab exist: per
 * bucket, the outgoing pack reads a tensor range before the incoming unpack
 * overwrites it (same kernel stream) and the outgoing D2H overwrites a slab
 * range only after the incoming H2D has read it (both copies of a bucket run
 * in up to 8 pieces, each D2H piece waiting only for its own H2D piece, so
 * the head and tail buckets overlap too).  Staging >= 2 x n_slots x
 * bucket.  Blocking, caller-stream ordered.  With PLEX_PLAN_ELIDE_PARAM: an
 * elided incoming slab and a derivable outgoing job both walk the shifted
 * grid (no param byte moves); an elided incoming slab and a non-derivable
 * outgoing job first store the outgoing PARAM prefix (slab bytes the
 * incoming state does not use); a fully stored incoming slab makes the
 * outgoing job go in full.  E_STATE if the slab holds no offloaded state;
 * E_INVAL for carried-bucket plans.  On
 * E_CHECKSUM the slab already holds the outgoing state (safe) and the tensors'
 * contents are unspecified. */
PLEX_API plex_status plex_state_swap(plex_ctx_t ctx, plex_plan_t plan, void* const* state, int32_t n_state,
                                     plex_slab_t slab, void* caller_stream);

/* ---- a8 - a11: train -> rollout weight sync ------------------------------- */
/* Collective over the ctx's world.  src_master[t] = this rank's fp32 master
 * shard of tensor t (FSDP-world rows).  dst_arena = this rank's bf16 rollout
 * arena (plan dst_arena_bytes; tensors at plex_plan_dst_tensor offsets).
 * Writes exactly fuse_g(slice_g(RNE(concat_r shard_r(master)))) (DESIGN.md
 * c1.3) into every rank's arena: each source rank casts its own rows once per
 * destination and stores them straight into the destination arena over
 * NVLink (peer-mapped), so no byte is sent twice. */
PLEX_API plex_status plex_weight_sync(plex_ctx_t ctx, plex_plan_t plan, const void* const* src_master, int32_t n_src,
                             void* dst_arena, void* caller_stream);
/* One source rank's share of the sync into explicitly given destination arenas
 * (dst_arenas[g], g < world; device pointers valid on ctx's device).  Not
 * collective, no barriers: used for single-GPU emulation of a W-rank group
 * and by plex_weight_sync itself.  Ordered on stream, blocking. */
PLEX_API plex_status plex_weight_sync_rank(plex_ctx_t ctx, plex_plan_t plan, int32_t rank, const void* const* src_master,
                                  int32_t n_src, void* const* dst_arenas, int32_t n_arenas, void* stream);

/* ---- a1 executed: the GPU group's residency authority ---------------------- */
/* PAPER.md:555 ("the scheduler maintains a map (group_executor_gpu_job)
 * tracking the Job ID currently resident on each GPU group ... If they differ,
 * the system automatically prepends offload and load operations") and :506
 * (StateManager, the "single node-local authority over residency").  A group
 * lives on one ctx (this rank's GPU of the group); every rank of the group
 * keeps its own group object and calls the same transitions in the same order.
 *
 * Storage (a5): the library never allocates device memory.  `storage` is
 * called to (re)acquire a job's device state before an onload (acquire = 1:
 * allocate and write the PLEX_NUM_KINDS x n_tensors pointer table into
 * `state`, same layout as plex_state_offload's src) and to release it after an
 * offload (acquire = 0).  It returns 0 on success, nonzero when the memory
 * cannot be acquired (then the executor switches sequentially: offload and
 * release the resident job first).  NULL storage = device state is never
 * released (pointer tables given at plex_group_add_job stay valid). */
typedef struct plex_group_s* plex_group_t;
typedef int32_t (*plex_storage_fn)(void* user, int64_t job, int32_t acquire, void** state, int32_t n_state);

PLEX_API plex_status plex_group_create(plex_ctx_t ctx, plex_storage_fn storage, void* user, plex_group_t* out);
PLEX_API plex_status plex_group_destroy(plex_group_t group);

/* Register job `job` (>= 0, unique) with its plan and pinned slab (NULL only
 * for a swap partner that never leaves the device alone: see storage_id).
 *   flags & PLEX_GROUP_RESIDENT: the job's state is on the device now (state =
 *     its pointer table; at most one resident job per group, R17); else the
 *     job is HOST-resident: slab must hold its offloaded state.
 *   state / n_state: pointer table of already-allocated device storage (or
 *     NULL: acquired through `storage` at its first onload).
 *   storage_id >= 0: jobs with equal ids share ONE set of device tensors
 *     (same plan required); switches between them are in-place swaps
 *     (plex_state_swap) and the pair's slab moves with the state.  -1 = own
 *     storage.
 * Errors: E_INVAL (duplicate id, plan of another world, bad table, replica
 * plans on a ctx without NCCL), E_STATE (second resident job, HOST job whose
 * slab holds no state). */
#define PLEX_GROUP_RESIDENT 0x1u
PLEX_API plex_status plex_group_add_job(plex_group_t group, int64_t job, plex_plan_t plan, plex_slab_t slab,
                                        int64_t storage_id, uint32_t flags, void* const* state, int32_t n_state);
/* *job = the job resident on the group (-1 = none). */
PLEX_API plex_status plex_group_resident(plex_group_t group, int64_t* job);
/* The slab currently holding `job`'s offloaded state (swaps move slabs). */
PLEX_API plex_status plex_group_job_slab(plex_group_t group, int64_t job, plex_slab_t* slab);

/* Run operation `op` (PLEX_OP_NONE, or PLEX_OP_SYNC for a weight sync) of job
 * `incoming` on the group: decides the ops with plex_transition_decide, then
 * executes them, choosing per switch
 *   SWAP        the two jobs share device storage (plex_state_swap);
 *   DUPLEX      the incoming job's storage can be acquired while the resident
 *               one is still on the device and staging holds both rings
 *               (plex_state_switch; then the outgoing storage is released);
 *   SEQUENTIAL  otherwise (offload, release, acquire, onload).
 * Replicated-param plans (PLEX_PLAN_REPLICA_PARAM) are all-gathered after
 * their onload.  SYNC: n_arenas == 1 -> collective plex_weight_sync into
 * dst_arenas[0]; n_arenas == world -> this rank's share into every given
 * arena (plex_weight_sync_rank, single-process emulation).  Blocking,
 * ordered after prior work on caller_stream.  *out (may be NULL) reports the
 * ops, the mode and the residency.  On error the group's map follows the
 * slabs (a failed onload leaves no job resident; E_CHECKSUM keeps the
 * outgoing state safe in its slab).  Plans with carried buckets must not fail
 * to acquire storage (E_TIER_FULL instead of a per-rank fallback, so that
 * every rank takes the same collective path). */
PLEX_API plex_status plex_group_transition(plex_group_t group, int64_t incoming, int32_t op, void* const* dst_arenas,
                                           int32_t n_arenas, void* caller_stream, plex_transition* out);

/* ---- NEXT-3: checkpoint materialisation from the offloaded state ---------- */
/* a checkpoint is a materialisation of managed (possibly
 * offloaded) state, written in the background off the critical path.  Writes
 * the HOST-resident slab of `plan` (rank = the slab's) to `path` as a standard
 * safetensors file: one tensor per slab segment in slab order, named by its
 * logical key (PARAM, BF16) or "optimizer.<master|exp_avg|exp_avg_sq>.<key>"
 * (F32), shaped as the rank's FSDP shard (R2), no padding; header metadata
 * "plex.world", "plex.rank", "plex.layout" and "plex.checksums" (the R14
 * (S1, S2) pairs recorded at offload, 16 hex digits each).  `threads` writers
 * at disjoint offsets, then fsync.  Host-only (no CUDA call), safe to run on
 * another thread while the job resumes from the same slab: the slab is
 * read-only meanwhile (offload into it, spill, restore -> E_STATE; onload and
 * sync-from-slab proceed).  E_STATE if the slab is not HOST-resident or holds elided
 * params; E_INVAL for plans that carry this rank's buckets; E_TIER_FULL on I/O
 * errors. */
PLEX_API plex_status plex_slab_checkpoint(plex_plan_t plan, plex_slab_t slab, const char* path, int32_t threads);
/* The same write on a library-owned background thread.  All checks run, and
 * the slab becomes read-only, in the calling thread before this returns, so a
 * swap / offload / restore issued right after it is refused (E_STATE) until
 * plex_ckpt_wait; onload and sync-from-slab may proceed.  *out is released by
 * plex_ckpt_wait, which joins the writer and returns its status (message via
 * plex_last_error). */
PLEX_API plex_status plex_slab_checkpoint_start(plex_plan_t plan, plex_slab_t slab, const char* path, int32_t threads,
                                                plex_ckpt_t* out);
PLEX_API plex_status plex_ckpt_wait(plex_ckpt_t ckpt);
/* Inverse: fill an idle slab of `plan` from a checkpoint written by
 * plex_slab_checkpoint for the same plan and rank; residency becomes HOST with
 * the file's checksums, so the next onload verifies every tensor
 * (E_CHECKSUM on corrupted data).  E_LAYOUT if the header is not exactly what
 * this plan/rank writes (other names, shapes, order or sizes) -- the slab is
 * then untouched; on an I/O error the slab holds no state (onload -> E_STATE). */
PLEX_API plex_status plex_slab_restore(plex_plan_t plan, plex_slab_t slab, const char* path, int32_t threads);

/* ---- NEXT-2: replicated-param restore (PLEX_PLAN_REPLICA_PARAM) ----------- */
/* Collective over the ctx's world.  param_arena = this rank's bf16 param
 * arena (plex_plan_param_arena layout) whose own FSDP rows of every tensor
 * in the plan's key subset are valid (e.g. just onloaded).  Every rank stores
 * its own rows straight into every peer's arena over NVLink (peer-mapped),
 * so on return every arena holds the full replicated params; each row is
 * sent once to each peer (the all-gather of PAPER.md:508's deduplicated
 * state).  Ordered after prior work on caller_stream; blocking. */
PLEX_API plex_status plex_param_allgather(plex_ctx_t ctx, plex_plan_t plan, void* param_arena, void* caller_stream);
/* One rank's share into explicitly given arenas (arenas[g], g < world, on
 * ctx's device): single-GPU emulation counterpart, not collective. */
PLEX_API plex_status plex_param_allgather_rank(plex_ctx_t ctx, plex_plan_t plan, int32_t rank, void* const* arenas,
                                               int32_t n_arenas, void* stream);

/* ---- NEXT-3: sync from the offloaded canonical state ---------------------- */
/* The sync of a SUSPENDED job, materialised "directly from managed memory"
 * (PAPER.md:510, :576): each rank's fp32 master rows are read by the push
 * kernel straight from its pinned slab (zero-copy over the host link) instead
 * of device shards.  slab: this rank's HOST-resident slab of `plan` carrying
 * MASTER for every tensor (E_STATE if not offloaded, E_INVAL if a tensor is
 * missing).  Output, collectives and blocking contract as plex_weight_sync. */
PLEX_API plex_status plex_weight_sync_from_slab(plex_ctx_t ctx, plex_plan_t plan, plex_slab_t slab, void* dst_arena,
                                                void* caller_stream);
/* Single-process emulation counterpart of plex_weight_sync_rank. */
PLEX_API plex_status plex_weight_sync_rank_from_slab(plex_ctx_t ctx, plex_plan_t plan, int32_t rank, plex_slab_t slab,
                                                     void* const* dst_arenas, int32_t n_arenas, void* stream);

/* ---- infrastructure (synthetic inputs / verification; not the method) ---- */
/* K6: counter-based generator of DESIGN.md §3 (D2) writing `count` elements of
 * the logical tensor `key` starting at logical flat index `index_base`. */
PLEX_API plex_status plex_synth_fill(void* dst, int32_t kind, uint64_t seed, const char* key, uint64_t index_base,
                            uint64_t count, int32_t special_bits, void* stream);
/* Multiplex "training step": bits ^= mutation(job_seed, step, key, kind, i) (o10). */
PLEX_API plex_status plex_synth_mutate(void* buf, int32_t kind, uint64_t job_seed, uint64_t step, const char* key,
                              uint64_t index_base, uint64_t count, void* stream);
/* K7: accumulate (S1, S2) of R14 over `count` elements of size `esize` (2|4)
 * into dev_out[0..1] (device, caller zeroes). */
PLEX_API plex_status plex_checksum(const void* src, int32_t esize, uint64_t index_base, uint64_t count,
                          uint64_t* dev_out, void* stream);
/* fp32 -> bf16 RNE of `count` contiguous elements (the a8 cast on its own). */
PLEX_API plex_status plex_cast_rne(const void* src_f32, void* dst_bf16, uint64_t count, void* stream);

/* ---- diagnostics (kernel measurement; not part of the method) ------------ */
/* Launch ONE K1 (mode bit 0 set) or K2 (bit 0 clear) kernel over bucket
 * `bucket` of ctx's rank of `plan`, between `state` (4 x n_tensors device
 * pointers, as plex_state_offload) and staging slot 0, on `stream`, with no
 * copy, no checksum verification and no residency change: the kernel as the
 * bucket pipeline launches it, timed on its own by tools/pack_insitu.py.  The
 * bucket's staging bytes start `staging_offset` bytes into the ctx's staging
 * buffer (256-B aligned; E_INVAL past its end).  The pointer table is uploaded first (a small H2D on `stream`) unless mode bit 1
 * is set (the previous diag call on this ctx uploaded the same table).  The
 * staging bytes (pack) or the state bytes (unpack) are overwritten.  E_INVAL
 * for a bucket out of range; E_STATE while an async prefetch/drain is in
 * flight on the ctx (it shares the staging ring and work counters). */
PLEX_API plex_status plex_diag_pack(plex_ctx_t ctx, plex_plan_t plan, const void* const* state, int32_t n_state,
                                    int32_t bucket, int32_t mode, uint64_t staging_offset, void* stream);
/* Select the K1/K2 build for every later launch in this process: 0 = default,
 * 1 = the same kernel with L2::evict_first cache policies on its bulk copies
 * (measurement of L2 residency effects).  E_INVAL for another value. */
PLEX_API plex_status plex_diag_pack_variant(int32_t variant);

#ifdef __cplusplus
}
#endif
#endif /* PLEX_H */
