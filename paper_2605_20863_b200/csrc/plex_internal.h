// Internal structures shared by the planner, runtime and kernels of libplex.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/plex.h"

namespace plex {

constexpr uint64_t kSegAlign = 256;                 // R4
constexpr uint64_t kDefaultBucket = 64ull << 20;    // R5
constexpr uint64_t kDefaultTile = 64ull << 10;

inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }
inline int kind_esize(int kind) { return kind == PLEX_KIND_PARAM ? 2 : 4; }

void set_error(const char* fmt, ...);

// ---- device-visible records (POD; uploaded as tables) ----------------------
// One slab segment: a (tensor, kind) shard at a 256-B-aligned slab offset.
struct SegDev {
    uint64_t slab_off;
    uint64_t bytes;
    uint64_t index_base;   // logical flat index of the shard's first element
    uint32_t ptr_slot;     // kind * n_tensors + tensor
    uint32_t esize;        // 2 | 4
};
static_assert(sizeof(SegDev) == 32, "SegDev layout");

// One pack/unpack work item: slab bytes [slab_lo, slab_lo + len) of segment
// `seg`'s slot (its bytes followed by its zero padding), inside one bucket.
struct PackItem {
    uint64_t slab_lo;
    uint32_t len;
    uint32_t seg;
};
static_assert(sizeof(PackItem) == 16, "PackItem layout");

// One reshard-push work item: a rows x cols fp32 rectangle of source tensor
// `tensor`'s local master shard (row stride src_stride elements) cast to bf16
// and stored at element dst_elem of rank dst_rank's arena (row stride
// dst_stride elements).
struct PushItem {
    uint64_t src_elem;
    uint64_t dst_elem;
    uint32_t tensor;
    uint32_t dst_rank;
    uint32_t rows;
    uint32_t cols;
    uint32_t src_stride;
    uint32_t dst_stride;
};
static_assert(sizeof(PushItem) == 40, "PushItem layout");

// ---- host plan ---------------------------------------------------------------
struct Tensor {
    std::string key;
    int64_t d0, d1;
    int32_t ndim, role, group, slot, expert, unit;
};

struct Piece {           // source rectangle placed into a destination tensor
    int32_t tensor;
    int64_t r0, r1, c0, c1;
    int64_t dst_row0;
};

struct DstTensor {
    int32_t group;
    int32_t first_tensor;
    uint64_t arena_off;
    int64_t rows, cols;
    std::vector<Piece> pieces;
};

struct RankPlan {
    // slab
    std::vector<SegDev> segs;
    std::vector<plex_seg_desc> seg_desc;
    std::vector<PackItem> items;
    std::vector<uint64_t> bucket_item_start;    // n_buckets + 1
    uint64_t slab_bytes = 0, payload_bytes = 0;
    // NEXT-2 derived-param elision: the PARAM prefix [0, elide_start) is derived
    // on the device; the rest moves on its own bucket grid starting there.
    uint64_t elide_start = 0;                   // 0 = no elision possible
    uint64_t n_param_items = 0;                 // items[0, n) cover [0, elide_start)
    std::vector<PackItem> items_el;             // items of [elide_start, slab_bytes)
    std::vector<uint64_t> bstart_el;            // n_buckets_el + 1
    // rollout
    std::vector<DstTensor> dst;
    uint64_t arena_bytes = 0;
    std::vector<PushItem> push;                 // items whose source is this rank
    std::vector<char> carried;                  // per own bucket: moved by another rank's host link
    int32_t carried_out = 0, carried_in = 0;
    uint64_t carry_bytes = 0;
    uint64_t send_bytes = 0, recv_bytes = 0, local_bytes = 0, src_read_bytes = 0;
    // NEXT-2 replicated params: this rank's rows of every param pushed to every peer
    std::vector<PushItem> gather;
    uint64_t gather_send = 0, gather_recv = 0;
};

struct CarryXfer {       // a whole bucket of `owner`'s slab moved through `carrier`'s host link
    int32_t owner, bucket, carrier;
    uint64_t lo, len;    // owner slab byte range
    uint64_t coff;       // offset in the carrier's carry region
};

struct Plan {
    std::vector<Tensor> tensors;
    std::vector<CarryXfer> carry;               // global, sorted by (owner, bucket)
    int32_t world = 1, tp = 0, dp = 0, ep = 1, rank_map = 0, layout = 0;
    uint32_t kind_mask = PLEX_KINDMASK_ALL;
    uint64_t bucket = kDefaultBucket, tile = kDefaultTile;
    uint32_t flags = 0;
    std::vector<int32_t> subset;                // sorted tensor indices in the slab
    std::vector<RankPlan> ranks;
    std::vector<uint64_t> ledger;               // world * world
    std::vector<uint64_t> param_off;            // PLEX_PLAN_REPLICA_PARAM: param arena offsets
    uint64_t param_arena_bytes = 0;
    plex_plan_stats stats{};
    uint64_t id = 0;                            // unique per plan (device cache key)
    // destination groups (index = group id): name, role, experts stacked (EXPERT)
    std::vector<std::string> group_names;
    std::vector<int32_t> group_role, group_experts;
};

// What the group executor needs to know about a ctx (plex_runtime.cu).
struct CtxInfo {
    uint64_t staging_bytes;
    int32_t n_slots, rank, world, device;
    bool has_comm;
};
void ctx_query(plex_ctx_t c, CtxInfo* out);

// a1: the op list of one transition.
void transition_ops(int64_t resident, int64_t incoming, int32_t op, plex_transition* out);

inline int32_t n_buckets(const Plan& p, const RankPlan& r) {
    return (int32_t)((r.slab_bytes + p.bucket - 1) / p.bucket);
}

}  // namespace plex

struct plex_plan_s {
    plex::Plan p;
};
