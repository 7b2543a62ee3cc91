// libplex runtime: context, pinned slabs, the suspend/resume bucket pipeline
// and the train->rollout weight sync (fused NVLink push, or the NCCL baseline).
//
// Blocking contract (§5.3): every state-transfer call orders
// itself after prior work on the caller's stream, runs on the ctx's side
// streams, and returns only when the transfer has completed, with the caller
// stream made to wait on it ("resident and safe to use on the default CUDA
// stream").
#include <cuda_runtime.h>
#include <nccl.h>
#include <errno.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <thread>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "plex_heap.h"
#include "plex_internal.h"

namespace plex {

cudaError_t launch_pack(bool pack, const PackItem* items, uint32_t n_items, const SegDev* segs, const uint64_t* ptrs,
                        uint8_t* staging, uint64_t bucket_lo, unsigned long long* cks, unsigned int* ctr,
                        cudaStream_t s);
void set_pack_variant(int v);
cudaError_t launch_verify(const unsigned long long* got, const unsigned long long* want, uint32_t n, int* bad,
                          cudaStream_t s);
cudaError_t launch_push(bool cast, const PushItem* items, uint64_t n_items, const uint64_t* src_ptrs,
                        const uint64_t* dst_arenas, cudaStream_t s);
cudaError_t launch_cast(const void* src, void* dst, uint64_t n, cudaStream_t s);
cudaError_t launch_synth(void* dst, int kind, uint64_t base, uint64_t index_base, uint64_t n, int special_bits,
                         cudaStream_t s);
cudaError_t launch_mutate(void* buf, int esize, uint64_t base, uint64_t index_base, uint64_t n, cudaStream_t s);
cudaError_t launch_checksum(const void* src, int es, uint64_t index_base, uint64_t n, unsigned long long* out,
                            cudaStream_t s);
cudaError_t launch_signal(unsigned long long* flag, unsigned long long v, cudaStream_t s);
cudaError_t launch_wait(const unsigned long long* flag, unsigned long long v, unsigned long long timeout_ns, int* err,
                        cudaStream_t s);
cudaError_t launch_derive(bool check, const PackItem* items, uint32_t n_items, const SegDev* segs, const uint64_t* ptrs,
                          uint32_t n_tensors, unsigned long long* cks, int* bad, cudaStream_t s);
// NCCL-baseline sync kernels (plex_nccl_sync.cu)
plex_status nccl_sync(plex_ctx_s* ctx, const Plan& p, const void* const* src, void* arena, cudaStream_t caller);

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            set_error("%s:%d %s: %s", __FILE__, __LINE__, #x, cudaGetErrorString(e_));         \
            (void)cudaGetLastError(); /* do not leak a handled error into the next launch */   \
            return PLEX_E_CUDA;                                                                \
        }                                                                                      \
    } while (0)
#define NK(x)                                                                                  \
    do {                                                                                       \
        ncclResult_t r_ = (x);                                                                 \
        if (r_ != ncclSuccess) {                                                               \
            set_error("%s:%d %s: %s", __FILE__, __LINE__, #x, ncclGetErrorString(r_));         \
            return PLEX_E_NCCL;                                                                \
        }                                                                                      \
    } while (0)

// Device-side copy of one rank's share of a plan (built lazily per ctx).
struct DevPlan {
    SegDev* segs = nullptr;
    PackItem* items = nullptr;
    PushItem* push = nullptr;
    PushItem* gather = nullptr;               // NEXT-2 replicated-param all-gather items
    // PLEX_CTX_SPLIT_PUSH: the push items split by destination (built on first use)
    PushItem* push_local = nullptr;
    PushItem* push_remote = nullptr;
    uint64_t n_push_local = 0, n_push_remote = 0, push_local_elems = 0, push_remote_elems = 0;
    bool push_split = false;
    unsigned long long* cks = nullptr;        // computed (S1,S2) per segment
    unsigned long long* cks_want = nullptr;   // expected, uploaded at onload
    unsigned long long* cks_in = nullptr;     // recomputed at onload
    // pinned host mirrors of the checksum tables: a device<->pageable copy would
    // block the calling thread until the stream drains (async drain/prefetch)
    uint64_t* h_cks_out = nullptr;            // offload: recorded (S1,S2), read back here
    uint64_t* h_cks_want = nullptr;           // onload: expected (S1,S2), uploaded from here
    std::vector<uint64_t> bucket_payload;     // data bytes per bucket (stats)
    uint64_t elide_payload = 0;               // PARAM data bytes (derived when eliding)
    PackItem* items_el = nullptr;             // NEXT-2 shifted grid
    std::vector<uint64_t> bucket_payload_el;
    // NCCL-baseline schedule (built lazily for one per-pair round quota Q)
    uint64_t nq = 0;                          // Q it was built for (0 = none)
    int rounds = 0;
    PushItem* local = nullptr;                // local rectangles: cast straight into the arena
    uint64_t n_local = 0, local_bytes = 0;
    PushItem* rpack = nullptr;                // K4: cast into send segments, per round
    PushItem* runpack = nullptr;              // K5: receive segments -> arena, per round
    std::vector<uint64_t> rpack_start, runpack_start;   // rounds + 1
    std::vector<uint64_t> rpack_bytes, runpack_bytes;   // algorithmic bytes per round
    std::vector<uint64_t> send_bytes, recv_bytes;       // rounds * world
};

struct Timed {
    int which;
    uint64_t bytes;
    cudaEvent_t a, b;
};

struct AsyncState;   // an in-flight plex_state_drain / plex_state_prefetch

constexpr uint64_t kMinWorkspace = 1ull << 20;
constexpr uint64_t kSwapPieces = 16;    // copies per bucket in the in-place swap (at most)
constexpr uint64_t kSwapPiecesDefault = 8;   // sweep 2 / 4 / 8 / 16: profiles/r02r_*
// Measurement knob: PLEX_SWAP_PIECES=n (1..16; 1 = whole-bucket copies) for
// A/B runs of the piecewise swap on one box; read once.
static uint64_t swap_pieces() {
    static const uint64_t v = [] {
        const char* e = std::getenv("PLEX_SWAP_PIECES");
        const long x = e ? std::strtol(e, nullptr, 10) : (long)kSwapPiecesDefault;
        return (uint64_t)std::min<long>((long)kSwapPieces, std::max<long>(1, x));
    }();
    return v;
}

// Device metadata lives in the caller's workspace (plex_ctx_create): the
// library never calls cudaMalloc (SURVEY §8(b) ownership).  OffsetHeap
// (plex_heap.h) hands out 256-B aligned offsets into [base, base + bytes).
struct DevHeap {
    uint8_t* base = nullptr;
    OffsetHeap h;
    std::mutex mu;
};

}  // namespace plex

using namespace plex;

struct plex_ctx_s {
    int device = 0;
    uint8_t* staging = nullptr;
    uint64_t staging_bytes = 0;
    int n_slots = 2;
    cudaStream_t pack = nullptr, copy = nullptr;
    int rank = 0, world = 1;
    uint32_t flags = 0;
    ncclComm_t comm = nullptr;
    // events
    cudaEvent_t ev_caller = nullptr, ev_pack_done = nullptr, ev_copy_done = nullptr;
    std::vector<cudaEvent_t> ev_pack, ev_copy;
    std::vector<cudaEvent_t> pool;
    size_t pool_used = 0;
    std::vector<Timed> pending;
    plex_kernel_stats stats[PLEX_NUM_STATS] = {};
    std::vector<plex_launch_record> trace;   // every timed launch since the last reset
    int32_t n_calls = 0;                     // timed blocking calls since the last reset
    // pointer tables (pinned host mirror -> device)
    uint64_t* h_ptrs = nullptr;
    uint64_t* d_ptrs = nullptr;
    size_t ptr_cap = 0;
    // second half of a duplex switch (NEXT-1): own pointer table, streams, events
    uint64_t* h_ptrs2 = nullptr;
    uint64_t* d_ptrs2 = nullptr;
    size_t ptr_cap2 = 0;
    cudaStream_t copy2 = nullptr;       // library-owned H2D stream of a duplex switch, created lazily
    // NEXT-1 async prefetch / drain: own kernel stream, D2H stream, ring events, pointer table
    cudaStream_t kasync = nullptr, copy3 = nullptr;
    std::vector<cudaEvent_t> ev_pack3, ev_copy3;
    uint64_t* h_ptrs3 = nullptr;
    uint64_t* d_ptrs3 = nullptr;
    size_t ptr_cap3 = 0;
    AsyncState* async[2] = {nullptr, nullptr};   // [0] drain (offload), [1] prefetch (onload)
    // NEXT-1 host-link balancing (carried buckets): caller-provided carry staging
    // (4 bucket slots: 0-1 offload direction, 2-3 onload direction), a kernel
    // stream, one NCCL stream for every carry send/recv, a carrier copy stream
    uint8_t* cstaging = nullptr;
    uint64_t cstaging_bytes = 0;
    cudaStream_t ckern = nullptr, cstream = nullptr, ccopy = nullptr;
    cudaEvent_t ev_cs[4] = {}, ev_cc[4] = {}, ev_cbeg = nullptr, ev_cend = nullptr;
    bool carry_used = false;            // the current blocking op enqueued carry work
    // peer-memory carry transport (default): handshake flags READY[4] FREE[4]
    // per rank (u64 sequence numbers) + a timeout flag; peers' carry staging
    // and flags mapped over CUDA IPC; one sequence epoch per carry phase
    unsigned long long* cflags = nullptr;
    int* cerr = nullptr;
    int* h_cerr = nullptr;
    std::vector<void*> peer_cstaging, peer_cflags;
    uint64_t cepoch = 0;
    std::vector<std::vector<unsigned long long>> carry_in_last;   // [owner][onload slot] last seq written
    std::vector<cudaEvent_t> ev_pack2, ev_copy2;
    std::vector<cudaEvent_t> ev_piece;  // in-place swap: H2D piece j of in-ring slot s done
    int* h_flag = nullptr;
    int* d_flag = nullptr;
    unsigned int* d_ctr = nullptr;      // pack/unpack work counters, one per pipe (+8: finished CTAs)
    // small device scratch for NCCL barriers and handle exchange
    uint8_t* d_scratch = nullptr;
    uint8_t* h_scratch = nullptr;
    size_t scratch_bytes = 0;
    // peer arenas opened over CUDA IPC: rank -> (peer's buffer id, mapped base)
    // peer mappings per (arena role, rank): role 0 = rollout arena, 1 = param arena
    std::map<int, std::pair<uint64_t, void*>> peers;
    // roles: 0 rollout arena, 1 param arena, 2 carry staging, 3 carry flags
    uint64_t my_buffer_id[4] = {0, 0, 0, 0};  // buffer last exported per role (and its cached handle)
    cudaIpcMemHandle_t my_handle[4]{};
    std::map<uint64_t, DevPlan> dev;    // plan id -> device tables
    cudaEvent_t ev_sync[6] = {};        // NCCL baseline: rpack / nccl / runpack x 2
    DevHeap heap;                       // caller's device workspace: every device table above
};

struct plex_ckpt_s {                   // a background checkpoint (plex_slab_checkpoint_start)
    std::thread th;
    plex_status status = PLEX_OK;
    std::string error;
};

struct plex_slab_s {
    uint64_t plan_id = 0;
    int rank = 0;
    uint64_t bytes = 0;
    uint8_t* host = nullptr;
    uint32_t flags = 0;        // PLEX_SLAB_* used to pin
    bool registered = false;   // mmap + cudaHostRegister path
    size_t map_bytes = 0;      // pinned bytes (>= bytes, 4 KiB / 2 MiB aligned)
    int residency = PLEX_RES_DEVICE;
    bool written = false;
    bool elided = false;                // NEXT-2: leading PARAM buckets derived, not stored
    std::atomic<bool> busy{false};      // an async drain / prefetch or a restore of this slab is in flight
    std::atomic<int> ckpt{0};           // checkpoints reading the slab (it is read-only meanwhile)
    std::mutex mu;                      // makes "start a checkpoint" and "start a restore" exclusive
    uint8_t* carry_host = nullptr;      // other ranks' carried buckets (pinned)
    uint64_t carry_bytes = 0;
    std::vector<uint64_t> cks;          // 2 per segment, recorded at offload
};

extern "C" {
static plex_status exchange_arenas(plex_ctx_s* c, int role, void* arena, std::vector<void*>& arenas);
}

namespace plex {

static std::mutex g_ctx_mu;
static std::set<plex_ctx_s*> g_ctxs;

static plex_status dev_alloc(plex_ctx_s* c, uint64_t n, void** out) {
    *out = nullptr;
    if (!n) return PLEX_OK;
    DevHeap& h = c->heap;
    std::lock_guard<std::mutex> lk(h.mu);
    const uint64_t off = h.h.alloc(n);
    if (off == OffsetHeap::kNone) {
        set_error("device metadata workspace exhausted: %llu B requested, %llu of %llu B in use "
                  "(pass a larger workspace to plex_ctx_create)", (unsigned long long)n,
                  (unsigned long long)h.h.in_use(), (unsigned long long)h.h.bytes());
        return PLEX_E_TIER_FULL;
    }
    *out = h.base + off;
    return PLEX_OK;
}

template <class T>
static plex_status dev_alloc_t(plex_ctx_s* c, uint64_t n, T** out) {
    void* p = nullptr;
    plex_status s = dev_alloc(c, n, &p);
    *out = reinterpret_cast<T*>(p);
    return s;
}

static void dev_free(plex_ctx_s* c, const void* p) {
    if (!p) return;
    DevHeap& h = c->heap;
    std::lock_guard<std::mutex> lk(h.mu);
    h.h.free((uint64_t)(reinterpret_cast<const uint8_t*>(p) - h.base));
}

// Every stream the ctx launches kernels or copies on has drained (cudaFree used
// to imply this; a workspace block may be handed out again right after a free).
static void quiesce(plex_ctx_s* c) {
    for (cudaStream_t s2 : {c->pack, c->copy, c->copy2, c->kasync, c->copy3, c->ckern, c->cstream, c->ccopy})
        if (s2) cudaStreamSynchronize(s2);
}

static void free_devplan(plex_ctx_s* c, DevPlan& d) {
    quiesce(c);
    for (const void* p : {(const void*)d.segs, (const void*)d.items, (const void*)d.push, (const void*)d.gather,
                          (const void*)d.push_local, (const void*)d.push_remote, (const void*)d.cks,
                          (const void*)d.cks_want, (const void*)d.cks_in, (const void*)d.items_el,
                          (const void*)d.local, (const void*)d.rpack, (const void*)d.runpack})
        dev_free(c, p);
    cudaFreeHost(d.h_cks_out);
    cudaFreeHost(d.h_cks_want);
    d = DevPlan{};
}

template <class T>
static plex_status upload(plex_ctx_s* c, T** dptr, const std::vector<T>& v) {
    *dptr = nullptr;
    if (v.empty()) return PLEX_OK;
    plex_status s = dev_alloc_t(c, sizeof(T) * v.size(), dptr);
    if (s) return s;
    CK(cudaMemcpy(*dptr, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    return PLEX_OK;
}

static plex_status get_devplan(plex_ctx_s* c, const Plan& p, DevPlan** out) {
    auto it = c->dev.find(p.id);
    if (it != c->dev.end()) { *out = &it->second; return PLEX_OK; }
    const RankPlan& R = p.ranks[c->rank];
    DevPlan d;
    plex_status s;
    if ((s = upload(c, &d.segs, R.segs)) || (s = upload(c, &d.items, R.items)) || (s = upload(c, &d.push, R.push)) ||
        (s = upload(c, &d.items_el, R.items_el)) || (s = upload(c, &d.gather, R.gather))) {
        free_devplan(c, d);
        return s;
    }
    const size_t nck = std::max<size_t>(1, 2 * R.segs.size());
    if ((s = dev_alloc_t(c, nck * 8, &d.cks)) || (s = dev_alloc_t(c, nck * 8, &d.cks_want)) ||
        (s = dev_alloc_t(c, nck * 8, &d.cks_in))) {
        free_devplan(c, d);
        return s;
    }
    if (cudaHostAlloc(&d.h_cks_out, nck * 8, cudaHostAllocDefault) != cudaSuccess ||
        cudaHostAlloc(&d.h_cks_want, nck * 8, cudaHostAllocDefault) != cudaSuccess) {
        (void)cudaGetLastError();
        free_devplan(c, d);
        set_error("cudaHostAlloc of checksum mirrors failed");
        return PLEX_E_CUDA;
    }
    const int32_t nb = n_buckets(p, R);
    d.bucket_payload.assign(nb, 0);
    for (const PackItem& it : R.items) {
        const SegDev& sg = R.segs[it.seg];
        const uint64_t o0 = it.slab_lo - sg.slab_off, o1 = o0 + it.len;
        const uint64_t de = std::min(o1, sg.bytes);
        if (de > o0) d.bucket_payload[it.slab_lo / p.bucket] += de - o0;
    }
    if (R.elide_start) {
        const int32_t nbe = (int32_t)R.bstart_el.size() - 1;
        d.bucket_payload_el.assign(nbe, 0);
        for (const PackItem& it : R.items_el) {
            const SegDev& sg = R.segs[it.seg];
            const uint64_t o0 = it.slab_lo - sg.slab_off, o1 = o0 + it.len;
            const uint64_t de = std::min(o1, sg.bytes);
            if (de > o0) d.bucket_payload_el[(it.slab_lo - R.elide_start) / p.bucket] += de - o0;
        }
        for (uint64_t k = 0; k < R.n_param_items; ++k) {
            const PackItem& it = R.items[k];
            const SegDev& sg = R.segs[it.seg];
            const uint64_t o0 = it.slab_lo - sg.slab_off, o1 = o0 + it.len;
            const uint64_t de = std::min(o1, sg.bytes);
            if (de > o0) d.elide_payload += de - o0;
        }
    }
    *out = &(c->dev[p.id] = d);
    return PLEX_OK;
}

static plex_status ensure_table(plex_ctx_s* c, uint64_t** h, uint64_t** d, size_t* capp, size_t n) {
    if (n <= *capp) return PLEX_OK;
    size_t cap = std::max<size_t>(n, 2 * *capp);
    if (*d) quiesce(c);
    cudaFreeHost(*h);
    dev_free(c, *d);
    *h = nullptr;
    *d = nullptr;
    *capp = 0;
    CK(cudaHostAlloc(h, cap * 8, cudaHostAllocDefault));
    plex_status s = dev_alloc_t(c, cap * 8, d);
    if (s) return s;
    *capp = cap;
    return PLEX_OK;
}
static plex_status ensure_ptrs(plex_ctx_s* c, size_t n) { return ensure_table(c, &c->h_ptrs, &c->d_ptrs, &c->ptr_cap, n); }

// ---- timing ------------------------------------------------------------------
static plex_status timed_begin(plex_ctx_s* c, cudaStream_t s, cudaEvent_t* a) {
    if (!(c->flags & PLEX_CTX_TIMING)) return PLEX_OK;
    while (c->pool_used + 2 > c->pool.size()) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        c->pool.push_back(e);
    }
    *a = c->pool[c->pool_used++];
    CK(cudaEventRecord(*a, s));
    return PLEX_OK;
}
static plex_status timed_end(plex_ctx_s* c, cudaStream_t s, cudaEvent_t a, int which, uint64_t bytes) {
    if (!(c->flags & PLEX_CTX_TIMING)) return PLEX_OK;
    cudaEvent_t b = c->pool[c->pool_used++];
    CK(cudaEventRecord(b, s));
    c->pending.push_back(Timed{which, bytes, a, b});
    return PLEX_OK;
}
static plex_status timed_collect(plex_ctx_s* c) {
    for (const Timed& t : c->pending) {
        float ms = 0, t0 = 0;
        CK(cudaEventElapsedTime(&ms, t.a, t.b));
        CK(cudaEventElapsedTime(&t0, c->pending.front().a, t.a));   // copy-engine / kernel timeline
        c->stats[t.which].launches += 1;
        c->stats[t.which].total_ms += ms;
        c->stats[t.which].bytes += t.bytes;
        if (c->trace.size() < (1u << 20)) c->trace.push_back(plex_launch_record{t.which, ms, t.bytes, t0, c->n_calls});
    }
    if (!c->pending.empty()) ++c->n_calls;
    c->pending.clear();
    c->pool_used = 0;
    return PLEX_OK;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d) {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// NVTX range around every exported transfer so nsys timelines show the
// a3-a12 phases next to the copy-engine rows and kernels.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

static plex_status finish(plex_ctx_s* c, cudaStream_t caller) {
    CK(cudaEventRecord(c->ev_pack_done, c->pack));
    CK(cudaEventRecord(c->ev_copy_done, c->copy));
    CK(cudaStreamWaitEvent(caller, c->ev_pack_done, 0));
    CK(cudaStreamWaitEvent(caller, c->ev_copy_done, 0));
    if (c->carry_used) {
        for (cudaStream_t s2 : {c->ckern, c->cstream, c->ccopy}) {
            CK(cudaEventRecord(c->ev_cend, s2));
            CK(cudaStreamWaitEvent(caller, c->ev_cend, 0));
            CK(cudaStreamSynchronize(s2));
        }
        c->carry_used = false;
        if (c->cerr) {
            CK(cudaMemcpy(c->h_cerr, c->cerr, sizeof(int), cudaMemcpyDeviceToHost));
            if (*c->h_cerr) {
                CK(cudaMemset(c->cerr, 0, sizeof(int)));
                *c->h_cerr = 0;
                // nothing of this call may still write the slab or the tensors once it
                // returns, and its events / pool slots must not leak into the next call
                CK(cudaStreamSynchronize(c->pack));
                CK(cudaStreamSynchronize(c->copy));
                plex_status st2 = timed_collect(c);
                if (st2) return st2;
                set_error("carried-bucket handshake with a peer timed out (a rank did not take part?)");
                return PLEX_E_CUDA;
            }
        }
    }
    CK(cudaStreamSynchronize(c->pack));
    CK(cudaStreamSynchronize(c->copy));
    return timed_collect(c);
}

void ctx_query(plex_ctx_t c, CtxInfo* o) {
    *o = CtxInfo{c->staging_bytes, c->n_slots, c->rank, c->world, c->device, c->comm != nullptr};
}

static plex_status check_common(plex_ctx_s* c, plex_plan_t plan) {
    if (!c || !plan) { set_error("NULL ctx/plan"); return PLEX_E_INVAL; }
    if (plan->p.world != c->world) {
        set_error("plan world %d != ctx world %d", plan->p.world, c->world);
        return PLEX_E_INVAL;
    }
    if (c->staging_bytes < (uint64_t)c->n_slots * plan->p.bucket) {
        set_error("staging %llu B < %d slots x bucket %llu B", (unsigned long long)c->staging_bytes, c->n_slots,
                  (unsigned long long)plan->p.bucket);
        return PLEX_E_INVAL;
    }
    return PLEX_OK;
}

static plex_status fill_state_ptrs(plex_ctx_s* c, const Plan& p, const void* const* ptrs, int32_t n, int table = 0) {
    const size_t nt = p.tensors.size();
    if (!ptrs || (size_t)n != PLEX_NUM_KINDS * nt) {
        set_error("expected %zu pointers (4 kinds x %zu tensors), got %d", PLEX_NUM_KINDS * nt, nt, n);
        return PLEX_E_INVAL;
    }
    plex_status s = table == 0   ? ensure_ptrs(c, PLEX_NUM_KINDS * nt)
                    : table == 1 ? ensure_table(c, &c->h_ptrs2, &c->d_ptrs2, &c->ptr_cap2, PLEX_NUM_KINDS * nt)
                                 : ensure_table(c, &c->h_ptrs3, &c->d_ptrs3, &c->ptr_cap3, PLEX_NUM_KINDS * nt);
    if (s) return s;
    uint64_t* h = table == 0 ? c->h_ptrs : table == 1 ? c->h_ptrs2 : c->h_ptrs3;
    const RankPlan& R = p.ranks[c->rank];
    for (size_t i = 0; i < PLEX_NUM_KINDS * nt; ++i) h[i] = reinterpret_cast<uint64_t>(ptrs[i]);
    for (const SegDev& sg : R.segs) {
        if (sg.bytes && !ptrs[sg.ptr_slot]) {
            set_error("NULL pointer for tensor %u kind %u", sg.ptr_slot % (uint32_t)nt, sg.ptr_slot / (uint32_t)nt);
            return PLEX_E_INVAL;
        }
        // NEXT-2 replicated params: the PARAM pointer is the full tensor; this
        // rank's segment starts at its first FSDP row
        if ((p.flags & PLEX_PLAN_REPLICA_PARAM) && sg.ptr_slot < nt && h[sg.ptr_slot])
            h[sg.ptr_slot] += sg.index_base * sg.esize;
    }
    return PLEX_OK;
}

// ---- bucket pipeline halves (a3+a4 offload, a6+a7 onload) -------------------------
// A Pipe is one direction's staging ring: slot s of a bucket b = b mod n_slots;
// ev_k[s] = the kernel finished with the slot, ev_c[s] = the copy finished.
struct Pipe {
    uint8_t* staging;
    int n_slots;
    cudaEvent_t* ev_k;
    cudaEvent_t* ev_c;
    cudaStream_t kern;
    cudaStream_t copy;
    uint64_t* h_ptrs;
    uint64_t* d_ptrs;
    unsigned int* ctr;      // per-launch work counter of the pack/unpack kernel
    int* d_flag;            // elision check / checksum verify result (device)
    int* h_flag;            // ... and its pinned host mirror
    bool untimed = false;   // async ops do not record per-launch events
};

static plex_status tbeg(plex_ctx_s* c, const Pipe& pp, cudaStream_t s, cudaEvent_t* a) {
    return pp.untimed ? PLEX_OK : timed_begin(c, s, a);
}
static plex_status tend(plex_ctx_s* c, const Pipe& pp, cudaStream_t s, cudaEvent_t a, int which, uint64_t bytes) {
    return pp.untimed ? PLEX_OK : timed_end(c, s, a, which, bytes);
}

struct Half {           // one offload or onload in flight
    const Plan* p;
    const RankPlan* R;
    DevPlan* d;
    plex_slab_s* slab;
    int32_t nb;
    std::vector<uint64_t> cks;     // offload: recorded checksums (host)
    bool elide = false;            // NEXT-2: PARAM prefix derived, not moved
    // bucket grid in use: buckets b cover [base + b*B, ...) with items
    // grid_items[bstart[b] .. bstart[b+1])
    uint64_t base = 0;
    const PackItem* grid_items = nullptr;
    const uint64_t* bstart = nullptr;
    const uint64_t* payload = nullptr;
};

static void use_grid(Half& h, bool elide) {
    h.elide = elide;
    if (elide) {
        h.base = h.R->elide_start;
        h.grid_items = h.d->items_el;
        h.bstart = h.R->bstart_el.data();
        h.payload = h.d->bucket_payload_el.data();
        h.nb = (int32_t)h.R->bstart_el.size() - 1;
    } else {
        h.base = 0;
        h.grid_items = h.d->items;
        h.bstart = h.R->bucket_item_start.data();
        h.payload = h.d->bucket_payload.data();
        h.nb = n_buckets(*h.p, *h.R);
    }
}

// ---- NEXT-1 host-link balancing: carried buckets -----------------------------------
// Every rank walks the plan's global carry list in order and takes part only in
// the transfers it owns or carries, on its carry streams: both ends of every
// pair see their common transfers in the same order, and the global order
// rules out cycles.
//
// Default transport, over peer memory (no NCCL, no carrier staging):
//   offload  owner:   [wait FREE[s]] pack bucket -> own slot s ; READY[s] = seq
//            carrier: wait owner's READY[s] ; D2H owner's slot (its copy engine
//                     reads the peer over NVLink) -> pinned carry region ;
//                     owner's FREE[s] = seq
//   onload   carrier: [wait owner's FREE[s]] H2D carry region -> owner's slot
//                     (written over NVLink) ; owner's READY[s] = seq
//            owner:   wait READY[s] ; unpack own slot s ; FREE[s] = seq
// Flags are u64 sequence numbers (epoch << 20 | transfer + 1) in the owner's
// memory, set by one-thread release stores and polled by one-thread acquire
// spins (timeout -> PLEX_E_CUDA, never a hung GPU).  PLEX_CTX_CARRY_NCCL keeps
// the NCCL send/recv transport (owner slot -> carrier slot -> D2H) as baseline.
static constexpr unsigned long long kCarryTimeoutNs = 120ull * 1000000000ull;
enum { kReady = 0, kFree = 4 };

static plex_status carry_ready(plex_ctx_s* c, const Plan& p) {
    if (p.carry.empty()) return PLEX_OK;
    if (!c->comm) { set_error("carried buckets need a ctx with an NCCL communicator"); return PLEX_E_INVAL; }
    if (!c->cstaging || c->cstaging_bytes < 4 * p.bucket) {
        set_error("carried buckets need carry staging >= 4 x bucket (plex_ctx_set_carry_staging)");
        return PLEX_E_INVAL;
    }
    if (!c->ckern) {
        CK(cudaStreamCreateWithFlags(&c->ckern, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->ccopy, cudaStreamNonBlocking));
        for (int i = 0; i < 4; ++i) {
            CK(cudaEventCreateWithFlags(&c->ev_cs[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c->ev_cc[i], cudaEventDisableTiming));
        }
        CK(cudaEventCreateWithFlags(&c->ev_cbeg, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_cend, cudaEventDisableTiming));
    }
    if (!(c->flags & PLEX_CTX_CARRY_NCCL)) {
        if (!c->cflags) {
            void* f = nullptr;
            plex_status sa = dev_alloc(c, 4096, &f);                // exported to the peers over CUDA IPC
            if (sa) return sa;
            CK(cudaMemset(f, 0, 4096));
            c->cflags = reinterpret_cast<unsigned long long*>(f);
            c->cerr = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(f) + 2048);
            CK(cudaHostAlloc(&c->h_cerr, sizeof(int), cudaHostAllocDefault));
            *c->h_cerr = 0;
        }
        plex_status st;
        if ((st = exchange_arenas(c, 2, c->cstaging, c->peer_cstaging)) ||
            (st = exchange_arenas(c, 3, c->cflags, c->peer_cflags)))
            return st;
    }
    return PLEX_OK;
}

static unsigned long long* peer_flag(plex_ctx_s* c, int rank, int idx) {
    return reinterpret_cast<unsigned long long*>(c->peer_cflags[rank]) + idx;
}

// offload direction over peer memory (owner slots 0-1)
static plex_status carry_out_p2p(plex_ctx_s* c, Pipe& pp, Half& h) {
    const Plan& p = *h.p;
    const RankPlan& R = *h.R;
    const unsigned long long epoch = ++c->cepoch;
    std::vector<int> k_of(p.world, 0);                          // transfers per owner so far
    std::vector<unsigned long long> last(2, 0);                 // own slots: seq of their last use
    plex_status st;
    for (size_t i = 0; i < p.carry.size(); ++i) {
        const CarryXfer& x = p.carry[i];
        const int k = k_of[x.owner]++;
        const int sl = k % 2;
        const unsigned long long seq = (epoch << 20) | (unsigned long long)(i + 1);
        cudaEvent_t ta = nullptr;
        if (x.owner == c->rank) {
            if (last[sl]) CK(launch_wait(peer_flag(c, c->rank, kFree + sl), last[sl], kCarryTimeoutNs, c->cerr, c->ckern));
            uint8_t* slot = c->cstaging + (uint64_t)sl * p.bucket;
            const uint64_t i0 = R.bucket_item_start[x.bucket], i1 = R.bucket_item_start[x.bucket + 1];
            if ((st = tbeg(c, pp, c->ckern, &ta))) return st;
            CK(launch_pack(true, h.d->items + i0, (uint32_t)(i1 - i0), h.d->segs, pp.d_ptrs, slot, x.lo, h.d->cks,
                           c->d_ctr + 4, c->ckern));
            if ((st = tend(c, pp, c->ckern, ta, PLEX_STAT_PACK, 2 * h.d->bucket_payload[x.bucket]))) return st;
            CK(launch_signal(peer_flag(c, c->rank, kReady + sl), seq, c->ckern));
            last[sl] = seq;
        } else if (x.carrier == c->rank) {
            CK(launch_wait(peer_flag(c, x.owner, kReady + sl), seq, kCarryTimeoutNs, c->cerr, c->ccopy));
            const uint8_t* src = reinterpret_cast<const uint8_t*>(c->peer_cstaging[x.owner]) + (uint64_t)sl * p.bucket;
            if ((st = tbeg(c, pp, c->ccopy, &ta))) return st;
            CK(cudaMemcpyAsync(h.slab->carry_host + x.coff, src, x.len, cudaMemcpyDeviceToHost, c->ccopy));
            if ((st = tend(c, pp, c->ccopy, ta, PLEX_STAT_D2H, x.len))) return st;
            CK(launch_signal(peer_flag(c, x.owner, kFree + sl), seq, c->ccopy));
        }
    }
    // the call ends only when every carrier has copied this rank's slots out
    for (int sl = 0; sl < 2; ++sl)
        if (last[sl]) CK(launch_wait(peer_flag(c, c->rank, kFree + sl), last[sl], kCarryTimeoutNs, c->cerr, c->ckern));
    return PLEX_OK;
}

// onload direction over peer memory (owner slots 2-3)
static plex_status carry_in_p2p(plex_ctx_s* c, Pipe& pp, Half& h) {
    const Plan& p = *h.p;
    const RankPlan& R = *h.R;
    const unsigned long long epoch = ++c->cepoch;
    std::vector<int> k_of(p.world, 0);
    // last sequence number written into (owner, onload slot), kept across calls:
    // the first write of a call into a slot must wait for that slot's FREE flag of
    // the previous call too (every rank derives the same values from the carry lists)
    auto& last = c->carry_in_last;
    if (last.size() != (size_t)p.world) last.assign(p.world, std::vector<unsigned long long>(2, 0));
    plex_status st;
    for (size_t i = 0; i < p.carry.size(); ++i) {
        const CarryXfer& x = p.carry[i];
        const int k = k_of[x.owner]++;
        const int sl = 2 + k % 2;
        const unsigned long long seq = (epoch << 20) | (unsigned long long)(i + 1);
        const unsigned long long prev = last[x.owner][sl - 2];
        last[x.owner][sl - 2] = seq;
        cudaEvent_t ta = nullptr;
        if (x.carrier == c->rank) {
            if (prev) CK(launch_wait(peer_flag(c, x.owner, kFree + sl), prev, kCarryTimeoutNs, c->cerr, c->ccopy));
            uint8_t* dst = reinterpret_cast<uint8_t*>(c->peer_cstaging[x.owner]) + (uint64_t)sl * p.bucket;
            if ((st = tbeg(c, pp, c->ccopy, &ta))) return st;
            CK(cudaMemcpyAsync(dst, h.slab->carry_host + x.coff, x.len, cudaMemcpyHostToDevice, c->ccopy));
            if ((st = tend(c, pp, c->ccopy, ta, PLEX_STAT_H2D, x.len))) return st;
            CK(launch_signal(peer_flag(c, x.owner, kReady + sl), seq, c->ccopy));
        } else if (x.owner == c->rank) {
            CK(launch_wait(peer_flag(c, c->rank, kReady + sl), seq, kCarryTimeoutNs, c->cerr, c->ckern));
            uint8_t* slot = c->cstaging + (uint64_t)sl * p.bucket;
            const uint64_t i0 = R.bucket_item_start[x.bucket], i1 = R.bucket_item_start[x.bucket + 1];
            if ((st = tbeg(c, pp, c->ckern, &ta))) return st;
            CK(launch_pack(false, h.d->items + i0, (uint32_t)(i1 - i0), h.d->segs, pp.d_ptrs, slot, x.lo,
                           h.d->cks_in, c->d_ctr + 5, c->ckern));
            if ((st = tend(c, pp, c->ckern, ta, PLEX_STAT_UNPACK, 2 * h.d->bucket_payload[x.bucket]))) return st;
            CK(launch_signal(peer_flag(c, c->rank, kFree + sl), seq, c->ckern));
        }
    }
    // a carrier's call ends only when the owners have unpacked what it wrote
    {
        std::vector<int> k2(p.world, 0);
        std::vector<std::vector<unsigned long long>> mine(p.world, std::vector<unsigned long long>(2, 0));
        for (size_t i = 0; i < p.carry.size(); ++i) {
            const CarryXfer& x = p.carry[i];
            const int k = k2[x.owner]++;
            if (x.carrier == c->rank) mine[x.owner][k % 2] = (epoch << 20) | (unsigned long long)(i + 1);
        }
        for (int g = 0; g < p.world; ++g)
            for (int j = 0; j < 2; ++j)
                if (mine[g][j]) CK(launch_wait(peer_flag(c, g, kFree + 2 + j), mine[g][j], kCarryTimeoutNs, c->cerr, c->ccopy));
    }
    return PLEX_OK;
}

// offload direction (slots 0-1): call after off_begin, before the own buckets
static plex_status carry_out(plex_ctx_s* c, Pipe& pp, Half& h) {
    const Plan& p = *h.p;
    if (p.carry.empty() || h.elide) return PLEX_OK;
    plex_status st;
    if ((st = carry_ready(c, p))) return st;
    c->carry_used = true;
    if (!(c->flags & PLEX_CTX_CARRY_NCCL)) {
        CK(cudaEventRecord(c->ev_cbeg, pp.kern));             // pointer table + zeroed checksums
        CK(cudaStreamWaitEvent(c->ckern, c->ev_cbeg, 0));
        CK(cudaStreamWaitEvent(c->ccopy, c->ev_cbeg, 0));
        return carry_out_p2p(c, pp, h);
    }
    CK(cudaEventRecord(c->ev_cbeg, pp.kern));                 // pointer table + zeroed checksums
    CK(cudaStreamWaitEvent(c->ckern, c->ev_cbeg, 0));
    CK(cudaStreamWaitEvent(c->cstream, c->ev_cbeg, 0));
    CK(cudaStreamWaitEvent(c->ccopy, c->ev_cbeg, 0));
    const RankPlan& R = *h.R;
    int k = 0;
    for (const CarryXfer& x : p.carry) {
        if (x.owner != c->rank && x.carrier != c->rank) continue;
        const int sl = k % 2;
        uint8_t* slot = c->cstaging + (uint64_t)sl * p.bucket;
        cudaEvent_t ta = nullptr;
        if (x.owner == c->rank) {
            if (k >= 2) CK(cudaStreamWaitEvent(c->ckern, c->ev_cs[sl], 0));      // slot's last send done
            const uint64_t i0 = R.bucket_item_start[x.bucket], i1 = R.bucket_item_start[x.bucket + 1];
            if ((st = tbeg(c, pp, c->ckern, &ta))) return st;
            CK(launch_pack(true, h.d->items + i0, (uint32_t)(i1 - i0), h.d->segs, pp.d_ptrs, slot, x.lo, h.d->cks,
                           c->d_ctr + 4, c->ckern));
            if ((st = tend(c, pp, c->ckern, ta, PLEX_STAT_PACK, 2 * h.d->bucket_payload[x.bucket]))) return st;
            CK(cudaEventRecord(c->ev_cc[sl], c->ckern));
            CK(cudaStreamWaitEvent(c->cstream, c->ev_cc[sl], 0));
            NK(ncclSend(slot, x.len, ncclUint8, x.carrier, c->comm, c->cstream));
            CK(cudaEventRecord(c->ev_cs[sl], c->cstream));
        } else {
            if (k >= 2) CK(cudaStreamWaitEvent(c->cstream, c->ev_cc[sl], 0));    // slot's last D2H done
            NK(ncclRecv(slot, x.len, ncclUint8, x.owner, c->comm, c->cstream));
            CK(cudaEventRecord(c->ev_cs[sl], c->cstream));
            CK(cudaStreamWaitEvent(c->ccopy, c->ev_cs[sl], 0));
            if ((st = tbeg(c, pp, c->ccopy, &ta))) return st;
            CK(cudaMemcpyAsync(h.slab->carry_host + x.coff, slot, x.len, cudaMemcpyDeviceToHost, c->ccopy));
            if ((st = tend(c, pp, c->ccopy, ta, PLEX_STAT_D2H, x.len))) return st;
            CK(cudaEventRecord(c->ev_cc[sl], c->ccopy));
        }
        ++k;
    }
    return PLEX_OK;
}

// onload direction (slots 2-3): call after on_begin, before the own buckets
static plex_status carry_in(plex_ctx_s* c, Pipe& pp, Half& h) {
    const Plan& p = *h.p;
    if (p.carry.empty() || h.elide) return PLEX_OK;
    plex_status st;
    if ((st = carry_ready(c, p))) return st;
    c->carry_used = true;
    if (!(c->flags & PLEX_CTX_CARRY_NCCL)) {
        CK(cudaEventRecord(c->ev_cbeg, pp.kern));
        CK(cudaStreamWaitEvent(c->ckern, c->ev_cbeg, 0));
        CK(cudaStreamWaitEvent(c->ccopy, c->ev_cbeg, 0));
        return carry_in_p2p(c, pp, h);
    }
    CK(cudaEventRecord(c->ev_cbeg, pp.kern));
    CK(cudaStreamWaitEvent(c->ckern, c->ev_cbeg, 0));
    CK(cudaStreamWaitEvent(c->cstream, c->ev_cbeg, 0));
    CK(cudaStreamWaitEvent(c->ccopy, c->ev_cbeg, 0));
    const RankPlan& R = *h.R;
    int k = 0;
    for (const CarryXfer& x : p.carry) {
        if (x.owner != c->rank && x.carrier != c->rank) continue;
        const int sl = 2 + k % 2;
        uint8_t* slot = c->cstaging + (uint64_t)sl * p.bucket;
        cudaEvent_t ta = nullptr;
        if (x.carrier == c->rank) {
            if (k >= 2) CK(cudaStreamWaitEvent(c->ccopy, c->ev_cs[sl], 0));      // slot's last send done
            if ((st = tbeg(c, pp, c->ccopy, &ta))) return st;
            CK(cudaMemcpyAsync(slot, h.slab->carry_host + x.coff, x.len, cudaMemcpyHostToDevice, c->ccopy));
            if ((st = tend(c, pp, c->ccopy, ta, PLEX_STAT_H2D, x.len))) return st;
            CK(cudaEventRecord(c->ev_cc[sl], c->ccopy));
            CK(cudaStreamWaitEvent(c->cstream, c->ev_cc[sl], 0));
            NK(ncclSend(slot, x.len, ncclUint8, x.owner, c->comm, c->cstream));
            CK(cudaEventRecord(c->ev_cs[sl], c->cstream));
        } else {
            if (k >= 2) CK(cudaStreamWaitEvent(c->cstream, c->ev_cc[sl], 0));    // slot's last unpack done
            NK(ncclRecv(slot, x.len, ncclUint8, x.carrier, c->comm, c->cstream));
            CK(cudaEventRecord(c->ev_cs[sl], c->cstream));
            CK(cudaStreamWaitEvent(c->ckern, c->ev_cs[sl], 0));
            const uint64_t i0 = R.bucket_item_start[x.bucket], i1 = R.bucket_item_start[x.bucket + 1];
            if ((st = tbeg(c, pp, c->ckern, &ta))) return st;
            CK(launch_pack(false, h.d->items + i0, (uint32_t)(i1 - i0), h.d->segs, pp.d_ptrs, slot, x.lo,
                           h.d->cks_in, c->d_ctr + 5, c->ckern));
            if ((st = tend(c, pp, c->ckern, ta, PLEX_STAT_UNPACK, 2 * h.d->bucket_payload[x.bucket]))) return st;
            CK(cudaEventRecord(c->ev_cc[sl], c->ckern));
        }
        ++k;
    }
    return PLEX_OK;
}

// Before the checksum read-back (offload) / verify (onload): the half's kernel
// stream waits for the carried buckets' pack / unpack kernels.  Enqueued after
// the own buckets so the own pipeline never queues behind carried transfers.
static plex_status carry_join(plex_ctx_s* c, Pipe& pp, Half& h) {
    if (h.p->carry.empty() || h.elide || !c->ckern) return PLEX_OK;
    CK(cudaEventRecord(c->ev_cend, c->ckern));
    CK(cudaStreamWaitEvent(pp.kern, c->ev_cend, 0));
    return PLEX_OK;
}

static plex_status off_begin(plex_ctx_s* c, Pipe& pp, Half& h) {
    const size_t np = PLEX_NUM_KINDS * h.p->tensors.size();
    const size_t ckb = 16 * std::max<size_t>(1, h.R->segs.size());
    CK(cudaMemcpyAsync(pp.d_ptrs, pp.h_ptrs, np * 8, cudaMemcpyHostToDevice, pp.kern));
    CK(cudaMemsetAsync(h.d->cks, 0, ckb, pp.kern));
    h.cks.assign(2 * h.R->segs.size(), 0);
    use_grid(h, false);
    if (h.R->elide_start) {
        // NEXT-2: does every bf16 param equal RNE(master)?  (checksums the params)
        CK(cudaMemsetAsync(pp.d_flag, 0, sizeof(int), pp.kern));
        cudaEvent_t ta = nullptr;
        plex_status st;
        if ((st = tbeg(c, pp, pp.kern, &ta))) return st;
        CK(launch_derive(true, h.d->items, (uint32_t)h.R->n_param_items, h.d->segs, pp.d_ptrs,
                         (uint32_t)h.p->tensors.size(), h.d->cks, pp.d_flag, pp.kern));
        if ((st = tend(c, pp, pp.kern, ta, PLEX_STAT_DERIVE, 3 * h.d->elide_payload))) return st;
        CK(cudaMemcpyAsync(pp.h_flag, pp.d_flag, sizeof(int), cudaMemcpyDeviceToHost, pp.kern));
        CK(cudaStreamSynchronize(pp.kern));
        if (*pp.h_flag == 0) use_grid(h, true);
        else CK(cudaMemsetAsync(h.d->cks, 0, ckb, pp.kern));    // full offload after all
    }
    return PLEX_OK;
}

static plex_status off_bucket(plex_ctx_s* c, Pipe& pp, Half& h, int32_t b) {
    const Plan& p = *h.p;
    const RankPlan& R = *h.R;
    if (!h.elide && R.carried[b]) return PLEX_OK;            // moved through another rank's host link
    const int slot = b % pp.n_slots;
    uint8_t* stg = pp.staging + (uint64_t)slot * p.bucket;
    const uint64_t lo = h.base + (uint64_t)b * p.bucket;
    const uint64_t len = std::min<uint64_t>(p.bucket, R.slab_bytes - lo);
    if (b >= pp.n_slots) CK(cudaStreamWaitEvent(pp.kern, pp.ev_c[slot], 0));
    const uint64_t i0 = h.bstart[b], i1 = h.bstart[b + 1];
    cudaEvent_t ta = nullptr;
    plex_status st;
    if ((st = tbeg(c, pp, pp.kern, &ta))) return st;
    CK(launch_pack(true, h.grid_items + i0, (uint32_t)(i1 - i0), h.d->segs, pp.d_ptrs, stg, lo, h.d->cks, pp.ctr,
                   pp.kern));
    if ((st = tend(c, pp, pp.kern, ta, PLEX_STAT_PACK, 2 * h.payload[b]))) return st;
    CK(cudaEventRecord(pp.ev_k[slot], pp.kern));
    CK(cudaStreamWaitEvent(pp.copy, pp.ev_k[slot], 0));
    if ((st = tbeg(c, pp, pp.copy, &ta))) return st;
    CK(cudaMemcpyAsync(h.slab->host + lo, stg, len, cudaMemcpyDeviceToHost, pp.copy));
    if ((st = tend(c, pp, pp.copy, ta, PLEX_STAT_D2H, len))) return st;
    CK(cudaEventRecord(pp.ev_c[slot], pp.copy));
    return PLEX_OK;
}

static plex_status off_end(plex_ctx_s* c, Pipe& pp, Half& h) {
    (void)c;
    if (!h.cks.empty()) CK(cudaMemcpyAsync(h.d->h_cks_out, h.d->cks, 8 * h.cks.size(), cudaMemcpyDeviceToHost, pp.kern));
    return PLEX_OK;
}

// After the offload's streams completed: the recorded checksums, from the pinned mirror.
static void off_collect(Half& h) {
    if (!h.cks.empty()) std::memcpy(h.cks.data(), h.d->h_cks_out, 8 * h.cks.size());
}

static plex_status on_begin(plex_ctx_s* c, Pipe& pp, Half& h) {
    const size_t np = PLEX_NUM_KINDS * h.p->tensors.size();
    const size_t nck = 2 * h.R->segs.size();
    CK(cudaMemcpyAsync(pp.d_ptrs, pp.h_ptrs, np * 8, cudaMemcpyHostToDevice, pp.kern));
    CK(cudaMemsetAsync(h.d->cks_in, 0, 8 * std::max<size_t>(2, nck), pp.kern));
    if (nck) {
        // the pinned mirror is read by the copy engine after this returns; no
        // earlier upload from it can still be pending (one onload per plan and
        // ctx at a time: blocking ones complete, a prefetch is waited first)
        std::memcpy(h.d->h_cks_want, h.slab->cks.data(), 8 * nck);
        CK(cudaMemcpyAsync(h.d->cks_want, h.d->h_cks_want, 8 * nck, cudaMemcpyHostToDevice, pp.kern));
    }
    CK(cudaMemsetAsync(pp.d_flag, 0, sizeof(int), pp.kern));
    use_grid(h, h.slab->elided);
    return PLEX_OK;
}

static plex_status on_bucket(plex_ctx_s* c, Pipe& pp, Half& h, int32_t b) {
    const Plan& p = *h.p;
    const RankPlan& R = *h.R;
    if (!h.elide && R.carried[b]) return PLEX_OK;            // comes back through another rank
    const int slot = b % pp.n_slots;
    uint8_t* stg = pp.staging + (uint64_t)slot * p.bucket;
    const uint64_t lo = h.base + (uint64_t)b * p.bucket;
    const uint64_t len = std::min<uint64_t>(p.bucket, R.slab_bytes - lo);
    if (b >= pp.n_slots) CK(cudaStreamWaitEvent(pp.copy, pp.ev_k[slot], 0));
    cudaEvent_t ta = nullptr;
    plex_status st;
    if ((st = tbeg(c, pp, pp.copy, &ta))) return st;
    CK(cudaMemcpyAsync(stg, h.slab->host + lo, len, cudaMemcpyHostToDevice, pp.copy));
    if ((st = tend(c, pp, pp.copy, ta, PLEX_STAT_H2D, len))) return st;
    CK(cudaEventRecord(pp.ev_c[slot], pp.copy));
    CK(cudaStreamWaitEvent(pp.kern, pp.ev_c[slot], 0));
    const uint64_t i0 = h.bstart[b], i1 = h.bstart[b + 1];
    if ((st = tbeg(c, pp, pp.kern, &ta))) return st;
    CK(launch_pack(false, h.grid_items + i0, (uint32_t)(i1 - i0), h.d->segs, pp.d_ptrs, stg, lo, h.d->cks_in, pp.ctr,
                   pp.kern));
    if ((st = tend(c, pp, pp.kern, ta, PLEX_STAT_UNPACK, 2 * h.payload[b]))) return st;
    CK(cudaEventRecord(pp.ev_k[slot], pp.kern));
    return PLEX_OK;
}

static plex_status on_end(plex_ctx_s* c, Pipe& pp, Half& h) {
    if (h.elide) {   // NEXT-2: re-derive the elided params from the restored master
        cudaEvent_t ta = nullptr;
        plex_status st;
        if ((st = tbeg(c, pp, pp.kern, &ta))) return st;
        CK(launch_derive(false, h.d->items, (uint32_t)h.R->n_param_items, h.d->segs, pp.d_ptrs,
                         (uint32_t)h.p->tensors.size(), h.d->cks_in, pp.d_flag, pp.kern));
        if ((st = tend(c, pp, pp.kern, ta, PLEX_STAT_DERIVE, 3 * h.d->elide_payload))) return st;
    }
    CK(launch_verify(h.d->cks_in, h.d->cks_want, (uint32_t)h.R->segs.size(), pp.d_flag, pp.kern));
    CK(cudaMemcpyAsync(pp.h_flag, pp.d_flag, sizeof(int), cudaMemcpyDeviceToHost, pp.kern));
    return PLEX_OK;
}

static plex_status check_slab(plex_ctx_s* c, plex_plan_t plan, plex_slab_t slab, bool write = false) {
    if (!slab || slab->plan_id != plan->p.id || slab->rank != c->rank) {
        set_error("slab does not belong to this plan/rank");
        return PLEX_E_INVAL;
    }
    if (slab->busy) { set_error("an async transfer of this slab is in flight: plex_state_wait first"); return PLEX_E_STATE; }
    if (write && slab->ckpt.load()) { set_error("a checkpoint of this slab is being written (slab is read-only)"); return PLEX_E_STATE; }
    return PLEX_OK;
}

struct AsyncState {
    Half h;
    Pipe pp;
    plex_slab_s* slab = nullptr;
    cudaEvent_t done_k = nullptr, done_c = nullptr;
    // A drain of an elision plan must read the derivability flag on the host
    // before it can lay out its buckets; that wait (for the caller's prior work
    // plus the check kernel) runs on this worker thread, not the caller's.
    std::thread worker;
    std::atomic<bool> enqueued{true};
    plex_status enq_status = PLEX_OK;
    std::string enq_error;
};

static void async_free(AsyncState* a) {
    if (!a) return;
    if (a->worker.joinable()) a->worker.join();
    if (a->done_k) cudaEventDestroy(a->done_k);
    if (a->done_c) cudaEventDestroy(a->done_c);
    delete a;
}

// Blocking state transfers use the rings the async ones run on.
static plex_status check_no_async(plex_ctx_s* c) {
    if (c->async[0] || c->async[1]) {
        set_error("async drain/prefetch in flight on this ctx: plex_state_wait first");
        return PLEX_E_STATE;
    }
    return PLEX_OK;
}

}  // namespace plex

extern "C" {

plex_status plex_nccl_unique_id(void* out128) {
    if (!out128) { set_error("NULL out"); return PLEX_E_INVAL; }
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
    return PLEX_OK;
}

plex_status plex_ctx_create(int32_t device, void* staging, uint64_t staging_bytes, void* workspace,
                            uint64_t workspace_bytes, int32_t n_slots, void* pack_stream, void* copy_stream,
                            const void* nccl_id, int32_t rank, int32_t world, uint32_t flags, plex_ctx_t* out) {
    if (!out) { set_error("NULL out"); return PLEX_E_INVAL; }
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world || n_slots < 1 || n_slots > 64 || !staging || !staging_bytes) {
        set_error("bad ctx arguments (rank %d world %d slots %d)", rank, world, n_slots);
        return PLEX_E_INVAL;
    }
    if (reinterpret_cast<uintptr_t>(staging) % 256) { set_error("staging must be 256-B aligned"); return PLEX_E_INVAL; }
    if (!workspace || reinterpret_cast<uintptr_t>(workspace) % 256 || workspace_bytes < kMinWorkspace) {
        set_error("workspace must be a 256-B aligned device buffer of >= %llu bytes",
                  (unsigned long long)kMinWorkspace);
        return PLEX_E_INVAL;
    }
    DeviceGuard g(device);
    auto* c = new plex_ctx_s();
    c->heap.base = reinterpret_cast<uint8_t*>(workspace);
    c->heap.h.reset(workspace_bytes);
    c->device = device;
    c->staging = reinterpret_cast<uint8_t*>(staging);
    c->staging_bytes = staging_bytes;
    c->n_slots = n_slots;
    c->pack = reinterpret_cast<cudaStream_t>(pack_stream);
    c->copy = reinterpret_cast<cudaStream_t>(copy_stream);
    c->rank = rank;
    c->world = world;
    c->flags = flags;
    auto fail = [&](plex_status s) {
        plex_ctx_destroy(c);
        return s;
    };
    if (cudaEventCreateWithFlags(&c->ev_caller, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_pack_done, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_copy_done, cudaEventDisableTiming) != cudaSuccess) {
        set_error("cudaEventCreate failed");
        return fail(PLEX_E_CUDA);
    }
    c->ev_pack.resize(n_slots);
    c->ev_copy.resize(n_slots);
    for (int i = 0; i < n_slots; ++i)
        if (cudaEventCreateWithFlags(&c->ev_pack[i], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_copy[i], cudaEventDisableTiming) != cudaSuccess) {
            set_error("cudaEventCreate failed");
            return fail(PLEX_E_CUDA);
        }
    for (auto& e : c->ev_sync)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
            set_error("cudaEventCreate failed");
            return fail(PLEX_E_CUDA);
        }
    c->scratch_bytes = 256 * (size_t)world + 256;
    {
        plex_status sa;
        if ((sa = dev_alloc_t(c, 64, &c->d_flag)) || (sa = dev_alloc_t(c, 64, &c->d_ctr)) ||
            (sa = dev_alloc_t(c, 2 * c->scratch_bytes, &c->d_scratch)))
            return fail(sa);
    }
    if (cudaHostAlloc(&c->h_flag, 64, cudaHostAllocDefault) != cudaSuccess ||
        cudaHostAlloc(&c->h_scratch, 2 * c->scratch_bytes, cudaHostAllocDefault) != cudaSuccess) {
        set_error("ctx pinned scratch allocation failed");
        return fail(PLEX_E_CUDA);
    }
    // pack/unpack claim counters [0, 8) and their finished-CTA counters [8, 16):
    // zero once here, every launch leaves them zeroed (pack_kernel)
    if (cudaMemset(c->d_ctr, 0, 64) != cudaSuccess) {
        set_error("ctx counter init failed");
        return fail(PLEX_E_CUDA);
    }
    if (nccl_id && world > 1) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
        if (r != ncclSuccess) {
            c->comm = nullptr;
            set_error("ncclCommInitRank: %s", ncclGetErrorString(r));
            return fail(PLEX_E_NCCL);
        }
    }
    {
        std::lock_guard<std::mutex> lk(g_ctx_mu);
        g_ctxs.insert(c);
    }
    *out = c;
    return PLEX_OK;
}

plex_status plex_ctx_workspace(plex_ctx_t c, uint64_t* in_use, uint64_t* high_water) {
    if (!c || !in_use || !high_water) { set_error("NULL argument"); return PLEX_E_INVAL; }
    std::lock_guard<std::mutex> lk(c->heap.mu);
    *in_use = c->heap.h.in_use();
    *high_water = c->heap.h.high_water();
    return PLEX_OK;
}

plex_status plex_ctx_destroy(plex_ctx_t c) {
    if (!c) return PLEX_OK;
    {
        std::lock_guard<std::mutex> lk(g_ctx_mu);
        g_ctxs.erase(c);
    }
    DeviceGuard g(c->device);
    for (auto& a : c->async)               // an enqueue worker must be done before the streams drain
        if (a && a->worker.joinable()) a->worker.join();
    if (c->pack) cudaStreamSynchronize(c->pack);
    if (c->copy) cudaStreamSynchronize(c->copy);
    if (c->copy2) cudaStreamSynchronize(c->copy2);
    if (c->kasync) cudaStreamSynchronize(c->kasync);
    for (cudaStream_t s2 : {c->ckern, c->cstream, c->ccopy})
        if (s2) cudaStreamSynchronize(s2);
    if (c->copy3) cudaStreamSynchronize(c->copy3);
    for (auto& a : c->async) {
        if (a) { a->slab->busy = false; async_free(a); a = nullptr; }
    }
    for (auto& kv : c->dev) free_devplan(c, kv.second);
    for (auto& kv : c->peers)
        if (kv.second.second) cudaIpcCloseMemHandle(kv.second.second);
    if (c->comm) ncclCommDestroy(c->comm);
    for (cudaEvent_t e : c->ev_pack) if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ev_copy) if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : c->pool) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ev_sync) if (e) cudaEventDestroy(e);
    if (c->ev_caller) cudaEventDestroy(c->ev_caller);
    if (c->ev_pack_done) cudaEventDestroy(c->ev_pack_done);
    if (c->ev_copy_done) cudaEventDestroy(c->ev_copy_done);
    cudaFreeHost(c->h_ptrs);
    cudaFreeHost(c->h_ptrs2);
    for (cudaEvent_t e : c->ev_pack2) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ev_piece) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ev_copy2) cudaEventDestroy(e);
    if (c->copy2) cudaStreamDestroy(c->copy2);
    if (c->kasync) cudaStreamDestroy(c->kasync);
    for (cudaStream_t s2 : {c->ckern, c->cstream, c->ccopy})
        if (s2) cudaStreamDestroy(s2);
    for (int i = 0; i < 4; ++i) {
        if (c->ev_cs[i]) cudaEventDestroy(c->ev_cs[i]);
        if (c->ev_cc[i]) cudaEventDestroy(c->ev_cc[i]);
    }
    if (c->ev_cbeg) cudaEventDestroy(c->ev_cbeg);
    if (c->ev_cend) cudaEventDestroy(c->ev_cend);
    if (c->copy3) cudaStreamDestroy(c->copy3);
    for (cudaEvent_t e : c->ev_pack3) cudaEventDestroy(e);
    for (cudaEvent_t e : c->ev_copy3) cudaEventDestroy(e);
    cudaFreeHost(c->h_ptrs3);
    cudaFreeHost(c->h_flag);
    cudaFreeHost(c->h_scratch);
    if (c->h_cerr) cudaFreeHost(c->h_cerr);
    delete c;
    return PLEX_OK;
}

plex_status plex_plan_destroy(plex_plan_t plan) {
    if (!plan) return PLEX_OK;
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    for (plex_ctx_s* c : g_ctxs) {
        for (int32_t r = -1; r < plan->p.world; ++r) {     // r >= 0: per-rank emulation tables
            const uint64_t key = r < 0 ? plan->p.id : plan->p.id ^ (0x9E3779B97F4A7C15ull * (uint64_t)(r + 1));
            auto it = c->dev.find(key);
            if (it == c->dev.end()) continue;
            DeviceGuard g(c->device);
            free_devplan(c, it->second);                  // drains the ctx's streams first
            c->dev.erase(it);
        }
    }
    delete plan;
    return PLEX_OK;
}

plex_status plex_ctx_set_carry_staging(plex_ctx_t c, void* staging, uint64_t bytes) {
    if (!c || (bytes && !staging) || (reinterpret_cast<uintptr_t>(staging) % 256)) {
        set_error("bad carry staging");
        return PLEX_E_INVAL;
    }
    c->cstaging = reinterpret_cast<uint8_t*>(staging);
    c->cstaging_bytes = bytes;
    return PLEX_OK;
}

plex_status plex_ctx_stats(plex_ctx_t c, int32_t which, plex_kernel_stats* out) {
    if (!c || !out || which < 0 || which >= PLEX_NUM_STATS) { set_error("bad stats query"); return PLEX_E_INVAL; }
    *out = c->stats[which];
    return PLEX_OK;
}

plex_status plex_ctx_set_flags(plex_ctx_t c, uint32_t value, uint32_t mask) {
    if (!c) { set_error("NULL ctx"); return PLEX_E_INVAL; }
    if (mask & ~(PLEX_CTX_TIMING | PLEX_CTX_SPLIT_PUSH)) { set_error("only TIMING / SPLIT_PUSH may change"); return PLEX_E_INVAL; }
    c->flags = (c->flags & ~mask) | (value & mask);
    return PLEX_OK;
}

plex_status plex_ctx_reset_stats(plex_ctx_t c) {
    if (!c) { set_error("NULL ctx"); return PLEX_E_INVAL; }
    for (auto& s : c->stats) s = plex_kernel_stats{};
    c->trace.clear();
    c->n_calls = 0;
    return PLEX_OK;
}

plex_status plex_ctx_trace(plex_ctx_t c, plex_launch_record* out, int32_t cap, int32_t* n) {
    if (!c || !n) { set_error("NULL argument"); return PLEX_E_INVAL; }
    *n = (int32_t)c->trace.size();
    if (out) std::memcpy(out, c->trace.data(), sizeof(plex_launch_record) * std::min<size_t>(cap, c->trace.size()));
    return PLEX_OK;
}

// ---- slabs ("the host tier uses pinned memory") ---------------
static void slab_unpin(plex_slab_s* s);

static plex_status slab_pin(plex_slab_s* s) {
    const size_t want = std::max<uint64_t>(s->bytes, 4096);
    if (s->flags & PLEX_SLAB_HUGEPAGE) {
        const size_t huge = 2ull << 20;
        const size_t n = align_up(want, huge);
        void* p = mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (p == MAP_FAILED) {
            set_error("mmap of %zu B failed", n);
            return PLEX_E_TIER_FULL;
        }
        madvise(p, n, MADV_HUGEPAGE);
        cudaError_t e = cudaHostRegister(p, n, cudaHostRegisterDefault);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            munmap(p, n);
            set_error("cudaHostRegister(%zu B): %s", n, cudaGetErrorString(e));
            return PLEX_E_TIER_FULL;
        }
        s->host = reinterpret_cast<uint8_t*>(p);
        s->map_bytes = n;
        s->registered = true;
    } else {
        const size_t n = align_up(want, 4096);
        cudaError_t e = cudaHostAlloc(&s->host, n, cudaHostAllocPortable);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            s->host = nullptr;
            set_error("cudaHostAlloc(%zu B): %s", n, cudaGetErrorString(e));
            return PLEX_E_TIER_FULL;
        }
        s->map_bytes = n;
        s->registered = false;
    }
    if (s->carry_bytes) {                       // other ranks' carried buckets (NEXT-1 balancing)
        cudaError_t e = cudaHostAlloc(&s->carry_host, s->carry_bytes, cudaHostAllocPortable);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            s->carry_host = nullptr;
            slab_unpin(s);
            set_error("cudaHostAlloc(%llu B carry region): %s", (unsigned long long)s->carry_bytes,
                      cudaGetErrorString(e));
            return PLEX_E_TIER_FULL;
        }
    }
    return PLEX_OK;
}

static void slab_unpin(plex_slab_s* s) {
    if (s->carry_host) {
        cudaFreeHost(s->carry_host);
        s->carry_host = nullptr;
    }
    if (!s->host) return;
    if (s->registered) {
        cudaHostUnregister(s->host);
        munmap(s->host, s->map_bytes);
    } else {
        cudaFreeHost(s->host);
    }
    s->host = nullptr;
}

plex_status plex_slab_create(plex_plan_t plan, int32_t rank, uint32_t flags, plex_slab_t* out) {
    if (!plan || !out || rank < 0 || rank >= plan->p.world) { set_error("bad slab arguments"); return PLEX_E_INVAL; }
    *out = nullptr;
    const RankPlan& R = plan->p.ranks[rank];
    auto* s = new plex_slab_s();
    s->plan_id = plan->p.id;
    s->rank = rank;
    s->bytes = R.slab_bytes;
    s->flags = flags;
    s->carry_bytes = R.carry_bytes;
    s->cks.assign(2 * R.segs.size(), 0);
    plex_status st = slab_pin(s);
    if (st) {
        delete s;
        return st;
    }
    *out = s;
    return PLEX_OK;
}

plex_status plex_slab_destroy(plex_slab_t s) {
    if (!s) return PLEX_OK;
    slab_unpin(s);
    delete s;
    return PLEX_OK;
}

// ---- NEXT-4 cold tier: spill / fill a slab to NVMe with direct I/O -------------------
// PAPER.md:505-506 (GPU / host / NVMe residency) and :574 ("the NVMe tier
// bypasses the page cache through direct I/O").  The slab's canonical bytes
// go to `path` with O_DIRECT (pinned slab memory is page-aligned and the
// transfer is padded to 4 KiB) by several threads at disjoint offsets, and
// the pinned memory is released: residency DISK.  fill re-pins and reads it
// back: residency HOST; the checksums recorded at offload travel with the
// slab object, so a corrupted file is caught by the next onload.
static plex_status pio(bool write, int fd, uint8_t* buf, size_t n, int threads) {
    const size_t chunk = 64ull << 20;
    std::atomic<size_t> next{0};
    std::atomic<int> err{0};
    auto work = [&]() {
        for (;;) {
            const size_t o = next.fetch_add(chunk);
            if (o >= n || err.load()) return;
            size_t len = std::min(chunk, n - o), done = 0;
            while (done < len) {
                const ssize_t r = write ? pwrite(fd, buf + o + done, len - done, (off_t)(o + done))
                                        : pread(fd, buf + o + done, len - done, (off_t)(o + done));
                if (r <= 0) { err.store(r == 0 ? EIO : errno); return; }
                done += (size_t)r;
            }
        }
    };
    std::vector<std::thread> ts;
    for (int i = 1; i < threads; ++i) ts.emplace_back(work);
    work();
    for (auto& t : ts) t.join();
    if (err.load()) {
        set_error("%s: %s", write ? "pwrite" : "pread", strerror(err.load()));
        return PLEX_E_TIER_FULL;
    }
    return PLEX_OK;
}

plex_status plex_slab_spill(plex_slab_t s, const char* path, int32_t threads) {
    if (!s || !path) { set_error("NULL slab/path"); return PLEX_E_INVAL; }
    if (s->residency != PLEX_RES_HOST || !s->host || s->busy || s->ckpt.load()) { set_error("spill needs a HOST-resident, idle slab"); return PLEX_E_STATE; }
    if (s->carry_bytes) { set_error("spill of a slab with a carry region is not supported"); return PLEX_E_INVAL; }
    const size_t n = align_up(std::max<uint64_t>(s->bytes, 1), 4096);
    int fd = open(path, O_WRONLY | O_CREAT | O_TRUNC | O_DIRECT, 0600);
    if (fd < 0) { set_error("open(%s, O_DIRECT): %s", path, strerror(errno)); return PLEX_E_INVAL; }
    plex_status st = pio(true, fd, s->host, n, std::max(1, threads));
    if (!st && fsync(fd) != 0) { set_error("fsync: %s", strerror(errno)); st = PLEX_E_TIER_FULL; }
    close(fd);
    if (st) return st;
    slab_unpin(s);
    s->residency = PLEX_RES_DISK;
    return PLEX_OK;
}

plex_status plex_slab_fill(plex_slab_t s, const char* path, int32_t threads) {
    if (!s || !path) { set_error("NULL slab/path"); return PLEX_E_INVAL; }
    if (s->residency != PLEX_RES_DISK) { set_error("fill needs a DISK-resident slab"); return PLEX_E_STATE; }
    const size_t n = align_up(std::max<uint64_t>(s->bytes, 1), 4096);
    int fd = open(path, O_RDONLY | O_DIRECT);
    if (fd < 0) { set_error("open(%s, O_DIRECT): %s", path, strerror(errno)); return PLEX_E_INVAL; }
    plex_status st = slab_pin(s);
    if (!st) st = pio(false, fd, s->host, n, std::max(1, threads));
    close(fd);
    if (st) {                   // no partial state change: stay on disk
        slab_unpin(s);
        return st;
    }
    s->residency = PLEX_RES_HOST;
    return PLEX_OK;
}

// ---- NEXT-3 checkpoint materialisation from the offloaded state -----------------------
// checkpoints are "materialization" of managed (possibly
// offloaded) state, done in the background off the critical path.  A HOST
// slab is written as a standard safetensors file (u64 LE header length, JSON
// header, raw little-endian data): one tensor per slab segment, named by its
// logical key (PARAM, bf16) or "optimizer.<kind>.<key>" (fp32), shaped as this
// rank's FSDP shard, data in slab order without the 256-B padding.  The
// header metadata carries world, rank and the (S1, S2) checksums recorded at
// offload, so a restored slab is verified by the next onload like any other.
static const char* kCkptKind[4] = {"param", "master", "exp_avg", "exp_avg_sq"};

static std::string ckpt_header(const Plan& p, int32_t rank, const std::vector<uint64_t>& cks) {
    const RankPlan& R = p.ranks[rank];
    std::string h = "{\"__metadata__\":{\"format\":\"pt\",\"plex.layout\":\"fsdp-dim0\",\"plex.world\":\"" +
                    std::to_string(p.world) + "\",\"plex.rank\":\"" + std::to_string(rank) + "\",\"plex.checksums\":\"";
    char buf[40];
    for (size_t i = 0; i < cks.size(); ++i) {
        snprintf(buf, sizeof(buf), "%s%016llx", i ? "," : "", (unsigned long long)cks[i]);
        h += buf;
    }
    h += "\"}";
    uint64_t off = 0;
    for (const plex_seg_desc& d : R.seg_desc) {
        const Tensor& T = p.tensors[d.tensor];
        std::string name = d.kind == PLEX_KIND_PARAM ? T.key : std::string("optimizer.") + kCkptKind[d.kind] + "." + T.key;
        std::string esc;
        for (char ch : name) {
            if (ch == '"' || ch == '\\') esc += '\\';
            esc += ch;
        }
        h += ",\"" + esc + "\":{\"dtype\":\"" + (d.kind == PLEX_KIND_PARAM ? "BF16" : "F32") + "\",\"shape\":[" +
             std::to_string(d.row1 - d.row0) + (T.ndim == 2 ? "," + std::to_string(T.d1) : std::string()) +
             "],\"data_offsets\":[" + std::to_string(off) + "," + std::to_string(off + d.nbytes) + "]}";
        off += d.nbytes;
    }
    h += "}";
    while ((8 + h.size()) % 8) h += ' ';
    return h;
}

// Segment pieces (file offset, slab offset, bytes) in <= 64 MiB chunks, run by `threads` workers.
static plex_status ckpt_io(bool write, int fd, const RankPlan& R, uint8_t* host, uint64_t data0, int threads) {
    struct Piece { uint64_t fo, so, n; };
    std::vector<Piece> pcs;
    uint64_t fo = data0;
    for (const plex_seg_desc& d : R.seg_desc) {
        for (uint64_t o = 0; o < d.nbytes; o += 64ull << 20)
            pcs.push_back(Piece{fo + o, d.slab_offset + o, std::min<uint64_t>(64ull << 20, d.nbytes - o)});
        fo += d.nbytes;
    }
    std::atomic<size_t> next{0};
    std::atomic<int> err{0};
    auto work = [&]() {
        for (;;) {
            const size_t i = next.fetch_add(1);
            if (i >= pcs.size() || err.load()) return;
            const Piece& q = pcs[i];
            size_t done = 0;
            while (done < q.n) {
                const ssize_t r = write ? pwrite(fd, host + q.so + done, q.n - done, (off_t)(q.fo + done))
                                        : pread(fd, host + q.so + done, q.n - done, (off_t)(q.fo + done));
                if (r <= 0) { err.store(r == 0 ? EIO : errno); return; }
                done += (size_t)r;
            }
        }
    };
    std::vector<std::thread> ts;
    for (int i = 1; i < threads; ++i) ts.emplace_back(work);
    work();
    for (auto& t : ts) t.join();
    if (err.load()) {
        set_error("checkpoint %s: %s", write ? "pwrite" : "pread", strerror(err.load()));
        return PLEX_E_TIER_FULL;
    }
    return PLEX_OK;
}

static plex_status ckpt_check(plex_plan_t plan, plex_slab_t s, const char* path) {
    if (!plan || !s || !path) { set_error("NULL plan/slab/path"); return PLEX_E_INVAL; }
    if (s->plan_id != plan->p.id) { set_error("slab does not belong to this plan"); return PLEX_E_INVAL; }
    if (plan->p.ranks[s->rank].carried_out) { set_error("checkpoint of a slab with carried buckets is not supported"); return PLEX_E_INVAL; }
    return PLEX_OK;
}

// The slab becomes read-only (ckpt > 0) in the CALLER's thread, before any
// background writer starts, under the slab mutex that restore also takes.
static plex_status ckpt_begin(plex_plan_t plan, plex_slab_t s, const char* path) {
    plex_status st = ckpt_check(plan, s, path);
    if (st) return st;
    std::lock_guard<std::mutex> lk(s->mu);
    if (s->residency != PLEX_RES_HOST || !s->host || !s->written) { set_error("checkpoint needs an offloaded (HOST) slab"); return PLEX_E_STATE; }
    if (s->elided) { set_error("slab holds derived (elided) params: offload without elision to checkpoint"); return PLEX_E_STATE; }
    if (s->busy) { set_error("an async transfer or a restore of this slab is in flight"); return PLEX_E_STATE; }
    s->ckpt.fetch_add(1);
    return PLEX_OK;
}

// The write itself (slab already marked by ckpt_begin; unmarks it).
static plex_status ckpt_write(plex_plan_t plan, plex_slab_t s, const char* path, int32_t threads) {
    plex_status st = PLEX_OK;
    const Plan& p = plan->p;
    const std::string h = ckpt_header(p, s->rank, s->cks);
    int fd = open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (fd < 0) { s->ckpt.fetch_sub(1); set_error("open(%s): %s", path, strerror(errno)); return PLEX_E_INVAL; }
    uint8_t len8[8];
    for (int i = 0; i < 8; ++i) len8[i] = (uint8_t)((uint64_t)h.size() >> (8 * i));
    if (pwrite(fd, len8, 8, 0) != 8 || pwrite(fd, h.data(), h.size(), 8) != (ssize_t)h.size()) {
        set_error("checkpoint header write: %s", strerror(errno));
        st = PLEX_E_TIER_FULL;
    }
    if (!st) st = ckpt_io(true, fd, p.ranks[s->rank], s->host, 8 + h.size(), std::max(1, threads));
    if (!st && fsync(fd) != 0) { set_error("fsync: %s", strerror(errno)); st = PLEX_E_TIER_FULL; }
    close(fd);
    s->ckpt.fetch_sub(1);
    return st;
}

plex_status plex_slab_checkpoint(plex_plan_t plan, plex_slab_t s, const char* path, int32_t threads) {
    plex_status st = ckpt_begin(plan, s, path);
    return st ? st : ckpt_write(plan, s, path, threads);
}

plex_status plex_slab_checkpoint_start(plex_plan_t plan, plex_slab_t s, const char* path, int32_t threads,
                                       plex_ckpt_t* out) {
    if (!out) { set_error("NULL out"); return PLEX_E_INVAL; }
    *out = nullptr;
    plex_status st = ckpt_begin(plan, s, path);
    if (st) return st;
    auto* h = new plex_ckpt_s();
    const std::string pth(path);
    try {
        h->th = std::thread([h, plan, s, pth, threads]() {
            h->status = ckpt_write(plan, s, pth.c_str(), threads);
            if (h->status) h->error = plex_last_error();
        });
    } catch (...) {
        s->ckpt.fetch_sub(1);
        delete h;
        set_error("cannot start the checkpoint thread");
        return PLEX_E_INVAL;
    }
    *out = h;
    return PLEX_OK;
}

plex_status plex_ckpt_wait(plex_ckpt_t h) {
    if (!h) { set_error("NULL checkpoint handle"); return PLEX_E_INVAL; }
    if (h->th.joinable()) h->th.join();
    const plex_status st = h->status;
    if (st) set_error("%s", h->error.c_str());
    delete h;
    return st;
}

plex_status plex_slab_restore(plex_plan_t plan, plex_slab_t s, const char* path, int32_t threads) {
    plex_status st = ckpt_check(plan, s, path);
    if (st) return st;
    {
        std::lock_guard<std::mutex> lk(s->mu);
        if (s->ckpt.load() || s->busy.load()) { set_error("slab is busy (checkpoint, restore or async transfer)"); return PLEX_E_STATE; }
        s->busy = true;
    }
    const Plan& p = plan->p;
    const RankPlan& R = p.ranks[s->rank];
    int fd = open(path, O_RDONLY);
    if (fd < 0) { s->busy = false; set_error("open(%s): %s", path, strerror(errno)); return PLEX_E_INVAL; }
    auto fail = [&](plex_status code) { close(fd); s->busy = false; return code; };
    uint8_t len8[8];
    if (pread(fd, len8, 8, 0) != 8) { set_error("checkpoint too short"); return fail(PLEX_E_LAYOUT); }
    uint64_t hl = 0;
    for (int i = 0; i < 8; ++i) hl |= (uint64_t)len8[i] << (8 * i);
    if (hl > (64ull << 20)) { set_error("checkpoint header of %llu B", (unsigned long long)hl); return fail(PLEX_E_LAYOUT); }
    std::string h(hl, '\0');
    if (pread(fd, &h[0], hl, 8) != (ssize_t)hl) { set_error("checkpoint header read"); return fail(PLEX_E_LAYOUT); }
    // checksums from the metadata; the rest must be exactly what this plan/rank writes
    std::vector<uint64_t> cks(2 * R.segs.size(), 0);
    const std::string tag = "\"plex.checksums\":\"";
    const size_t a = h.find(tag);
    if (a == std::string::npos) { set_error("checkpoint carries no plex checksums"); return fail(PLEX_E_LAYOUT); }
    size_t q = a + tag.size();
    for (size_t i = 0; i < cks.size(); ++i) {
        if (i && (q >= h.size() || h[q++] != ',')) { set_error("checkpoint checksum list too short"); return fail(PLEX_E_LAYOUT); }
        if (q + 16 > h.size()) { set_error("checkpoint checksum list truncated"); return fail(PLEX_E_LAYOUT); }
        cks[i] = strtoull(h.substr(q, 16).c_str(), nullptr, 16);
        q += 16;
    }
    if (h != ckpt_header(p, s->rank, cks)) {
        set_error("checkpoint does not match this plan/rank (tensor names, shapes or order differ)");
        return fail(PLEX_E_LAYOUT);
    }
    const off_t size = lseek(fd, 0, SEEK_END);
    if (size != (off_t)(8 + hl + R.payload_bytes)) { set_error("checkpoint data size mismatch"); return fail(PLEX_E_LAYOUT); }
    if (!s->host && (st = slab_pin(s))) return fail(st);
    if ((st = ckpt_io(false, fd, R, s->host, 8 + hl, std::max(1, threads)))) {
        s->written = false;                                // the slab now holds no valid state
        s->residency = PLEX_RES_DEVICE;
        return fail(st);
    }
    uint64_t cur = 0;                                      // zero the padding (R4)
    for (const plex_seg_desc& d : R.seg_desc) {
        if (d.slab_offset > cur) std::memset(s->host + cur, 0, d.slab_offset - cur);
        cur = d.slab_offset + d.nbytes;
    }
    if (s->bytes > cur) std::memset(s->host + cur, 0, s->bytes - cur);
    s->cks = cks;
    s->written = true;
    s->elided = false;
    s->residency = PLEX_RES_HOST;
    return fail(PLEX_OK);
}

plex_status plex_slab_info(plex_slab_t s, void** host_ptr, uint64_t* bytes, int32_t* residency) {
    if (!s) { set_error("NULL slab"); return PLEX_E_INVAL; }
    if (host_ptr) *host_ptr = s->host;
    if (bytes) *bytes = s->bytes;
    if (residency) *residency = s->residency;
    return PLEX_OK;
}

plex_status plex_slab_carry(plex_slab_t s, void** host_ptr, uint64_t* bytes) {
    if (!s) { set_error("NULL slab"); return PLEX_E_INVAL; }
    if (host_ptr) *host_ptr = s->carry_host;
    if (bytes) *bytes = s->carry_bytes;
    return PLEX_OK;
}

plex_status plex_slab_elided(plex_slab_t s, int32_t* elided) {
    if (!s || !elided) { set_error("NULL argument"); return PLEX_E_INVAL; }
    *elided = s->elided ? 1 : 0;
    return PLEX_OK;
}

plex_status plex_slab_checksums(plex_slab_t s, uint64_t* out, int32_t n) {
    if (!s || !out || (size_t)n != s->cks.size()) { set_error("need %zu entries", s ? s->cks.size() : 0); return PLEX_E_INVAL; }
    std::memcpy(out, s->cks.data(), 8 * s->cks.size());
    return PLEX_OK;
}

// ---- a3 + a4: suspend -----------------------------------------------------------
plex_status plex_state_offload(plex_ctx_t c, plex_plan_t plan, const void* const* src, int32_t n_src, plex_slab_t slab,
                               void* caller_stream) {
    plex_status st = check_common(c, plan);
    if (st || (st = check_slab(c, plan, slab, slab && slab->residency != PLEX_RES_HOST)) || (st = check_no_async(c)))
        return st;
    if (slab->residency == PLEX_RES_HOST) return PLEX_OK;     // idempotent
    if (slab->residency == PLEX_RES_DISK) { set_error("slab is on the NVMe tier"); return PLEX_E_STATE; }
    DeviceGuard g(c->device);
    NvtxRange nv("plex_state_offload");
    Half h{&plan->p, &plan->p.ranks[c->rank], nullptr, slab, 0, {}, false, 0, nullptr, nullptr, nullptr};
    if ((st = fill_state_ptrs(c, plan->p, src, n_src)) || (st = get_devplan(c, plan->p, &h.d))) return st;
    Pipe pp{c->staging, c->n_slots, c->ev_pack.data(), c->ev_copy.data(), c->pack, c->copy, c->h_ptrs, c->d_ptrs,
            c->d_ctr, c->d_flag, c->h_flag};
    cudaStream_t caller = reinterpret_cast<cudaStream_t>(caller_stream);
    CK(cudaEventRecord(c->ev_caller, caller));
    CK(cudaStreamWaitEvent(c->pack, c->ev_caller, 0));
    CK(cudaStreamWaitEvent(c->copy, c->ev_caller, 0));
    if ((st = off_begin(c, pp, h)) || (st = carry_out(c, pp, h))) return st;
    for (int32_t b = 0; b < h.nb; ++b)
        if ((st = off_bucket(c, pp, h, b))) return st;
    if ((st = carry_join(c, pp, h)) || (st = off_end(c, pp, h)) || (st = finish(c, caller))) return st;
    off_collect(h);
    slab->cks.swap(h.cks);
    slab->residency = PLEX_RES_HOST;
    slab->written = true;
    slab->elided = h.elide;
    return PLEX_OK;
}

// ---- a6 + a7: resume ---------------------------------------------------------------
plex_status plex_state_onload(plex_ctx_t c, plex_plan_t plan, plex_slab_t slab, void* const* dst, int32_t n_dst,
                              void* caller_stream) {
    plex_status st = check_common(c, plan);
    if (st || (st = check_slab(c, plan, slab)) || (st = check_no_async(c))) return st;
    if (slab->residency == PLEX_RES_DEVICE) {
        if (!slab->written) { set_error("slab holds no offloaded state"); return PLEX_E_STATE; }
        return PLEX_OK;                                     // idempotent
    }
    if (slab->residency == PLEX_RES_DISK) { set_error("slab is on the NVMe tier: plex_slab_fill first"); return PLEX_E_STATE; }
    DeviceGuard g(c->device);
    NvtxRange nv("plex_state_onload");
    Half h{&plan->p, &plan->p.ranks[c->rank], nullptr, slab, 0, {}, false, 0, nullptr, nullptr, nullptr};
    if ((st = fill_state_ptrs(c, plan->p, reinterpret_cast<const void* const*>(dst), n_dst)) ||
        (st = get_devplan(c, plan->p, &h.d)))
        return st;
    Pipe pp{c->staging, c->n_slots, c->ev_pack.data(), c->ev_copy.data(), c->pack, c->copy, c->h_ptrs, c->d_ptrs,
            c->d_ctr, c->d_flag, c->h_flag};
    cudaStream_t caller = reinterpret_cast<cudaStream_t>(caller_stream);
    CK(cudaEventRecord(c->ev_caller, caller));
    CK(cudaStreamWaitEvent(c->pack, c->ev_caller, 0));
    CK(cudaStreamWaitEvent(c->copy, c->ev_caller, 0));
    if ((st = on_begin(c, pp, h)) || (st = carry_in(c, pp, h))) return st;
    for (int32_t b = 0; b < h.nb; ++b)
        if ((st = on_bucket(c, pp, h, b))) return st;
    if ((st = carry_join(c, pp, h)) || (st = on_end(c, pp, h)) || (st = finish(c, caller))) return st;
    if (*pp.h_flag) {
        set_error("onload: %d segment checksum(s) differ from offload", *pp.h_flag);
        return PLEX_E_CHECKSUM;
    }
    slab->residency = PLEX_RES_DEVICE;
    return PLEX_OK;
}

// ---- NEXT-1: duplex switch -----------------------------------------------------------
// Offload the resident job A and onload the incoming job B at the same time:
// A's buckets stream D2H on the ctx copy stream while B's stream H2D on a
// second, library-owned copy stream, so the two directions of the host link
// run concurrently and C_setup = T_offload + T_load (Eq. 3)
// becomes ~max(T_offload, T_load).  Staging holds both rings back to back.
plex_status plex_state_switch(plex_ctx_t c, plex_plan_t plan_out, const void* const* src_out, int32_t n_src,
                              plex_slab_t slab_out, plex_plan_t plan_in, plex_slab_t slab_in, void* const* dst_in,
                              int32_t n_dst, void* caller_stream) {
    plex_status st = check_common(c, plan_out);
    if (st || (st = check_common(c, plan_in)) ||
        (st = check_slab(c, plan_out, slab_out, slab_out && slab_out->residency != PLEX_RES_HOST)) ||
        (st = check_slab(c, plan_in, slab_in)) || (st = check_no_async(c)))
        return st;
    if (slab_out == slab_in) { set_error("switch needs two different slabs"); return PLEX_E_INVAL; }
    if (slab_in->residency == PLEX_RES_DEVICE && !slab_in->written) {
        set_error("incoming slab holds no offloaded state");
        return PLEX_E_STATE;
    }
    const uint64_t need = (uint64_t)c->n_slots * (plan_out->p.bucket + plan_in->p.bucket);
    if (c->staging_bytes < need) {
        set_error("switch needs staging >= n_slots x (bucket_out + bucket_in) = %llu B", (unsigned long long)need);
        return PLEX_E_INVAL;
    }
    DeviceGuard g(c->device);
    NvtxRange nv("plex_state_switch");
    const bool do_off = slab_out->residency == PLEX_RES_DEVICE;
    const bool do_on = slab_in->residency == PLEX_RES_HOST;
    Half ho{&plan_out->p, &plan_out->p.ranks[c->rank], nullptr, slab_out, 0, {}, false, 0, nullptr, nullptr, nullptr};
    Half hi{&plan_in->p, &plan_in->p.ranks[c->rank], nullptr, slab_in, 0, {}, false, 0, nullptr, nullptr, nullptr};
    if (do_off && ((st = fill_state_ptrs(c, plan_out->p, src_out, n_src, 0)) || (st = get_devplan(c, plan_out->p, &ho.d))))
        return st;
    if (do_on && ((st = fill_state_ptrs(c, plan_in->p, reinterpret_cast<const void* const*>(dst_in), n_dst, 1)) ||
                  (st = get_devplan(c, plan_in->p, &hi.d))))
        return st;
    if (!c->copy2) {
        CK(cudaStreamCreateWithFlags(&c->copy2, cudaStreamNonBlocking));
        c->ev_pack2.resize(c->n_slots);
        c->ev_copy2.resize(c->n_slots);
        for (int i = 0; i < c->n_slots; ++i) {
            CK(cudaEventCreateWithFlags(&c->ev_pack2[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c->ev_copy2[i], cudaEventDisableTiming));
        }
    }
    Pipe po{c->staging, c->n_slots, c->ev_pack.data(), c->ev_copy.data(), c->pack, c->copy, c->h_ptrs, c->d_ptrs,
            c->d_ctr, c->d_flag + 2, c->h_flag + 2};
    // Both halves' kernels share the pack stream.  The two rings run at the
    // host link's pace and would otherwise launch their pack/unpack kernels at
    // the same moments (phase-locked), halving each kernel's SMs; serialised,
    // each launch gets the whole GPU, and since kernels take ~1 % of a bucket's
    // copy time the coupling costs nothing (measured: 1545-1574 vs 1584-1612 ms
    // per 7B N=2 step, kernels at 0.94-0.96 vs 0.87-0.89 of HBM).
    Pipe pi{c->staging + (uint64_t)c->n_slots * plan_out->p.bucket, c->n_slots, c->ev_pack2.data(),
            c->ev_copy2.data(), c->pack, c->copy2, c->h_ptrs2, c->d_ptrs2, c->d_ctr + 1, c->d_flag + 1,
            c->h_flag + 1};
    cudaStream_t caller = reinterpret_cast<cudaStream_t>(caller_stream);
    CK(cudaEventRecord(c->ev_caller, caller));
    for (cudaStream_t s2 : {c->pack, c->copy, c->copy2}) CK(cudaStreamWaitEvent(s2, c->ev_caller, 0));
    if (do_off && ((st = off_begin(c, po, ho)) || (st = carry_out(c, po, ho)))) return st;
    if (do_on && ((st = on_begin(c, pi, hi)) || (st = carry_in(c, pi, hi)))) return st;
    const int32_t no = do_off ? ho.nb : 0, ni = do_on ? hi.nb : 0;
    for (int32_t k = 0; k < std::max(no, ni); ++k) {   // interleave so both directions start at once
        if (k < no && (st = off_bucket(c, po, ho, k))) return st;
        if (k < ni && (st = on_bucket(c, pi, hi, k))) return st;
    }
    if (do_off && ((st = carry_join(c, po, ho)) || (st = off_end(c, po, ho)))) return st;
    if (do_on && ((st = carry_join(c, pi, hi)) || (st = on_end(c, pi, hi)))) return st;
    CK(cudaEventRecord(c->ev_pack_done, c->copy2));
    CK(cudaStreamWaitEvent(caller, c->ev_pack_done, 0));
    CK(cudaStreamSynchronize(c->copy2));
    if ((st = finish(c, caller))) return st;
    if (do_off) {
        off_collect(ho);
        slab_out->cks.swap(ho.cks);
        slab_out->residency = PLEX_RES_HOST;
        slab_out->written = true;
        slab_out->elided = ho.elide;
    }
    if (do_on) {
        if (*pi.h_flag) {
            set_error("switch onload: %d segment checksum(s) differ from offload", *pi.h_flag);
            return PLEX_E_CHECKSUM;
        }
        slab_in->residency = PLEX_RES_DEVICE;
    }
    return PLEX_OK;
}

// ---- NEXT-1: in-place swap of two same-layout jobs ---------------------------------------
// PAPER.md:555 context switch when the GPU group holds ONE job's device state
// (R17) and the host ONE slab: the resident job A's state goes out of the
// device tensors into the slab while the incoming job B's state comes from the
// same slab into the same tensors.  Per bucket k: H2D B_k (slab -> in ring) ;
// pack A_k (tensors -> out ring) ; unpack B_k (in ring -> tensors, after pack
// A_k on the same kernel stream) ; D2H A_k (out ring -> slab, after H2D B_k
// has read that slab range).  D2H A_k overlaps H2D B_{k+1}: both directions of
// the host link stay busy with a single copy of each job's state.
plex_status plex_state_swap(plex_ctx_t c, plex_plan_t plan, void* const* state, int32_t n_state, plex_slab_t slab,
                            void* caller_stream) {
    plex_status st = check_common(c, plan);
    if (st || (st = check_slab(c, plan, slab, true)) || (st = check_no_async(c))) return st;
    const Plan& p = plan->p;
    if (slab->residency != PLEX_RES_HOST || !slab->written) { set_error("swap needs the incoming job's state in the slab (HOST)"); return PLEX_E_STATE; }
    if (p.ranks[c->rank].carried_out || p.ranks[c->rank].carried_in) { set_error("swap with carried buckets is not supported"); return PLEX_E_INVAL; }
    if (c->staging_bytes < 2ull * c->n_slots * p.bucket) {
        set_error("swap needs staging >= 2 x n_slots x bucket = %llu B", (unsigned long long)(2ull * c->n_slots * p.bucket));
        return PLEX_E_INVAL;
    }
    DeviceGuard g(c->device);
    NvtxRange nv("plex_state_swap");
    const void* const* ptrs = reinterpret_cast<const void* const*>(state);
    Half ho{&p, &p.ranks[c->rank], nullptr, slab, 0, {}, false, 0, nullptr, nullptr, nullptr};
    if ((st = fill_state_ptrs(c, p, ptrs, n_state, 0)) || (st = fill_state_ptrs(c, p, ptrs, n_state, 1)) ||
        (st = get_devplan(c, p, &ho.d)))
        return st;
    Half hi = ho;
    if (!c->copy2) {
        CK(cudaStreamCreateWithFlags(&c->copy2, cudaStreamNonBlocking));
        c->ev_pack2.resize(c->n_slots);
        c->ev_copy2.resize(c->n_slots);
        for (int i = 0; i < c->n_slots; ++i) {
            CK(cudaEventCreateWithFlags(&c->ev_pack2[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c->ev_copy2[i], cudaEventDisableTiming));
        }
    }
    if (c->ev_piece.empty()) {
        c->ev_piece.resize((size_t)c->n_slots * kSwapPieces);
        for (auto& e : c->ev_piece) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    Pipe po{c->staging, c->n_slots, c->ev_pack.data(), c->ev_copy.data(), c->pack, c->copy, c->h_ptrs, c->d_ptrs,
            c->d_ctr, c->d_flag + 2, c->h_flag + 2};
    Pipe pi{c->staging + (uint64_t)c->n_slots * p.bucket, c->n_slots, c->ev_pack2.data(), c->ev_copy2.data(), c->pack,
            c->copy2, c->h_ptrs2, c->d_ptrs2, c->d_ctr + 1, c->d_flag + 1, c->h_flag + 1};
    cudaStream_t caller = reinterpret_cast<cudaStream_t>(caller_stream);
    CK(cudaEventRecord(c->ev_caller, caller));
    for (cudaStream_t s2 : {c->pack, c->copy, c->copy2}) CK(cudaStreamWaitEvent(s2, c->ev_caller, 0));
    // on_begin uploads B's recorded checksums before anything overwrites the slab's;
    // off_begin runs A's NEXT-2 derivability check (elision plans)
    if ((st = on_begin(c, pi, hi)) || (st = off_begin(c, po, ho))) return st;
    const RankPlan& R = p.ranks[c->rank];
    // Grids (NEXT-2): B elided -> both halves walk the shifted grid from the first
    // MASTER byte; if A's params are not derivable its PARAM prefix goes out
    // first on its own (B never reads slab bytes below that point).  B stored
    // in full -> A goes in full too, even if derivable.
    bool a_prefix = false;
    if (!hi.elide && ho.elide) {
        CK(cudaMemsetAsync(ho.d->cks, 0, 16 * std::max<size_t>(1, R.segs.size()), po.kern));
        use_grid(ho, false);
    } else if (hi.elide && !ho.elide) {
        a_prefix = true;
        use_grid(ho, true);
    }
    const bool shifted = hi.elide;
    int32_t oseq = 0;                                   // out-ring sequence number (slot = oseq % n_slots)
    cudaEvent_t ta = nullptr;
    if (a_prefix) {                                     // A's PARAM prefix [0, elide_start), full-grid buckets
        const uint64_t e0 = R.elide_start;
        for (int32_t k = 0; (uint64_t)k * p.bucket < e0; ++k, ++oseq) {
            const int slot = oseq % c->n_slots;
            uint8_t* so = po.staging + (uint64_t)slot * p.bucket;
            const uint64_t lo = (uint64_t)k * p.bucket, hi_b = std::min<uint64_t>(e0, lo + p.bucket);
            const uint64_t i0 = R.bucket_item_start[k];
            const uint64_t i1 = std::min<uint64_t>(R.bucket_item_start[k + 1], R.n_param_items);
            if (oseq >= c->n_slots) CK(cudaStreamWaitEvent(po.kern, po.ev_c[slot], 0));
            if ((st = tbeg(c, po, po.kern, &ta))) return st;
            CK(launch_pack(true, ho.d->items + i0, (uint32_t)(i1 - i0), ho.d->segs, po.d_ptrs, so, lo, ho.d->cks,
                           po.ctr, po.kern));
            if ((st = tend(c, po, po.kern, ta, PLEX_STAT_PACK, 2 * (hi_b - lo)))) return st;
            CK(cudaEventRecord(po.ev_k[slot], po.kern));
            CK(cudaStreamWaitEvent(po.copy, po.ev_k[slot], 0));
            if ((st = tbeg(c, po, po.copy, &ta))) return st;
            CK(cudaMemcpyAsync(slab->host + lo, so, hi_b - lo, cudaMemcpyDeviceToHost, po.copy));
            if ((st = tend(c, po, po.copy, ta, PLEX_STAT_D2H, hi_b - lo))) return st;
            CK(cudaEventRecord(po.ev_c[slot], po.copy));
        }
    }
    const int32_t nb = shifted ? hi.nb : ho.nb;
    const uint64_t base = shifted ? R.elide_start : 0;
    for (int32_t k = 0; k < nb; ++k, ++oseq) {
        const int si_slot = k % c->n_slots, so_slot = oseq % c->n_slots;
        uint8_t* so = po.staging + (uint64_t)so_slot * p.bucket;
        uint8_t* si = pi.staging + (uint64_t)si_slot * p.bucket;
        const uint64_t lo = base + (uint64_t)k * p.bucket;
        const uint64_t len = std::min<uint64_t>(p.bucket, R.slab_bytes - lo);
        const uint64_t i0 = hi.bstart[k], i1 = hi.bstart[k + 1];
        // H2D B_k, in pieces: A_k's D2H may overwrite a slab range as soon as
        // B_k's piece of it has been read, so the first and last buckets (which
        // run one direction alone) shrink to one piece each
        const uint64_t np = std::min<uint64_t>(swap_pieces(), std::max<uint64_t>(1, len / 4096));
        const uint64_t ps = ((len + np - 1) / np + 255) & ~255ull;
        if (k >= c->n_slots) CK(cudaStreamWaitEvent(pi.copy, pi.ev_k[si_slot], 0));
        for (uint64_t j = 0; j * ps < len; ++j) {
            const uint64_t o = j * ps, n = std::min(ps, len - o);
            if ((st = tbeg(c, pi, pi.copy, &ta))) return st;
            CK(cudaMemcpyAsync(si + o, slab->host + lo + o, n, cudaMemcpyHostToDevice, pi.copy));
            if ((st = tend(c, pi, pi.copy, ta, PLEX_STAT_H2D, n))) return st;
            CK(cudaEventRecord(c->ev_piece[(size_t)si_slot * kSwapPieces + j], pi.copy));
        }
        CK(cudaEventRecord(pi.ev_c[si_slot], pi.copy));
        // pack A_k
        if (oseq >= c->n_slots) CK(cudaStreamWaitEvent(po.kern, po.ev_c[so_slot], 0));
        if ((st = tbeg(c, po, po.kern, &ta))) return st;
        CK(launch_pack(true, hi.grid_items + i0, (uint32_t)(i1 - i0), ho.d->segs, po.d_ptrs, so, lo, ho.d->cks, po.ctr,
                       po.kern));
        if ((st = tend(c, po, po.kern, ta, PLEX_STAT_PACK, 2 * hi.payload[k]))) return st;
        CK(cudaEventRecord(po.ev_k[so_slot], po.kern));
        // unpack B_k (same stream: after pack A_k read these tensor bytes)
        CK(cudaStreamWaitEvent(pi.kern, pi.ev_c[si_slot], 0));
        if ((st = tbeg(c, pi, pi.kern, &ta))) return st;
        CK(launch_pack(false, hi.grid_items + i0, (uint32_t)(i1 - i0), hi.d->segs, pi.d_ptrs, si, lo, hi.d->cks_in,
                       pi.ctr, pi.kern));
        if ((st = tend(c, pi, pi.kern, ta, PLEX_STAT_UNPACK, 2 * hi.payload[k]))) return st;
        CK(cudaEventRecord(pi.ev_k[si_slot], pi.kern));
        // D2H A_k, piece j after H2D B_k has read that piece of the slab range
        CK(cudaStreamWaitEvent(po.copy, po.ev_k[so_slot], 0));
        for (uint64_t j = 0; j * ps < len; ++j) {
            const uint64_t o = j * ps, n = std::min(ps, len - o);
            CK(cudaStreamWaitEvent(po.copy, c->ev_piece[(size_t)si_slot * kSwapPieces + j], 0));
            if ((st = tbeg(c, po, po.copy, &ta))) return st;
            CK(cudaMemcpyAsync(slab->host + lo + o, so + o, n, cudaMemcpyDeviceToHost, po.copy));
            if ((st = tend(c, po, po.copy, ta, PLEX_STAT_D2H, n))) return st;
        }
        CK(cudaEventRecord(po.ev_c[so_slot], po.copy));
    }
    // on_end re-derives B's params (elided) after every A pack on the same stream
    if ((st = off_end(c, po, ho)) || (st = on_end(c, pi, hi))) return st;
    CK(cudaEventRecord(c->ev_pack_done, c->copy2));
    CK(cudaStreamWaitEvent(caller, c->ev_pack_done, 0));
    CK(cudaStreamSynchronize(c->copy2));
    if ((st = finish(c, caller))) return st;
    off_collect(ho);
    slab->cks.swap(ho.cks);                    // the slab now holds A (checksums recorded by its pack)
    slab->residency = PLEX_RES_HOST;
    slab->written = true;
    slab->elided = shifted && !a_prefix;
    if (*pi.h_flag) {
        set_error("swap: %d segment checksum(s) of the incoming state differ from its offload", *pi.h_flag);
        return PLEX_E_CHECKSUM;
    }
    return PLEX_OK;
}

// ---- NEXT-1: scheduler-directed prefetch and asynchronous drain -----------------------
// PAPER.md:506 "when an upcoming context switch is predicted, StateManager can
// proactively move state upward in the hierarchy before the corresponding
// deployment becomes active"; :513 "state can be prefetched or drained across
// the memory hierarchy asynchronously", keeping "only operations that directly
// access or mutate the active GPU-resident deployment" on the critical path.
// A drain (offload) / prefetch (onload) is enqueued on library-owned side
// streams and returns at once; the caller keeps computing; plex_state_wait
// completes it (verify, residency flip, caller-stream ordering).
}  // extern "C"

namespace plex {
static plex_status async_resources(plex_ctx_s* c) {
    if (!c->kasync) CK(cudaStreamCreateWithFlags(&c->kasync, cudaStreamNonBlocking));
    if (!c->copy2) CK(cudaStreamCreateWithFlags(&c->copy2, cudaStreamNonBlocking));
    if (!c->copy3) CK(cudaStreamCreateWithFlags(&c->copy3, cudaStreamNonBlocking));
    auto mk = [&](std::vector<cudaEvent_t>& v) -> plex_status {
        if (!v.empty()) return PLEX_OK;
        v.resize(c->n_slots);
        for (auto& e : v) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        return PLEX_OK;
    };
    plex_status st;
    if ((st = mk(c->ev_pack2)) || (st = mk(c->ev_copy2)) || (st = mk(c->ev_pack3)) || (st = mk(c->ev_copy3))) return st;
    return PLEX_OK;
}

}  // namespace plex

extern "C" {

plex_status plex_state_drain(plex_ctx_t c, plex_plan_t plan, const void* const* src, int32_t n_src, plex_slab_t slab,
                             void* caller_stream) {
    plex_status st = check_common(c, plan);
    if (st || (st = check_slab(c, plan, slab, slab && slab->residency != PLEX_RES_HOST))) return st;
    if (c->async[0]) { set_error("a drain is already in flight"); return PLEX_E_STATE; }
    if (!plan->p.carry.empty()) { set_error("async drain does not support carried buckets"); return PLEX_E_INVAL; }
    if (slab->residency != PLEX_RES_DEVICE) return PLEX_OK;      // already offloaded: nothing to drain
    if ((uint64_t)c->n_slots * plan->p.bucket > c->staging_bytes / 2) {
        set_error("async transfers need staging >= 2 x n_slots x bucket");
        return PLEX_E_INVAL;
    }
    DeviceGuard g(c->device);
    NvtxRange nv("plex_state_drain");
    if ((st = async_resources(c)) || (st = fill_state_ptrs(c, plan->p, src, n_src, 2))) return st;
    auto* a = new AsyncState();
    a->h = Half{&plan->p, &plan->p.ranks[c->rank], nullptr, slab, 0, {}, false, 0, nullptr, nullptr, nullptr};
    a->pp = Pipe{c->staging, c->n_slots, c->ev_pack3.data(), c->ev_copy3.data(), c->kasync, c->copy3, c->h_ptrs3,
                 c->d_ptrs3, c->d_ctr + 2, c->d_flag + 3, c->h_flag + 3, true};
    a->slab = slab;
    auto fail = [&](plex_status e) { async_free(a); return e; };
    if ((st = get_devplan(c, plan->p, &a->h.d))) return fail(st);
    if (cudaEventCreateWithFlags(&a->done_k, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&a->done_c, cudaEventDisableTiming) != cudaSuccess) {
        (void)cudaGetLastError();
        set_error("cudaEventCreate failed");
        return fail(PLEX_E_CUDA);
    }
    cudaStream_t caller = reinterpret_cast<cudaStream_t>(caller_stream);
    if (cudaEventRecord(c->ev_caller, caller) != cudaSuccess ||
        cudaStreamWaitEvent(c->kasync, c->ev_caller, 0) != cudaSuccess ||
        cudaStreamWaitEvent(c->copy3, c->ev_caller, 0) != cudaSuccess) {
        (void)cudaGetLastError();
        set_error("drain: stream ordering failed");
        return fail(PLEX_E_CUDA);
    }
    auto enqueue = [c, a]() -> plex_status {
        plex_status s2;
        if ((s2 = off_begin(c, a->pp, a->h))) return s2;
        for (int32_t b = 0; b < a->h.nb; ++b)
            if ((s2 = off_bucket(c, a->pp, a->h, b))) return s2;
        if ((s2 = off_end(c, a->pp, a->h))) return s2;
        if (cudaEventRecord(a->done_k, c->kasync) != cudaSuccess || cudaEventRecord(a->done_c, c->copy3) != cudaSuccess) {
            (void)cudaGetLastError();
            set_error("drain: event record failed");
            return PLEX_E_CUDA;
        }
        return PLEX_OK;
    };
    if (plan->p.ranks[c->rank].elide_start) {
        // NEXT-2 elision plan: the derivability check is read back on the host
        // (off_begin) -- on a worker thread, so this call returns at once
        a->enqueued = false;
        const int dev = c->device;
        try {
            a->worker = std::thread([a, enqueue, dev]() {
                cudaSetDevice(dev);
                a->enq_status = enqueue();
                if (a->enq_status) a->enq_error = plex_last_error();
                a->enqueued = true;
            });
        } catch (...) {
            set_error("drain: cannot start the enqueue thread");
            return fail(PLEX_E_INVAL);
        }
    } else if ((st = enqueue())) {
        return fail(st);
    }
    slab->busy = true;
    c->async[0] = a;
    return PLEX_OK;
}

plex_status plex_state_prefetch(plex_ctx_t c, plex_plan_t plan, plex_slab_t slab, void* const* dst, int32_t n_dst,
                                void* caller_stream) {
    plex_status st = check_common(c, plan);
    if (st || (st = check_slab(c, plan, slab))) return st;
    if (c->async[1]) { set_error("a prefetch is already in flight"); return PLEX_E_STATE; }
    if (!plan->p.carry.empty()) { set_error("async prefetch does not support carried buckets"); return PLEX_E_INVAL; }
    if (slab->residency == PLEX_RES_DEVICE) {
        if (!slab->written) { set_error("slab holds no offloaded state"); return PLEX_E_STATE; }
        return PLEX_OK;
    }
    if (slab->residency == PLEX_RES_DISK) { set_error("slab is on the NVMe tier: plex_slab_fill first"); return PLEX_E_STATE; }
    if ((uint64_t)c->n_slots * plan->p.bucket > c->staging_bytes / 2) {
        set_error("async transfers need staging >= 2 x n_slots x bucket");
        return PLEX_E_INVAL;
    }
    DeviceGuard g(c->device);
    NvtxRange nv("plex_state_prefetch");
    if ((st = async_resources(c)) ||
        (st = fill_state_ptrs(c, plan->p, reinterpret_cast<const void* const*>(dst), n_dst, 1)))
        return st;
    auto* a = new AsyncState();
    a->h = Half{&plan->p, &plan->p.ranks[c->rank], nullptr, slab, 0, {}, false, 0, nullptr, nullptr, nullptr};
    a->pp = Pipe{c->staging + ((c->staging_bytes / 2) & ~255ull), c->n_slots, c->ev_pack2.data(), c->ev_copy2.data(),
                 c->kasync, c->copy2, c->h_ptrs2, c->d_ptrs2, c->d_ctr + 1, c->d_flag + 1, c->h_flag + 1, true};
    a->slab = slab;
    auto fail = [&](plex_status e) { async_free(a); return e; };
    if ((st = get_devplan(c, plan->p, &a->h.d))) return fail(st);
    if (cudaEventCreateWithFlags(&a->done_k, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&a->done_c, cudaEventDisableTiming) != cudaSuccess) {
        (void)cudaGetLastError();
        set_error("cudaEventCreate failed");
        return fail(PLEX_E_CUDA);
    }
    cudaStream_t caller = reinterpret_cast<cudaStream_t>(caller_stream);
    if (cudaEventRecord(c->ev_caller, caller) != cudaSuccess ||
        cudaStreamWaitEvent(c->kasync, c->ev_caller, 0) != cudaSuccess ||
        cudaStreamWaitEvent(c->copy2, c->ev_caller, 0) != cudaSuccess) {
        (void)cudaGetLastError();
        set_error("prefetch: stream ordering failed");
        return fail(PLEX_E_CUDA);
    }
    if ((st = on_begin(c, a->pp, a->h))) return fail(st);
    for (int32_t b = 0; b < a->h.nb; ++b)
        if ((st = on_bucket(c, a->pp, a->h, b))) return fail(st);
    if ((st = on_end(c, a->pp, a->h))) return fail(st);
    if (cudaEventRecord(a->done_k, c->kasync) != cudaSuccess || cudaEventRecord(a->done_c, c->copy2) != cudaSuccess) {
        (void)cudaGetLastError();
        set_error("prefetch: event record failed");
        return fail(PLEX_E_CUDA);
    }
    slab->busy = true;
    c->async[1] = a;
    return PLEX_OK;
}

plex_status plex_state_poll(plex_ctx_t c, int32_t op, int32_t* done) {
    if (!c || !done || (op != PLEX_OP_OFFLOAD && op != PLEX_OP_ONLOAD)) { set_error("bad poll"); return PLEX_E_INVAL; }
    AsyncState* a = c->async[op == PLEX_OP_OFFLOAD ? 0 : 1];
    if (!a) { *done = 1; return PLEX_OK; }
    if (!a->enqueued.load()) { *done = 0; return PLEX_OK; }   // events not recorded yet
    DeviceGuard g(c->device);
    const cudaError_t ek = cudaEventQuery(a->done_k), ec = cudaEventQuery(a->done_c);
    if ((ek != cudaSuccess && ek != cudaErrorNotReady) || (ec != cudaSuccess && ec != cudaErrorNotReady)) {
        (void)cudaGetLastError();
        set_error("async transfer failed: %s", cudaGetErrorString(ek != cudaSuccess ? ek : ec));
        return PLEX_E_CUDA;
    }
    *done = (ek == cudaSuccess && ec == cudaSuccess) ? 1 : 0;
    return PLEX_OK;
}

plex_status plex_state_wait(plex_ctx_t c, int32_t op, void* caller_stream) {
    if (!c || (op != PLEX_OP_OFFLOAD && op != PLEX_OP_ONLOAD)) { set_error("bad wait"); return PLEX_E_INVAL; }
    const int k = op == PLEX_OP_OFFLOAD ? 0 : 1;
    AsyncState* a = c->async[k];
    if (!a) return PLEX_OK;
    DeviceGuard g(c->device);
    cudaStream_t caller = reinterpret_cast<cudaStream_t>(caller_stream);
    c->async[k] = nullptr;
    a->slab->busy = false;
    if (a->worker.joinable()) a->worker.join();
    if (a->enq_status) {
        set_error("%s", a->enq_error.c_str());
        const plex_status es = a->enq_status;
        (void)cudaStreamSynchronize(c->kasync);            // nothing it enqueued is still running
        (void)cudaStreamSynchronize(c->copy3);
        async_free(a);
        return es;
    }
    cudaError_t e = cudaEventSynchronize(a->done_k);
    if (e == cudaSuccess) e = cudaEventSynchronize(a->done_c);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(caller, a->done_k, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(caller, a->done_c, 0);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        set_error("async transfer failed: %s", cudaGetErrorString(e));
        async_free(a);
        return PLEX_E_CUDA;
    }
    plex_status st = PLEX_OK;
    if (k == 0) {
        off_collect(a->h);
        a->slab->cks.swap(a->h.cks);
        a->slab->residency = PLEX_RES_HOST;
        a->slab->written = true;
        a->slab->elided = a->h.elide;
    } else if (*a->pp.h_flag) {
        set_error("prefetch: %d segment checksum(s) differ from offload", *a->pp.h_flag);
        st = PLEX_E_CHECKSUM;                     // residency stays HOST
    } else {
        a->slab->residency = PLEX_RES_DEVICE;
    }
    async_free(a);
    return st;
}

// ---- a8 - a11: weight sync -------------------------------------------------------------
static plex_status push_rank(plex_ctx_s* c, const Plan& p, int32_t rank, const void* const* src, int32_t n_src,
                             void* const* arenas, cudaStream_t s, const PushItem* d_items,
                             const DevPlan* split = nullptr) {
    const size_t nt = p.tensors.size();
    if (!src || (size_t)n_src != nt) { set_error("expected %zu master pointers, got %d", nt, n_src); return PLEX_E_INVAL; }
    const RankPlan& R = p.ranks[rank];
    plex_status st = ensure_ptrs(c, nt + p.world);
    if (st) return st;
    for (size_t t = 0; t < nt; ++t) c->h_ptrs[t] = reinterpret_cast<uint64_t>(src[t]);
    for (int32_t g = 0; g < p.world; ++g) {
        if (!arenas[g] && p.ranks[g].arena_bytes) { set_error("NULL arena for rank %d", g); return PLEX_E_INVAL; }
        c->h_ptrs[nt + g] = reinterpret_cast<uint64_t>(arenas[g]);
    }
    CK(cudaMemcpyAsync(c->d_ptrs, c->h_ptrs, (nt + p.world) * 8, cudaMemcpyHostToDevice, s));
    cudaEvent_t ta = nullptr;
    if (split) {
        // diagnostic: local items (HBM only) then remote items (NVLink), each timed
        if ((st = timed_begin(c, s, &ta))) return st;
        CK(launch_push(true, split->push_local, split->n_push_local, c->d_ptrs, c->d_ptrs + nt, s));
        if ((st = timed_end(c, s, ta, PLEX_STAT_PUSH_LOCAL, 6 * split->push_local_elems))) return st;
        if ((st = timed_begin(c, s, &ta))) return st;
        CK(launch_push(true, split->push_remote, split->n_push_remote, c->d_ptrs, c->d_ptrs + nt, s));
        return timed_end(c, s, ta, PLEX_STAT_PUSH_REMOTE, 2 * split->push_remote_elems);
    }
    if ((st = timed_begin(c, s, &ta))) return st;
    CK(launch_push(true, d_items, R.push.size(), c->d_ptrs, c->d_ptrs + nt, s));
    if ((st = timed_end(c, s, ta, PLEX_STAT_PUSH, R.src_read_bytes + R.src_read_bytes / 2))) return st;
    return PLEX_OK;
}

// PLEX_CTX_SPLIT_PUSH tables: this rank's push items partitioned by destination.
static plex_status split_push(plex_ctx_s* c, const Plan& p, DevPlan* d) {
    if (d->push_split) return PLEX_OK;
    std::vector<PushItem> loc, rem;
    for (const PushItem& it : p.ranks[c->rank].push) {
        const uint64_t n = (uint64_t)it.rows * it.cols;
        if ((int32_t)it.dst_rank == c->rank) { loc.push_back(it); d->push_local_elems += n; }
        else { rem.push_back(it); d->push_remote_elems += n; }
    }
    plex_status st;
    if ((st = upload(c, &d->push_local, loc)) || (st = upload(c, &d->push_remote, rem))) return st;
    d->n_push_local = loc.size();
    d->n_push_remote = rem.size();
    d->push_split = true;
    return PLEX_OK;
}

plex_status plex_weight_sync_rank(plex_ctx_t c, plex_plan_t plan, int32_t rank, const void* const* src_master,
                                  int32_t n_src, void* const* dst_arenas, int32_t n_arenas, void* stream) {
    if (!c || !plan) { set_error("NULL ctx/plan"); return PLEX_E_INVAL; }
    const Plan& p = plan->p;
    if (p.tp == 0) { set_error("plan has no rollout layout"); return PLEX_E_INVAL; }
    if (rank < 0 || rank >= p.world || n_arenas != p.world || !dst_arenas) { set_error("bad rank/arenas"); return PLEX_E_INVAL; }
    DeviceGuard g(c->device);
    // device tables of `rank` (emulation may drive several ranks from one ctx)
    const uint64_t key = p.id ^ (0x9E3779B97F4A7C15ull * (uint64_t)(rank + 1));
    auto it = c->dev.find(key);
    if (it == c->dev.end()) {
        DevPlan d;
        plex_status s = upload(c, &d.push, p.ranks[rank].push);
        if (s) return s;
        it = c->dev.emplace(key, d).first;
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    plex_status st = push_rank(c, p, rank, src_master, n_src, dst_arenas, s, it->second.push);
    if (st) return st;
    CK(cudaStreamSynchronize(s));
    return timed_collect(c);
}

typedef int (*cuPointerGetAttribute_t)(void*, int, unsigned long long);
static constexpr int kAttrBufferId = 7;      // CU_POINTER_ATTRIBUTE_BUFFER_ID
static constexpr int kAttrRangeStart = 11;   // CU_POINTER_ATTRIBUTE_RANGE_START_ADDR

// Every rank publishes (CUDA-IPC handle, process-unique buffer id, offset) of
// its arena of the given role; peers open a handle only when that (role, rank,
// buffer id) is new, so steady-state calls reuse their NVLink mappings.
static plex_status exchange_arenas(plex_ctx_s* c, int role, void* arena, std::vector<void*>& arenas) {
    static cuPointerGetAttribute_t getattr = nullptr;
    if (!getattr) {
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuPointerGetAttribute", reinterpret_cast<void**>(&getattr), cudaEnableDefault, &q));
        if (!getattr) { set_error("cuPointerGetAttribute unavailable"); return PLEX_E_CUDA; }
    }
    unsigned long long base = 0, bid = 0;
    const unsigned long long a = reinterpret_cast<unsigned long long>(arena);
    if (getattr(&base, kAttrRangeStart, a) != 0 || getattr(&bid, kAttrBufferId, a) != 0) {
        set_error("cuPointerGetAttribute failed for the rollout arena");
        return PLEX_E_CUDA;
    }
    struct Pub {
        cudaIpcMemHandle_t h;
        uint64_t offset;
        uint64_t buffer_id;
        uint64_t pad[6];
    };
    static_assert(sizeof(Pub) <= 256, "Pub");
    Pub me{};
    if (c->my_buffer_id[role] != bid) {
        CK(cudaIpcGetMemHandle(&c->my_handle[role], reinterpret_cast<void*>(base)));
        c->my_buffer_id[role] = bid;
    }
    me.h = c->my_handle[role];
    me.offset = a - base;
    me.buffer_id = bid;
    std::memcpy(c->h_scratch, &me, sizeof(me));
    uint8_t* d_send = c->d_scratch;
    uint8_t* d_all = c->d_scratch + 256;
    CK(cudaMemcpyAsync(d_send, c->h_scratch, 256, cudaMemcpyHostToDevice, c->pack));
    NK(ncclAllGather(d_send, d_all, 256, ncclUint8, c->comm, c->pack));
    CK(cudaMemcpyAsync(c->h_scratch + 256, d_all, 256 * (size_t)c->world, cudaMemcpyDeviceToHost, c->pack));
    CK(cudaStreamSynchronize(c->pack));
    arenas.assign(c->world, nullptr);
    for (int g = 0; g < c->world; ++g) {
        if (g == c->rank) { arenas[g] = arena; continue; }
        Pub pub;
        std::memcpy(&pub, c->h_scratch + 256 + 256 * (size_t)g, sizeof(pub));
        const int pk = role * 4096 + g;
        auto it = c->peers.find(pk);
        if (it == c->peers.end() || it->second.first != pub.buffer_id) {
            if (it != c->peers.end() && it->second.second) cudaIpcCloseMemHandle(it->second.second);
            c->peers.erase(pk);
            void* mapped = nullptr;
            CK(cudaIpcOpenMemHandle(&mapped, pub.h, cudaIpcMemLazyEnablePeerAccess));
            c->peers[pk] = {pub.buffer_id, mapped};
        }
        arenas[g] = reinterpret_cast<uint8_t*>(c->peers[pk].second) + pub.offset;
    }
    return PLEX_OK;
}

plex_status plex_weight_sync(plex_ctx_t c, plex_plan_t plan, const void* const* src_master, int32_t n_src,
                             void* dst_arena, void* caller_stream) {
    plex_status st = check_common(c, plan);
    if (st) return st;
    const Plan& p = plan->p;
    if (p.tp == 0) { set_error("plan has no rollout layout"); return PLEX_E_INVAL; }
    if (!dst_arena && p.ranks[c->rank].arena_bytes) { set_error("NULL arena"); return PLEX_E_INVAL; }
    if (c->world > 1 && !c->comm) { set_error("world > 1 needs a ctx created with an NCCL id"); return PLEX_E_INVAL; }
    DeviceGuard g(c->device);
    NvtxRange nv("plex_weight_sync");
    cudaStream_t caller = reinterpret_cast<cudaStream_t>(caller_stream);
    if (c->flags & PLEX_CTX_SYNC_NCCL) return nccl_sync(c, p, src_master, dst_arena, caller);
    DevPlan* d;
    if ((st = get_devplan(c, p, &d))) return st;
    std::vector<void*> arenas(1, dst_arena);
    if (c->world > 1 && (st = exchange_arenas(c, 0, dst_arena, arenas))) return st;
    CK(cudaEventRecord(c->ev_caller, caller));
    CK(cudaStreamWaitEvent(c->pack, c->ev_caller, 0));
    int* d_bar = reinterpret_cast<int*>(c->d_scratch + 256 + 256 * (size_t)c->world);
    if (c->world > 1) {                                   // all arenas free (waits for the slowest rank)
        cudaEvent_t tb = nullptr;
        if ((st = timed_begin(c, c->pack, &tb))) return st;
        NK(ncclAllReduce(d_bar, d_bar, 1, ncclInt32, ncclSum, c->comm, c->pack));
        if ((st = timed_end(c, c->pack, tb, PLEX_STAT_BARRIER, 0))) return st;
    }
    const bool split = (c->flags & PLEX_CTX_SPLIT_PUSH) && c->world > 1;
    if (split && (st = split_push(c, p, d))) return st;
    if ((st = push_rank(c, p, c->rank, src_master, n_src, arenas.data(), c->pack, d->push, split ? d : nullptr)))
        return st;
    if (c->world > 1) NK(ncclAllReduce(d_bar, d_bar, 1, ncclInt32, ncclSum, c->comm, c->pack));   // all pushes landed
    return finish(c, caller);
}

// ---- NEXT-2: replicated-param restore -------------------------------------------------
static plex_status gather_rank(plex_ctx_s* c, const Plan& p, int32_t rank, void* const* arenas, cudaStream_t s,
                               const PushItem* d_items) {
    const RankPlan& R = p.ranks[rank];
    plex_status st = ensure_ptrs(c, 1 + p.world);
    if (st) return st;
    for (int32_t g = 0; g < p.world; ++g) {
        if (!arenas[g]) { set_error("NULL param arena for rank %d", g); return PLEX_E_INVAL; }
        c->h_ptrs[1 + g] = reinterpret_cast<uint64_t>(arenas[g]);
    }
    c->h_ptrs[0] = c->h_ptrs[1 + rank];
    CK(cudaMemcpyAsync(c->d_ptrs, c->h_ptrs, (1 + p.world) * 8, cudaMemcpyHostToDevice, s));
    cudaEvent_t ta = nullptr;
    if ((st = timed_begin(c, s, &ta))) return st;
    CK(launch_push(false, d_items, R.gather.size(), c->d_ptrs, c->d_ptrs + 1, s));
    return timed_end(c, s, ta, PLEX_STAT_GATHER, 2 * R.gather_send);
}

static plex_status check_replica(plex_ctx_s* c, plex_plan_t plan) {
    if (!c || !plan) { set_error("NULL ctx/plan"); return PLEX_E_INVAL; }
    if (!(plan->p.flags & PLEX_PLAN_REPLICA_PARAM)) { set_error("plan has no replicated params"); return PLEX_E_INVAL; }
    if (plan->p.world != c->world) { set_error("plan world %d != ctx world %d", plan->p.world, c->world); return PLEX_E_INVAL; }
    return PLEX_OK;
}

plex_status plex_param_allgather_rank(plex_ctx_t c, plex_plan_t plan, int32_t rank, void* const* arenas,
                                      int32_t n_arenas, void* stream) {
    plex_status st = check_replica(c, plan);
    if (st) return st;
    const Plan& p = plan->p;
    if (rank < 0 || rank >= p.world || n_arenas != p.world || !arenas) { set_error("bad rank/arenas"); return PLEX_E_INVAL; }
    DeviceGuard g(c->device);
    const uint64_t key = p.id ^ (0xC2B2AE3D27D4EB4Full * (uint64_t)(rank + 1));
    auto it = c->dev.find(key);
    if (it == c->dev.end()) {
        DevPlan d;
        if ((st = upload(c, &d.gather, p.ranks[rank].gather))) return st;
        it = c->dev.emplace(key, d).first;
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if ((st = gather_rank(c, p, rank, arenas, s, it->second.gather))) return st;
    CK(cudaStreamSynchronize(s));
    return timed_collect(c);
}

plex_status plex_param_allgather(plex_ctx_t c, plex_plan_t plan, void* param_arena, void* caller_stream) {
    plex_status st = check_replica(c, plan);
    if (st) return st;
    const Plan& p = plan->p;
    if (!param_arena) { set_error("NULL param arena"); return PLEX_E_INVAL; }
    if (c->world > 1 && !c->comm) { set_error("world > 1 needs a ctx created with an NCCL id"); return PLEX_E_INVAL; }
    DeviceGuard g(c->device);
    NvtxRange nv("plex_param_allgather");
    cudaStream_t caller = reinterpret_cast<cudaStream_t>(caller_stream);
    if (c->world == 1) return PLEX_OK;
    DevPlan* d;
    if ((st = get_devplan(c, p, &d))) return st;
    std::vector<void*> arenas(1, param_arena);
    if ((st = exchange_arenas(c, 1, param_arena, arenas))) return st;
    CK(cudaEventRecord(c->ev_caller, caller));
    CK(cudaStreamWaitEvent(c->pack, c->ev_caller, 0));
    int* d_bar = reinterpret_cast<int*>(c->d_scratch + 256 + 256 * (size_t)c->world);
    // every rank's own rows are in place (each rank orders this after its onload)
    NK(ncclAllReduce(d_bar, d_bar, 1, ncclInt32, ncclSum, c->comm, c->pack));
    if ((st = gather_rank(c, p, c->rank, arenas.data(), c->pack, d->gather))) return st;
    NK(ncclAllReduce(d_bar, d_bar, 1, ncclInt32, ncclSum, c->comm, c->pack));   // every store landed
    return finish(c, caller);
}

// ---- NEXT-3: sync from the offloaded canonical state ------------------------------------
// the StateManager "can materialize rollout-visible shards
// directly from managed memory".  Each rank's fp32 master rows are read by the
// push kernel straight out of its pinned slab (zero-copy over the host link)
// while the job stays suspended; destinations and bytes are those of
// plex_weight_sync.
static plex_status slab_master_ptrs(const Plan& p, plex_slab_t slab, std::vector<const void*>& src) {
    if (!slab || slab->plan_id != p.id) { set_error("slab does not belong to this plan"); return PLEX_E_INVAL; }
    // carried buckets live in the carrier's carry region, not in this slab: any
    // master rows there would be read as stale bytes
    if (p.ranks[slab->rank].carried_out) {
        set_error("sync from slab: %d of this rank's buckets are carried by other ranks (plan with link_weights)",
                  p.ranks[slab->rank].carried_out);
        return PLEX_E_INVAL;
    }
    if (slab->residency != PLEX_RES_HOST || !slab->written || slab->busy) {
        set_error("sync from slab needs HOST-resident offloaded state (and no transfer in flight)");
        return PLEX_E_STATE;
    }
    void* dev = nullptr;
    CK(cudaHostGetDevicePointer(&dev, slab->host, 0));
    const RankPlan& R = p.ranks[slab->rank];
    src.assign(p.tensors.size(), nullptr);
    std::vector<char> seen(p.tensors.size(), 0);
    for (const plex_seg_desc& d : R.seg_desc)
        if (d.kind == PLEX_KIND_MASTER) {
            src[d.tensor] = d.nbytes ? reinterpret_cast<uint8_t*>(dev) + d.slab_offset : nullptr;
            seen[d.tensor] = 1;
        }
    for (size_t t = 0; t < seen.size(); ++t)
        if (!seen[t]) { set_error("slab carries no master rows of tensor %zu", t); return PLEX_E_INVAL; }
    return PLEX_OK;
}

plex_status plex_weight_sync_from_slab(plex_ctx_t c, plex_plan_t plan, plex_slab_t slab, void* dst_arena,
                                       void* caller_stream) {
    if (!c || !plan) { set_error("NULL ctx/plan"); return PLEX_E_INVAL; }
    if (slab && slab->rank != c->rank) { set_error("slab belongs to rank %d, ctx is rank %d", slab->rank, c->rank); return PLEX_E_INVAL; }
    DeviceGuard g(c->device);
    std::vector<const void*> src;
    plex_status st = slab_master_ptrs(plan->p, slab, src);
    if (st) return st;
    return plex_weight_sync(c, plan, src.data(), (int32_t)src.size(), dst_arena, caller_stream);
}

plex_status plex_weight_sync_rank_from_slab(plex_ctx_t c, plex_plan_t plan, int32_t rank, plex_slab_t slab,
                                            void* const* dst_arenas, int32_t n_arenas, void* stream) {
    if (!c || !plan || !slab || slab->rank != rank) { set_error("bad ctx/plan/slab"); return PLEX_E_INVAL; }
    DeviceGuard g(c->device);
    std::vector<const void*> src;
    plex_status st = slab_master_ptrs(plan->p, slab, src);
    if (st) return st;
    return plex_weight_sync_rank(c, plan, rank, src.data(), (int32_t)src.size(), dst_arenas, n_arenas, stream);
}

// ---- infrastructure --------------------------------------------------------------------
static uint64_t fnv1a64(const char* s) {
    uint64_t h = 0xCBF29CE484222325ull;
    for (; *s; ++s) {
        h ^= (uint8_t)*s;
        h *= 0x100000001B3ull;
    }
    return h;
}
static uint64_t stream_base(uint64_t seed, const char* key, int kind) {
    return (seed * 0xD1B54A32D192ED03ull) ^ fnv1a64(key) ^ ((uint64_t)kind << 56);
}

plex_status plex_synth_fill(void* dst, int32_t kind, uint64_t seed, const char* key, uint64_t index_base, uint64_t count,
                            int32_t special_bits, void* stream) {
    if ((!dst && count) || !key || kind < 0 || kind >= PLEX_NUM_KINDS || special_bits < 0 || special_bits > 63) {
        set_error("bad synth arguments");
        return PLEX_E_INVAL;
    }
    CK(launch_synth(dst, kind, stream_base(seed, key, kind), index_base, count, kind ? special_bits : 0,
                    reinterpret_cast<cudaStream_t>(stream)));
    return PLEX_OK;
}

plex_status plex_synth_mutate(void* buf, int32_t kind, uint64_t job_seed, uint64_t step, const char* key,
                              uint64_t index_base, uint64_t count, void* stream) {
    if ((!buf && count) || !key || kind < 0 || kind >= PLEX_NUM_KINDS) { set_error("bad mutate arguments"); return PLEX_E_INVAL; }
    const uint64_t base = stream_base(job_seed, key, kind) ^ ((step + 1) * 0xA24BAED4963EE407ull);
    CK(launch_mutate(buf, kind_esize(kind), base, index_base, count, reinterpret_cast<cudaStream_t>(stream)));
    return PLEX_OK;
}

// ---- diagnostics (kernel measurement, not the method) ----------------------------------
plex_status plex_diag_pack(plex_ctx_t c, plex_plan_t plan, const void* const* state, int32_t n_state, int32_t bucket,
                           int32_t mode, uint64_t staging_offset, void* stream) {
    const bool pack = (mode & 1) != 0, upload = (mode & 2) == 0;
    plex_status st = check_common(c, plan);
    if (st || (st = check_no_async(c))) return st;              // shares the staging ring and counters
    const Plan& p = plan->p;
    const RankPlan& R = p.ranks[c->rank];
    if (bucket < 0 || bucket >= n_buckets(p, R)) { set_error("bucket %d out of range", bucket); return PLEX_E_INVAL; }
    if ((staging_offset & 255) || staging_offset + p.bucket > c->staging_bytes) {
        set_error("staging offset %llu: not 256-B aligned or past the staging buffer", (unsigned long long)staging_offset);
        return PLEX_E_INVAL;
    }
    DeviceGuard g(c->device);
    DevPlan* d;
    if ((st = fill_state_ptrs(c, p, state, n_state)) || (st = get_devplan(c, p, &d))) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (upload)
        CK(cudaMemcpyAsync(c->d_ptrs, c->h_ptrs, sizeof(uint64_t) * PLEX_NUM_KINDS * p.tensors.size(),
                           cudaMemcpyHostToDevice, s));
    const uint64_t i0 = R.bucket_item_start[bucket], i1 = R.bucket_item_start[bucket + 1];
    CK(launch_pack(pack, d->items + i0, (uint32_t)(i1 - i0), d->segs, c->d_ptrs, c->staging + staging_offset,
                   (uint64_t)bucket * p.bucket, pack ? d->cks : d->cks_in, c->d_ctr, s));
    return PLEX_OK;
}

plex_status plex_diag_pack_variant(int32_t variant) {
    if (variant < 0 || variant > 1) { set_error("pack variant %d unknown", variant); return PLEX_E_INVAL; }
    set_pack_variant(variant);
    return PLEX_OK;
}

plex_status plex_checksum(const void* src, int32_t esize, uint64_t index_base, uint64_t count, uint64_t* dev_out,
                          void* stream) {
    if ((!src && count) || !dev_out || (esize != 2 && esize != 4)) { set_error("bad checksum arguments"); return PLEX_E_INVAL; }
    CK(launch_checksum(src, esize, index_base, count, reinterpret_cast<unsigned long long*>(dev_out),
                       reinterpret_cast<cudaStream_t>(stream)));
    return PLEX_OK;
}

plex_status plex_cast_rne(const void* src_f32, void* dst_bf16, uint64_t count, void* stream) {
    if ((!src_f32 || !dst_bf16) && count) { set_error("bad cast arguments"); return PLEX_E_INVAL; }
    CK(launch_cast(src_f32, dst_bf16, count, reinterpret_cast<cudaStream_t>(stream)));
    return PLEX_OK;
}

}  // extern "C"

namespace plex {

// ---- NCCL baseline transport of the weight sync (PLEX_CTX_SYNC_NCCL) --------
// K4 casts every (source = me, destination d) rectangle into d's contiguous
// send segment, one grouped ncclSend/ncclRecv per round exchanges all
// segments (N1), K5 copies received rectangles into the arena.  Rounds bound
// staging: the ctx staging is split into send/recv x double buffer, each with
// (world-1) per-pair regions of Q bytes.  K4(k+1) and the exchange of round k
// overlap; K5(k) follows the exchange.  Same bytes as the fused push (the
// ledger), so the two transports are measured against each other.
static uint64_t pad16(uint64_t b) { return (b + 15) & ~15ull; }

static plex_status build_nccl_sched(plex_ctx_s* c, const Plan& p, DevPlan* d, uint64_t Q) {
    const int W = p.world, me = c->rank;
    auto slot = [&](int x) { return x < me ? x : x - 1; };
    std::vector<PushItem> local, rp, ru;
    std::vector<std::vector<PushItem>> rp_r, ru_r;
    std::vector<uint64_t> rpb, rub, sb, rb;
    int R = 0;
    // pass 1: rounds of every pair (needs every rank's list, identical on all ranks)
    std::vector<int> rounds_pair((size_t)W * W, 0);
    for (int src = 0; src < W; ++src) {
        std::vector<uint64_t> cum(W, 0);
        std::vector<int> rnd(W, 0), any(W, 0);
        for (const PushItem& it : p.ranks[src].push) {
            const int dst = (int)it.dst_rank;
            if (dst == src) continue;
            const uint64_t b = pad16((uint64_t)it.rows * it.cols * 2);
            if (cum[dst] + b > Q && cum[dst] > 0) { ++rnd[dst]; cum[dst] = 0; }
            cum[dst] += b;
            any[dst] = 1;
        }
        for (int dst = 0; dst < W; ++dst)
            if (any[dst]) { rounds_pair[(size_t)src * W + dst] = rnd[dst] + 1; R = std::max(R, rnd[dst] + 1); }
    }
    rp_r.assign(R, {});
    ru_r.assign(R, {});
    rpb.assign(R, 0);
    rub.assign(R, 0);
    sb.assign((size_t)R * W, 0);
    rb.assign((size_t)R * W, 0);
    uint64_t local_bytes = 0;
    // pass 2: my send items (K4) and my local items
    {
        std::vector<uint64_t> cum(W, 0);
        std::vector<int> rnd(W, 0);
        for (const PushItem& it : p.ranks[me].push) {
            const int dst = (int)it.dst_rank;
            const uint64_t n = (uint64_t)it.rows * it.cols;
            if (dst == me) { local.push_back(it); local_bytes += 6 * n; continue; }
            const uint64_t b = pad16(n * 2);
            if (cum[dst] + b > Q && cum[dst] > 0) { ++rnd[dst]; cum[dst] = 0; }
            PushItem q = it;
            q.dst_elem = ((uint64_t)slot(dst) * Q + cum[dst]) / 2;
            q.dst_rank = (uint32_t)(W + (rnd[dst] & 1));
            q.dst_stride = it.cols;
            rp_r[rnd[dst]].push_back(q);
            rpb[rnd[dst]] += 6 * n;
            cum[dst] += b;
            sb[(size_t)rnd[dst] * W + dst] = cum[dst];
        }
    }
    // pass 3: what every peer sends me (K5), in the sender's order
    for (int src = 0; src < W; ++src) {
        if (src == me) continue;
        uint64_t cum = 0;
        int rnd = 0;
        for (const PushItem& it : p.ranks[src].push) {
            if ((int)it.dst_rank != me) continue;
            const uint64_t n = (uint64_t)it.rows * it.cols;
            const uint64_t b = pad16(n * 2);
            if (cum + b > Q && cum > 0) { ++rnd; cum = 0; }
            PushItem q = it;
            q.src_elem = ((uint64_t)slot(src) * Q + cum) / 2;
            q.src_stride = it.cols;
            q.tensor = (uint32_t)(rnd & 1);
            q.dst_rank = (uint32_t)me;
            ru_r[rnd].push_back(q);
            rub[rnd] += 4 * n;
            cum += b;
            rb[(size_t)rnd * W + src] = cum;
        }
    }
    std::vector<uint64_t> rps(R + 1, 0), rus(R + 1, 0);
    for (int k = 0; k < R; ++k) {
        rps[k + 1] = rps[k] + rp_r[k].size();
        rus[k + 1] = rus[k] + ru_r[k].size();
        rp.insert(rp.end(), rp_r[k].begin(), rp_r[k].end());
        ru.insert(ru.end(), ru_r[k].begin(), ru_r[k].end());
    }
    if (d->local || d->rpack || d->runpack) quiesce(c);
    dev_free(c, d->local);
    dev_free(c, d->rpack);
    dev_free(c, d->runpack);
    d->local = d->rpack = d->runpack = nullptr;
    plex_status st;
    if ((st = upload(c, &d->local, local)) || (st = upload(c, &d->rpack, rp)) || (st = upload(c, &d->runpack, ru)))
        return st;
    d->n_local = local.size();
    d->local_bytes = local_bytes;
    d->rounds = R;
    d->rpack_start = rps;
    d->runpack_start = rus;
    d->rpack_bytes = rpb;
    d->runpack_bytes = rub;
    d->send_bytes = sb;
    d->recv_bytes = rb;
    d->nq = Q;
    return PLEX_OK;
}

plex_status nccl_sync(plex_ctx_s* c, const Plan& p, const void* const* src, void* arena, cudaStream_t caller) {
    const int W = p.world, me = c->rank;
    const size_t nt = p.tensors.size();
    if (!src) { set_error("NULL master pointers"); return PLEX_E_INVAL; }
    plex_status st;
    DevPlan* d;
    if ((st = get_devplan(c, p, &d))) return st;
    const uint64_t Q = W > 1 ? (c->staging_bytes / (4ull * (W - 1))) & ~255ull : 0;
    if (W > 1 && Q < 4096) { set_error("staging too small for the NCCL sync transport"); return PLEX_E_INVAL; }
    if (d->nq != Q && (st = build_nccl_sched(c, p, d, std::max<uint64_t>(Q, 256)))) return st;
    uint8_t* send[2] = {c->staging, c->staging + (uint64_t)(W - 1) * Q};
    uint8_t* recv[2] = {c->staging + 2ull * (W - 1) * Q, c->staging + 3ull * (W - 1) * Q};
    // pointer table: [nt masters][W + 2 destinations][2 receive buffers]
    if ((st = ensure_ptrs(c, nt + W + 4))) return st;
    for (size_t t = 0; t < nt; ++t) c->h_ptrs[t] = reinterpret_cast<uint64_t>(src[t]);
    uint64_t* hd = c->h_ptrs + nt;
    for (int g = 0; g < W; ++g) hd[g] = 0;
    hd[me] = reinterpret_cast<uint64_t>(arena);
    hd[W] = reinterpret_cast<uint64_t>(send[0]);
    hd[W + 1] = reinterpret_cast<uint64_t>(send[1]);
    hd[W + 2] = reinterpret_cast<uint64_t>(recv[0]);
    hd[W + 3] = reinterpret_cast<uint64_t>(recv[1]);
    const uint64_t* d_src = c->d_ptrs;
    const uint64_t* d_dst = c->d_ptrs + nt;
    const uint64_t* d_rcv = c->d_ptrs + nt + W + 2;
    CK(cudaEventRecord(c->ev_caller, caller));
    CK(cudaStreamWaitEvent(c->pack, c->ev_caller, 0));
    CK(cudaStreamWaitEvent(c->copy, c->ev_caller, 0));
    CK(cudaMemcpyAsync(c->d_ptrs, c->h_ptrs, (nt + W + 4) * 8, cudaMemcpyHostToDevice, c->pack));
    CK(cudaEventRecord(c->ev_sync[0], c->pack));
    CK(cudaStreamWaitEvent(c->copy, c->ev_sync[0], 0));      // pointer table visible before any K5
    cudaEvent_t ta = nullptr;
    if ((st = timed_begin(c, c->pack, &ta))) return st;
    CK(launch_push(true, d->local, d->n_local, d_src, d_dst, c->pack));
    if ((st = timed_end(c, c->pack, ta, PLEX_STAT_PUSH, d->local_bytes))) return st;
    cudaEvent_t* evR = c->ev_sync;       // K4 done, per buffer
    cudaEvent_t* evN = c->ev_sync + 2;   // exchange done
    cudaEvent_t* evU = c->ev_sync + 4;   // K5 done
    const int R = d->rounds;
    auto rpack = [&](int k) -> plex_status {
        const uint64_t i0 = d->rpack_start[k], i1 = d->rpack_start[k + 1];
        cudaEvent_t t = nullptr;
        plex_status s2;
        if ((s2 = timed_begin(c, c->pack, &t))) return s2;
        CK(launch_push(true, d->rpack + i0, i1 - i0, d_src, d_dst, c->pack));
        if ((s2 = timed_end(c, c->pack, t, PLEX_STAT_RPACK, d->rpack_bytes[k]))) return s2;
        CK(cudaEventRecord(evR[k & 1], c->pack));
        return PLEX_OK;
    };
    if (R > 0 && (st = rpack(0))) return st;
    for (int k = 0; k < R; ++k) {
        const int b = k & 1;
        CK(cudaStreamWaitEvent(c->copy, evR[b], 0));
        if (k >= 2) CK(cudaStreamWaitEvent(c->copy, evU[b], 0));
        if ((st = timed_begin(c, c->copy, &ta))) return st;
        uint64_t ssum = 0, rsum = 0;
        NK(ncclGroupStart());
        for (int g = 0; g < W; ++g) {
            if (g == me) continue;
            const int sl = g < me ? g : g - 1;
            const uint64_t sbytes = d->send_bytes[(size_t)k * W + g], rbytes = d->recv_bytes[(size_t)k * W + g];
            if (sbytes) NK(ncclSend(send[b] + (uint64_t)sl * Q, sbytes, ncclUint8, g, c->comm, c->copy));
            if (rbytes) NK(ncclRecv(recv[b] + (uint64_t)sl * Q, rbytes, ncclUint8, g, c->comm, c->copy));
            ssum += sbytes;
            rsum += rbytes;
        }
        NK(ncclGroupEnd());
        if ((st = timed_end(c, c->copy, ta, PLEX_STAT_NCCL, std::max(ssum, rsum)))) return st;
        CK(cudaEventRecord(evN[b], c->copy));
        if (k + 1 < R && (st = rpack(k + 1))) return st;
        CK(cudaStreamWaitEvent(c->pack, evN[b], 0));
        const uint64_t i0 = d->runpack_start[k], i1 = d->runpack_start[k + 1];
        if ((st = timed_begin(c, c->pack, &ta))) return st;
        CK(launch_push(false, d->runpack + i0, i1 - i0, d_rcv, d_dst, c->pack));
        if ((st = timed_end(c, c->pack, ta, PLEX_STAT_RUNPACK, d->runpack_bytes[k]))) return st;
        CK(cudaEventRecord(evU[b], c->pack));
    }
    return finish(c, caller);
}

}  // namespace plex
