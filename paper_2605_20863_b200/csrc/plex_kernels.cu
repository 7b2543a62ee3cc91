// sm_100a kernels of the state-transition hot path.
//
// K1 gather-pack (+R14 checksum)   a3   PAPER.md:462 (migrating model states HBM->host)
// K2 scatter-unpack (+verify)      a7   PAPER.md:572 (resident and safe to use)
// K3+K4 fused RNE cast + reshard push over NVLink   a8-a11
// K6 synthetic init / mutation, K7 checksum, plain cast: infrastructure.
//
// Everything here is HBM- (or NVLink-) bound data movement with a few integer
// ops per element: no tensor cores (nothing is a contraction).
//  * K1/K2: persistent TMA bulk-copy pipeline (cp.async.bulk global<->shared,
//    mbarrier complete_tx), 2 CTAs/SM, dynamic work claiming spread across the
//    bucket; the checksum is folded from shared memory.
//  * push / cast / derive: one 256-thread CTA per planner work item, 16-B
//    vectorised streaming loads (ld.global.nc.L1::no_allocate) and stores;
//    the push kernel's stores go to peer-mapped arenas over NVLink; strided
//    (row-parallel) rectangles use a 2-D warp-per-row mapping.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "plex_internal.h"

namespace plex {

constexpr int kThreads = 256;

__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void st_v4(void* p, const uint4& v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// ---- R14 checksum of one 16-B vector whose first element has logical index i0.
struct Cks {
    unsigned long long s1 = 0, s2 = 0;
    __device__ __forceinline__ void add_sum(uint64_t s, uint64_t t, uint64_t i0) {
        s1 += s;
        s2 += (i0 + 1) * s + t;
    }
    __device__ __forceinline__ void add_vec(const uint4& v, int esize, uint64_t i0) {
        if (esize == 4) {
            const uint64_t s = (uint64_t)v.x + v.y + v.z + v.w;
            const uint64_t t = (uint64_t)v.y + 2ull * v.z + 3ull * v.w;
            add_sum(s, t, i0);
        } else {
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
            uint32_t s = 0, t = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t lo = w[k] & 0xFFFFu, hi = w[k] >> 16;
                s += lo + hi;
                t += (2 * k) * lo + (2 * k + 1) * hi;
            }
            add_sum(s, t, i0);
        }
    }
    __device__ __forceinline__ void add_elem(uint32_t b, uint64_t i) {
        s1 += b;
        s2 += (i + 1) * (uint64_t)b;
    }
};

__device__ __forceinline__ void block_reduce_add(Cks c, unsigned long long* out) {
    __shared__ unsigned long long sh[2][kThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        c.s1 += __shfl_xor_sync(0xffffffffu, c.s1, o);
        c.s2 += __shfl_xor_sync(0xffffffffu, c.s2, o);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { sh[0][w] = c.s1; sh[1][w] = c.s2; }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long a = 0, b = 0;
#pragma unroll
        for (int k = 0; k < kThreads / 32; ++k) { a += sh[0][k]; b += sh[1][k]; }
        atomicAdd(out, a);
        atomicAdd(out + 1, b);
    }
}

// ---- K1 / K2: pack (tensor -> staging) or unpack (staging -> tensor) -------
// Persistent, PackCfg = TmaCfg<3, 32, 4, 2>: two CTAs per SM, each a TMA
// bulk-copy pipeline (cp.async.bulk, SASS UBLKCP) with a 3-stage ring of
// 32 KiB chunks.  The producer warp (warp 4, lane 0) claims PackItems from a
// per-launch counter (dynamic balancing, see below) and streams their chunks
// global->shared (mbarrier complete_tx); consumer warps 0-3 fold the R14
// checksum from shared memory while consumer thread 0 streams the same stage
// back out shared->global (bulk_group).  A stage is released once every
// consumer warp and the bulk store have read it.  Byte ranges that TMA cannot
// move (a tensor not 16-B aligned, or the <16-B tail of a segment) go through
// the consumer threads directly; padding bytes of a slot are written as zeros
// on pack and skipped on unpack.  Work: the bucket's PackItems (slot byte
// ranges <= 64 KiB).

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sdst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
}
// L2 eviction-priority variants (diagnostic variant 1 of the pack kernel):
// the same bulk copies carrying an L2::evict_first cache policy.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_load_hint(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void bulk_store_hint(void* gdst, const void* ssrc, uint32_t bytes, uint64_t pol) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ uint4 lds128(const void* p) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(smem_u32(p)));
    return r;
}

// Geometry of one item, identical for producer and consumers.
struct ItemGeo {
    uint8_t* tens;      // tensor bytes at the item's first slot byte
    uint8_t* buf;       // staging bytes at the item's first slot byte
    uint64_t ib;        // logical index of the item's first element
    uint32_t len;       // slot bytes of the item
    uint32_t data;      // data bytes of the item (rest is padding)
    uint32_t seg;
    int es;
    bool vec;           // tensor side 16-B aligned -> bulk copies allowed
};

__device__ __forceinline__ ItemGeo item_geo(const PackItem& it, const SegDev* segs, const uint64_t* ptrs,
                                            uint8_t* staging, uint64_t bucket_lo) {
    const SegDev s = segs[it.seg];
    ItemGeo g;
    const uint64_t o0 = it.slab_lo - s.slab_off;
    g.tens = reinterpret_cast<uint8_t*>(ptrs[s.ptr_slot]) + o0;
    g.buf = staging + (it.slab_lo - bucket_lo);
    g.es = (int)s.esize;
    g.ib = s.index_base + o0 / s.esize;
    g.len = it.len;
    g.data = o0 >= s.bytes ? 0u : (uint32_t)(s.bytes - o0 < it.len ? s.bytes - o0 : it.len);
    g.seg = it.seg;
    g.vec = (reinterpret_cast<uintptr_t>(g.tens) & 15) == 0;
    return g;
}

// bulk bytes of chunk [co, co + chunk) of an item
__device__ __forceinline__ uint32_t chunk_bulk(const ItemGeo& g, uint32_t co, uint32_t chunk) {
    if (!g.vec || co >= g.data) return 0;
    const uint32_t e = g.data - co < chunk ? g.data - co : chunk;
    return e & ~15u;
}

// One staged chunk: which item/offset it belongs to (written by the producer
// before it arrives on the stage's full barrier, read by the consumers after
// their wait: mbarrier arrive/wait order it).
struct StageMeta {
    ItemGeo g;
    uint32_t co;        // chunk offset within the item
    uint32_t flags;     // kMetaDone: no more work
};
constexpr uint32_t kMetaDone = 2u;

template <int STAGES, int CHUNK_KB, int CWARPS, int CTAS>
struct TmaCfg {
    static constexpr int kStages = STAGES;
    static constexpr uint32_t kChunk = (uint32_t)CHUNK_KB * 1024u;
    static constexpr int kConsumers = CWARPS * 32;
    static constexpr int kThreads = kConsumers + 32;
    static constexpr int kCtasPerSm = CTAS;
    static constexpr size_t kMetaOff = (size_t)STAGES * kChunk;
    static constexpr size_t kBarOff = kMetaOff + STAGES * sizeof(StageMeta);
    static constexpr size_t kSmem = kBarOff + 2 * STAGES * sizeof(uint64_t);
};
using PackCfg = TmaCfg<3, 32, 4, 2>;     // 2 CTAs/SM x 3 stages x 32 KiB (see profiles/ kbench runs)

// Work distribution is dynamic: each CTA's producer claims the next PackItem
// from a per-launch counter (one claim ahead, so the claim + descriptor-fetch
// latency hides behind the chunks already in flight) and tags every staged
// chunk with its item geometry.  CTAs that run faster simply take more items,
// which removes the static round-robin tail.
template <bool kPack, class Cfg, int kHint = 0>
__global__ void __launch_bounds__(Cfg::kThreads, Cfg::kCtasPerSm)
    pack_kernel(const PackItem* __restrict__ items, uint32_t n_items, const SegDev* __restrict__ segs,
                const uint64_t* __restrict__ ptrs, uint8_t* __restrict__ staging, uint64_t bucket_lo,
                unsigned long long* __restrict__ cks, unsigned int* __restrict__ ctr, uint32_t perm) {
    constexpr int kStages = Cfg::kStages;
    constexpr uint32_t kChunk = Cfg::kChunk;
    constexpr int kConsumers = Cfg::kConsumers;
    extern __shared__ __align__(128) uint8_t smem[];
    StageMeta* meta = reinterpret_cast<StageMeta*>(smem + Cfg::kMetaOff);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::kBarOff);
    uint64_t* empty = full + kStages;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            // released by every consumer warp (done reading) + the bulk store (done reading)
            mbar_init(&empty[i], kConsumers / 32 + 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (tid >= kConsumers) {
        // ---------------- producer: claim items, TMA-load their chunks ----------------
        if (tid != kConsumers) return;
        const uint64_t pol = kHint ? policy_evict_first() : 0;
        uint32_t q = 0;
        // claim c -> item (c * perm) mod n (perm = 1: slab order; perm coprime
        // to n spreads concurrently processed items across the bucket)
        auto claim = [&]() -> uint32_t {
            const uint32_t c = atomicAdd(ctr, 1u);
            return c < n_items ? (uint32_t)(((uint64_t)c * perm) % n_items) : n_items;
        };
        uint32_t i = claim();
        ItemGeo g;
        if (i < n_items) g = item_geo(items[i], segs, ptrs, staging, bucket_lo);
        while (i < n_items) {
            const uint32_t inext = claim();                     // claim ahead
            const uint8_t* src = kPack ? g.tens : g.buf;
            for (uint32_t co = 0; co < g.len; co += kChunk, ++q) {
                const int st = (int)(q % kStages);
                if (q >= (uint32_t)kStages) mbar_wait(&empty[st], ((q / kStages) - 1) & 1);
                meta[st].g = g;
                meta[st].co = co;
                meta[st].flags = 0u;
                const uint32_t nb = chunk_bulk(g, co, kChunk);
                if (nb) {
                    mbar_arrive_tx(&full[st], nb);
                    if (kHint) bulk_load_hint(smem + (size_t)st * kChunk, src + co, nb, &full[st], pol);
                    else bulk_load(smem + (size_t)st * kChunk, src + co, nb, &full[st]);
                } else {
                    mbar_arrive(&full[st]);
                }
            }
            i = inext;
            if (i < n_items) g = item_geo(items[i], segs, ptrs, staging, bucket_lo);
        }
        const int st = (int)(q % kStages);
        if (q >= (uint32_t)kStages) mbar_wait(&empty[st], ((q / kStages) - 1) & 1);
        meta[st].flags = kMetaDone;
        mbar_arrive(&full[st]);
        return;
    }
    // ---------------- consumers: checksum + TMA stores ----------------
    // Each warp keeps one running (S1, S2) for the segment of the items it is
    // folding and adds it to the segment's global pair only when the segment
    // changes (R14 is additive over any partition) or at the end: a bucket
    // inside one large tensor (embed / lm_head) would otherwise send every
    // item's atomics to the same two addresses, and those serialise in L2
    // (+40 % kernel time on such buckets, profiles/r02f_pack_insitu.jsonl).
    const uint64_t spol = (kHint && tid == 0) ? policy_evict_first() : 0;
    Cks c;
    uint32_t cseg = 0xFFFFFFFFu;                    // segment c belongs to (warp-uniform)
    auto flush = [&]() {
        if (cseg == 0xFFFFFFFFu) return;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            c.s1 += __shfl_xor_sync(0xffffffffu, c.s1, o);
            c.s2 += __shfl_xor_sync(0xffffffffu, c.s2, o);
        }
        if (lane == 0) {
            atomicAdd(cks + 2 * cseg, c.s1);
            atomicAdd(cks + 2 * cseg + 1, c.s2);
        }
        c = Cks();
    };
    for (uint32_t q = 0;; ++q) {
        const int st = (int)(q % kStages);
        mbar_wait(&full[st], (q / kStages) & 1);
        const uint32_t flags = meta[st].flags;
        if (flags & kMetaDone) break;
        const ItemGeo g = meta[st].g;
        const uint32_t co = meta[st].co;
        if (co < g.data && g.seg != cseg) {          // this chunk carries data of another segment
            flush();
            cseg = g.seg;
        }
        const uint8_t* src = kPack ? g.tens : g.buf;
        uint8_t* dst = kPack ? g.buf : g.tens;
        const uint8_t* sm = smem + (size_t)st * kChunk;
        const uint32_t nb = chunk_bulk(g, co, kChunk);
        const uint32_t cend = g.len - co < kChunk ? g.len : co + kChunk;
        const uint32_t dend = g.data < cend ? g.data : cend;            // data end within chunk
        if (tid == 0 && nb) {
            if (kHint) bulk_store_hint(dst + co, sm, nb, spol);
            else bulk_store(dst + co, sm, nb);                          // write back while we checksum
            bulk_commit();
        }
        // checksum of the bulk part, read back from shared memory
        for (uint32_t v = tid; v < nb / 16; v += kConsumers)
            c.add_vec(lds128(sm + 16 * v), g.es, g.ib + (co + 16 * v) / g.es);
        // non-bulk data (misaligned tensor or <16-B tail): element by element
        const uint32_t t0 = co + nb;
        if (t0 < dend) {
            const uint32_t ne = (dend - t0) / g.es;
            for (uint32_t e = tid; e < ne; e += kConsumers) {
                const uint32_t off = t0 + e * g.es;
                uint32_t b;
                if (g.es == 4) {
                    b = *reinterpret_cast<const uint32_t*>(src + off);
                    *reinterpret_cast<uint32_t*>(dst + off) = b;
                } else {
                    b = *reinterpret_cast<const uint16_t*>(src + off);
                    *reinterpret_cast<uint16_t*>(dst + off) = (uint16_t)b;
                }
                c.add_elem(b, g.ib + off / g.es);
            }
        }
        if (kPack && dend < cend) {
            const uint32_t p0 = co > g.data ? co : g.data;
            for (uint32_t b = p0 + tid; b < cend; b += kConsumers) dst[b] = 0;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);                         // this warp is done with stage st
        if (tid == 0) {
            if (nb) bulk_wait_read_all();                               // the bulk store has read stage st
            mbar_arrive(&empty[st]);
        }
    }
    flush();
    if (tid == 0) {
        bulk_wait_all();                           // every bulk store complete before exit
        // Self-resetting claim counter (no memset node before each launch): this
        // CTA's producer made its last claim before it signalled kMetaDone, so
        // once every CTA has checked in, no claim is outstanding.  ctr[8] counts
        // finished CTAs; the last one zeroes both for the next launch.
        __threadfence();
        if (atomicAdd(ctr + 8, 1u) == gridDim.x - 1) {
            atomicExch(ctr, 0u);
            atomicExch(ctr + 8, 0u);
        }
    }
}

__global__ void verify_kernel(const unsigned long long* __restrict__ got, const unsigned long long* __restrict__ want,
                              uint32_t n, int* __restrict__ bad) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (got[2 * i] != want[2 * i] || got[2 * i + 1] != want[2 * i + 1]) atomicAdd(bad, 1);
}

// ---- a8: fp32 -> bf16 round-to-nearest-even (R8), integer bit math ---------
// r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16; any NaN -> 0x7FC0.  Subnormals are
// rounded like any other value (no flush); overflow rounds to +-inf.
__device__ __forceinline__ uint32_t rne_bf16(uint32_t u) {
    const uint32_t r = (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
    return ((u & 0x7FFFFFFFu) > 0x7F800000u) ? 0x7FC0u : r;
}
__device__ __forceinline__ uint32_t rne_pack2(uint32_t lo, uint32_t hi) {
    return rne_bf16(lo) | (rne_bf16(hi) << 16);
}
__device__ __forceinline__ uint4 rne_8(const uint4& a, const uint4& b) {
    return make_uint4(rne_pack2(a.x, a.y), rne_pack2(a.z, a.w), rne_pack2(b.x, b.y), rne_pack2(b.z, b.w));
}

// ---- K3+K4: fused cast + reshard push ---------------------------------------
// One CTA per PushItem: rows x cols fp32 rectangle of this rank's master shard
// -> RNE -> bf16 rectangle of destination dst_rank's buffer, which is a
// peer-mapped arena (NVLink store), the local arena, or (NCCL baseline, K4) a
// send segment.  kCast = false is K5 of the NCCL baseline: a bf16 -> bf16
// rectangle copy from a receive segment into the arena.
template <bool kCast>
__global__ void __launch_bounds__(kThreads) push_kernel(const PushItem* __restrict__ items, uint64_t n_items,
                                                        const uint64_t* __restrict__ src_ptrs,
                                                        const uint64_t* __restrict__ dst_arenas) {
  // one item per CTA (the launch uses grid = items; the loop form also
  // covers a grid smaller than the item list)
  for (uint64_t ii = blockIdx.x; ii < n_items; ii += gridDim.x) {
    const PushItem it = items[ii];
    constexpr int kSrcEs = kCast ? 4 : 2;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(src_ptrs[it.tensor]) + (uint64_t)it.src_elem * kSrcEs;
    uint16_t* dst = reinterpret_cast<uint16_t*>(dst_arenas[it.dst_rank]) + it.dst_elem;
    const uint32_t rows = it.rows, cols = it.cols, ss = it.src_stride, ds = it.dst_stride;
    const bool vec = ((reinterpret_cast<uintptr_t>(src) & 15) == 0) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) &&
                     (cols % 8 == 0) && ((ss * kSrcEs) % 16 == 0) && (ds % 8 == 0);
    auto load8 = [&](uint64_t e) -> uint4 {      // 8 elements starting at source element e
        if (kCast) {
            const uint4 a = ld_stream(src + 4 * e), b = ld_stream(src + 4 * e + 16);
            return rne_8(a, b);
        } else {
            return ld_stream(src + 2 * e);
        }
    };
    if (vec) {
        const uint32_t vpr = cols / 8;
        if (rows == 1) {
            const uint32_t total = vpr;
            uint32_t v = threadIdx.x;
            for (; v + kThreads < total; v += 2 * kThreads) {
                const uint4 x0 = load8(8ull * v);
                const uint4 x1 = load8(8ull * (v + kThreads));
                st_v4(dst + 8ull * v, x0);
                st_v4(dst + 8ull * (v + kThreads), x1);
            }
            for (; v < total; v += kThreads) st_v4(dst + 8ull * v, load8(8ull * v));
        } else {
            // Strided rectangle (row-parallel o_proj / down_proj slices, fused-group
            // pieces): a 2-D warp mapping, no per-vector index division.  wpr warps
            // share one row (lanes stride its 16-B vectors, coalesced on both
            // sides); rows_in_flight rows are processed at once, the CTA strides
            // over the rest.  The one division is per thread, not per vector.
            constexpr uint32_t kWarps = kThreads / 32;
            const uint32_t wpr = rows >= kWarps ? 1u : kWarps / rows;
            const uint32_t rif = kWarps / wpr;
            const uint32_t w = threadIdx.x >> 5;
            const uint32_t r0 = w / wpr;
            const uint32_t c0 = (w - r0 * wpr) * 32 + (threadIdx.x & 31), cs = wpr * 32;
            if (r0 < rif) {
                for (uint32_t r = r0; r < rows; r += rif) {
                    const uint64_t so = (uint64_t)r * ss, dof = (uint64_t)r * ds;
                    uint32_t c = c0;
                    for (; c + cs < vpr; c += 2 * cs) {                 // two 32-B fp32 loads in flight
                        const uint4 x0 = load8(so + 8 * c);
                        const uint4 x1 = load8(so + 8 * (c + cs));
                        st_v4(dst + dof + 8 * c, x0);
                        st_v4(dst + dof + 8 * (c + cs), x1);
                    }
                    for (; c < vpr; c += cs) st_v4(dst + dof + 8 * c, load8(so + 8 * c));
                }
            }
        }
    } else {
        const uint64_t total = (uint64_t)rows * cols;
        for (uint64_t e = threadIdx.x; e < total; e += kThreads) {
            const uint64_t r = e / cols, c = e - r * cols;
            const uint64_t si = r * ss + c;
            dst[r * ds + c] = kCast ? (uint16_t)rne_bf16(reinterpret_cast<const uint32_t*>(src)[si])
                                    : reinterpret_cast<const uint16_t*>(src)[si];
        }
    }
  }
}

// ---- NEXT-2: derived-param check / re-derivation -------------------------------
// Over PackItems of PARAM segments: kCheck -> count elements whose bf16 param
// differs from RNE(master) (R8) and checksum the params; !kCheck -> write
// param = RNE(master) and checksum what was written.  The master shard of
// tensor t sits at pointer slot ptr_slot + n_tensors (kind 1 vs kind 0).
template <bool kCheck>
__global__ void __launch_bounds__(kThreads) derive_kernel(const PackItem* __restrict__ items, uint32_t n_items,
                                                          const SegDev* __restrict__ segs,
                                                          const uint64_t* __restrict__ ptrs, uint32_t n_tensors,
                                                          unsigned long long* __restrict__ cks, int* __restrict__ bad) {
    // Grid-stride over the items; the block keeps one running (S1, S2) while
    // its items stay in one segment and adds it to the segment's pair when the
    // segment changes (as K1/K2: a bf16 embed / lm_head segment spans ~16 k
    // items, whose per-item atomics would serialise on one L2 address).
    Cks c;
    uint32_t cseg = 0xFFFFFFFFu;
    int miss = 0;
    for (uint32_t i = blockIdx.x; i < n_items; i += gridDim.x) {
        const PackItem it = items[i];
        const SegDev s = segs[it.seg];
        const uint64_t o0 = it.slab_lo - s.slab_off;
        if (o0 >= s.bytes) continue;                                // padding only (block-uniform)
        if (it.seg != cseg) {
            if (cseg != 0xFFFFFFFFu) {
                block_reduce_add(c, cks + 2 * cseg);
                __syncthreads();                                    // shared partials reused by the next flush
            }
            c = Cks();
            cseg = it.seg;
        }
        const uint64_t nbytes = (s.bytes - o0 < it.len ? s.bytes - o0 : it.len);
        const uint64_t n = nbytes / 2;                              // bf16 elements
        uint16_t* param = reinterpret_cast<uint16_t*>(ptrs[s.ptr_slot] + o0);
        const uint32_t* master = reinterpret_cast<const uint32_t*>(ptrs[s.ptr_slot + n_tensors] + 2 * o0);
        const uint64_t ib = s.index_base + o0 / 2;
        const bool vec =
            ((reinterpret_cast<uintptr_t>(param) & 15) == 0) && ((reinterpret_cast<uintptr_t>(master) & 15) == 0);
        const uint64_t nv = vec ? n / 8 : 0;
        for (uint64_t v = threadIdx.x; v < nv; v += kThreads) {
            const uint4 r = rne_8(ld_stream(master + 8 * v), ld_stream(master + 8 * v + 4));
            if (kCheck) {
                const uint4 x = ld_stream(param + 8 * v);
                miss |= (x.x != r.x) | (x.y != r.y) | (x.z != r.z) | (x.w != r.w);
                c.add_vec(x, 2, ib + 8 * v);
            } else {
                st_v4(param + 8 * v, r);
                c.add_vec(r, 2, ib + 8 * v);
            }
        }
        for (uint64_t e = nv * 8 + threadIdx.x; e < n; e += kThreads) {
            const uint32_t r = rne_bf16(master[e]);
            uint32_t b = r;
            if (kCheck) {
                b = param[e];
                miss |= (b != r);
            } else {
                param[e] = (uint16_t)r;
            }
            c.add_elem(b, ib + e);
        }
    }
    if (cseg != 0xFFFFFFFFu) block_reduce_add(c, cks + 2 * cseg);
    if (kCheck && __syncthreads_or(miss) && threadIdx.x == 0) atomicAdd(bad, 1);
}

static int g_num_sms = 0;

cudaError_t launch_derive(bool check, const PackItem* items, uint32_t n_items, const SegDev* segs, const uint64_t* ptrs,
                          uint32_t n_tensors, unsigned long long* cks, int* bad, cudaStream_t s) {
    if (!n_items) return cudaSuccess;
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    const uint32_t cap = (uint32_t)g_num_sms * 8u;                 // 8 x 256 threads resident per SM
    const uint32_t grid = n_items < cap ? n_items : cap;
    if (check) derive_kernel<true><<<grid, kThreads, 0, s>>>(items, n_items, segs, ptrs, n_tensors, cks, bad);
    else derive_kernel<false><<<grid, kThreads, 0, s>>>(items, n_items, segs, ptrs, n_tensors, cks, bad);
    return cudaGetLastError();
}

__global__ void cast_kernel(const uint32_t* __restrict__ src, uint16_t* __restrict__ dst, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(src) & 15) == 0) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
    uint64_t done = 0;
    if (vec) {
        const uint64_t nv = n / 8;
        for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv; v += stride)
            st_v4(dst + 8 * v, rne_8(ld_stream(src + 8 * v), ld_stream(src + 8 * v + 4)));
        done = nv * 8;
    }
    for (uint64_t e = done + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n; e += stride)
        dst[e] = (uint16_t)rne_bf16(src[e]);
}

// ---- K6: counter-based synthetic generator (D2) ---------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__constant__ uint32_t c_specials[16] = {
    0x00000000u, 0x80000000u, 0x00000001u, 0x00018000u, 0x007FFFFFu, 0x3F808000u, 0x3F818000u, 0x3F808001u,
    0x3F807FFFu, 0x7F7FFFFFu, 0x7F7F8000u, 0x7F800000u, 0xFF800000u, 0x7FC00000u, 0x7F800001u, 0xFFC12345u};

__global__ void synth_kernel(void* __restrict__ dst, int kind, uint64_t base, uint64_t index_base, uint64_t n,
                             int special_bits) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t smask = special_bits > 0 ? ((1ull << special_bits) - 1) : 0;
    const uint32_t lo = kind == 1 ? 0x76u : kind == 2 ? 0x68u : 0x58u;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t z = splitmix64(base ^ (index_base + i));
        if (kind == 0) {
            const uint32_t b = (uint32_t)(z >> 63) << 15 | (0x76u + (uint32_t)((z >> 32) & 7)) << 7 |
                               (uint32_t)((z >> 8) & 0x7F);
            reinterpret_cast<uint16_t*>(dst)[i] = (uint16_t)b;
        } else {
            const uint32_t sign = kind == 3 ? 0u : (uint32_t)(z >> 63);
            uint32_t b = sign << 31 | (lo + (uint32_t)((z >> 32) & 7)) << 23 | (uint32_t)((z >> 8) & 0x7FFFFF);
            if (special_bits > 0 && (z & smask) == 0) b = c_specials[(z >> 20) & 15];
            reinterpret_cast<uint32_t*>(dst)[i] = b;
        }
    }
}

__global__ void mutate_kernel(void* __restrict__ buf, int esize, uint64_t base, uint64_t index_base, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t m = (uint32_t)(splitmix64(base ^ (index_base + i)) & 0xFF);
        if (esize == 4) reinterpret_cast<uint32_t*>(buf)[i] ^= m;
        else reinterpret_cast<uint16_t*>(buf)[i] ^= (uint16_t)m;
    }
}

// ---- K7: checksum of an arbitrary contiguous tensor -------------------------
__global__ void __launch_bounds__(kThreads) checksum_kernel(const uint8_t* __restrict__ src, int es,
                                                            uint64_t index_base, uint64_t n_elems,
                                                            unsigned long long* __restrict__ out) {
    Cks c;
    const uint64_t stride = (uint64_t)gridDim.x * kThreads;
    const bool vec = (reinterpret_cast<uintptr_t>(src) & 15) == 0;
    const uint32_t epv = 16 / es;
    const uint64_t nv = vec ? n_elems / epv : 0;
    for (uint64_t v = blockIdx.x * (uint64_t)kThreads + threadIdx.x; v < nv; v += stride)
        c.add_vec(ld_stream(src + 16 * v), es, index_base + v * epv);
    for (uint64_t e = nv * epv + blockIdx.x * (uint64_t)kThreads + threadIdx.x; e < n_elems; e += stride) {
        const uint32_t b = es == 4 ? reinterpret_cast<const uint32_t*>(src)[e] : reinterpret_cast<const uint16_t*>(src)[e];
        c.add_elem(b, index_base + e);
    }
    block_reduce_add(c, out);
}

// ---- launchers ----------------------------------------------------------------
static int g_pack_variant = 0;          // diagnostic only (plex_diag_pack_variant)

template <bool kPack, int kHint>
static cudaError_t launch_pack_t(const PackItem* items, uint32_t n_items, const SegDev* segs, const uint64_t* ptrs,
                                 uint8_t* staging, uint64_t bucket_lo, unsigned long long* cks, unsigned int* ctr,
                                 cudaStream_t s) {
    static bool attr[64] = {};                 // per device: the attribute lives in each context
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(pack_kernel<kPack, PackCfg, kHint>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)PackCfg::kSmem);
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < 64) attr[dev] = true;
    }
    const uint32_t cap = (uint32_t)g_num_sms * PackCfg::kCtasPerSm;
    const uint32_t grid = n_items < cap ? n_items : cap;
    // Claim order: item (c * perm) mod n with perm ~ n/3 coprime to n, so the
    // ~600 items in flight at any moment are spread over the whole bucket
    // instead of one contiguous ~40 MB window: +20-25 % DRAM throughput on
    // large tensors (profiles/r01_kbench_spread.log).
    uint32_t perm = 1;
    if (n_items > 2) {
        uint32_t m = (n_items / 3u) | 1u;
        auto gcd = [](uint32_t a, uint32_t b) { while (b) { uint32_t t = a % b; a = b; b = t; } return a; };
        while (gcd(m, n_items) != 1) m += 2;
        perm = m;
    }
    pack_kernel<kPack, PackCfg, kHint><<<grid, PackCfg::kThreads, PackCfg::kSmem, s>>>(items, n_items, segs, ptrs,
                                                                                       staging, bucket_lo, cks, ctr, perm);
    return cudaGetLastError();
}

cudaError_t launch_pack(bool pack, const PackItem* items, uint32_t n_items, const SegDev* segs, const uint64_t* ptrs,
                        uint8_t* staging, uint64_t bucket_lo, unsigned long long* cks, unsigned int* ctr,
                        cudaStream_t s) {
    if (n_items == 0) return cudaSuccess;
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    if (g_pack_variant == 1)
        return pack ? launch_pack_t<true, 1>(items, n_items, segs, ptrs, staging, bucket_lo, cks, ctr, s)
                    : launch_pack_t<false, 1>(items, n_items, segs, ptrs, staging, bucket_lo, cks, ctr, s);
    return pack ? launch_pack_t<true, 0>(items, n_items, segs, ptrs, staging, bucket_lo, cks, ctr, s)
                : launch_pack_t<false, 0>(items, n_items, segs, ptrs, staging, bucket_lo, cks, ctr, s);
}

void set_pack_variant(int v) { g_pack_variant = v; }

cudaError_t launch_verify(const unsigned long long* got, const unsigned long long* want, uint32_t n, int* bad,
                          cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint32_t blocks = (n + kThreads - 1) / kThreads;
    verify_kernel<<<blocks < 1024 ? blocks : 1024, kThreads, 0, s>>>(got, want, n, bad);
    return cudaGetLastError();
}

// One CTA per item: a persistent grid-stride variant (148 x 8 CTAs) measured
// 0.82 vs 0.92 of the peer copy at 7B TP-2 x DP-2 and 0.88 vs 1.06 of HBM at
// 32B TP-4 (profiles/r02aa_push_persistent_ab.jsonl): the block scheduler's
// dynamic placement of 64 KiB items beats a static stride.
cudaError_t launch_push(bool cast, const PushItem* items, uint64_t n_items, const uint64_t* src_ptrs,
                        const uint64_t* dst_arenas, cudaStream_t s) {
    if (!n_items) return cudaSuccess;
    // one CTA per item; grid.x limit is 2^31-1: chunk very long item lists
    const uint64_t kMax = 1ull << 30;
    for (uint64_t o = 0; o < n_items; o += kMax) {
        const uint64_t n = n_items - o < kMax ? n_items - o : kMax;
        if (cast) push_kernel<true><<<(uint32_t)n, kThreads, 0, s>>>(items + o, n, src_ptrs, dst_arenas);
        else push_kernel<false><<<(uint32_t)n, kThreads, 0, s>>>(items + o, n, src_ptrs, dst_arenas);
    }
    return cudaGetLastError();
}

// ---- NEXT-1 carried buckets over peer memory: cross-GPU stream handshakes --------------
// One thread.  signal: make this stream's prior work visible system-wide, then
// publish `v` at `flag` (local or peer-mapped).  wait: spin (acquire, system
// scope) until `*flag >= v`; gives up after `timeout_ns` and raises `*err`
// instead of hanging the GPU.
__global__ void signal_kernel(unsigned long long* flag, unsigned long long v) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void wait_kernel(const unsigned long long* flag, unsigned long long v, unsigned long long timeout_ns,
                            int* err) {
    const unsigned long long t0 = globaltimer_ns();
    for (;;) {
        unsigned long long x;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(flag) : "memory");
        if (x >= v) return;
        if (globaltimer_ns() - t0 > timeout_ns) {
            atomicExch(err, 1);
            return;
        }
        __nanosleep(1000);
    }
}

cudaError_t launch_signal(unsigned long long* flag, unsigned long long v, cudaStream_t s) {
    signal_kernel<<<1, 1, 0, s>>>(flag, v);
    return cudaGetLastError();
}

cudaError_t launch_wait(const unsigned long long* flag, unsigned long long v, unsigned long long timeout_ns, int* err,
                        cudaStream_t s) {
    wait_kernel<<<1, 1, 0, s>>>(flag, v, timeout_ns, err);
    return cudaGetLastError();
}

static inline uint32_t grid_for(uint64_t work, uint32_t per_block) {
    uint64_t b = (work + per_block - 1) / per_block;
    const uint64_t cap = 148ull * 16;
    if (b > cap) b = cap;
    return b ? (uint32_t)b : 1u;
}

cudaError_t launch_cast(const void* src, void* dst, uint64_t n, cudaStream_t s) {
    if (!n) return cudaSuccess;
    cast_kernel<<<grid_for(n / 8 + 1, kThreads), kThreads, 0, s>>>(reinterpret_cast<const uint32_t*>(src),
                                                                     reinterpret_cast<uint16_t*>(dst), n);
    return cudaGetLastError();
}

cudaError_t launch_synth(void* dst, int kind, uint64_t base, uint64_t index_base, uint64_t n, int special_bits,
                         cudaStream_t s) {
    if (!n) return cudaSuccess;
    synth_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(dst, kind, base, index_base, n, special_bits);
    return cudaGetLastError();
}

cudaError_t launch_mutate(void* buf, int esize, uint64_t base, uint64_t index_base, uint64_t n, cudaStream_t s) {
    if (!n) return cudaSuccess;
    mutate_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(buf, esize, base, index_base, n);
    return cudaGetLastError();
}

cudaError_t launch_checksum(const void* src, int es, uint64_t index_base, uint64_t n, unsigned long long* out,
                            cudaStream_t s) {
    if (!n) return cudaSuccess;
    checksum_kernel<<<grid_for(n / (16 / es) + 1, kThreads), kThreads, 0, s>>>(
        reinterpret_cast<const uint8_t*>(src), es, index_base, n, out);
    return cudaGetLastError();
}

}  // namespace plex
