// First-fit sub-allocator over a caller-provided region (the device metadata
// workspace of plex_ctx_create): offsets only, no CUDA, so it is unit-tested
// on the host (tests/test_heap_cpu.py).  256-B granules; a free coalesces
// with both neighbours.  Not thread-safe by itself (the ctx holds a mutex).
#pragma once

#include <algorithm>
#include <cstdint>
#include <iterator>
#include <map>

namespace plex {

class OffsetHeap {
  public:
    static constexpr uint64_t kGranule = 256;
    static constexpr uint64_t kNone = ~0ull;

    void reset(uint64_t bytes) {
        bytes_ = bytes & ~(kGranule - 1);
        free_.clear();
        used_.clear();
        in_use_ = high_water_ = 0;
        if (bytes_) free_[0] = bytes_;
    }
    // offset of a block of >= n bytes, or kNone when no free block is large enough
    uint64_t alloc(uint64_t n) {
        if (!n) return kNone;
        const uint64_t need = (n + kGranule - 1) & ~(kGranule - 1);
        for (auto it = free_.begin(); it != free_.end(); ++it) {
            if (it->second < need) continue;
            const uint64_t off = it->first, sz = it->second;
            free_.erase(it);
            if (sz > need) free_[off + need] = sz - need;
            used_[off] = need;
            in_use_ += need;
            high_water_ = std::max(high_water_, in_use_);
            return off;
        }
        return kNone;
    }
    // false for an offset that is not the start of a live block
    bool free(uint64_t off) {
        auto u = used_.find(off);
        if (u == used_.end()) return false;
        uint64_t o = off, sz = u->second;
        in_use_ -= sz;
        used_.erase(u);
        auto nx = free_.lower_bound(o);
        if (nx != free_.end() && o + sz == nx->first) {      // merge with the next free block
            sz += nx->second;
            nx = free_.erase(nx);
        }
        if (nx != free_.begin()) {                            // ... and the previous one
            auto pv = std::prev(nx);
            if (pv->first + pv->second == o) {
                pv->second += sz;
                return true;
            }
        }
        free_[o] = sz;
        return true;
    }
    uint64_t bytes() const { return bytes_; }
    uint64_t in_use() const { return in_use_; }
    uint64_t high_water() const { return high_water_; }
    size_t free_blocks() const { return free_.size(); }
    uint64_t largest_free() const {
        uint64_t m = 0;
        for (auto& kv : free_) m = std::max(m, kv.second);
        return m;
    }

  private:
    uint64_t bytes_ = 0;
    std::map<uint64_t, uint64_t> free_;      // offset -> size
    std::map<uint64_t, uint64_t> used_;      // offset -> size
    uint64_t in_use_ = 0, high_water_ = 0;
};

}  // namespace plex
