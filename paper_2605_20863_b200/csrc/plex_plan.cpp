// a1 + a2: transition decision and plan (pure host; no CUDA calls).
//
// a1 — PAPER.md:555 (§5.2.2 "Automatic Context Switching"): if the incoming
//      operation's job differs from the resident one, prepend offload(resident)
//      and load(incoming).
// a2 — canonical manifest ("indexing offloaded tensors by logical
//      keys") -> per-rank slab segments (R4), bucket/work-item tables (R5),
//      rollout destination tensors (R3) and the zero-redundancy
//      push ledger.
#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <unordered_map>
#include <new>

#include "plex_internal.h"

namespace plex {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

static std::atomic<uint64_t> g_plan_ids{1};

// a1 -- PAPER.md:555 (§5.2.2): "compares the incoming operation's target Job ID
// with this map.  If they differ, the system automatically prepends offload and
// load operations".  resident < 0 = nothing resident (load only).
void transition_ops(int64_t resident, int64_t incoming, int32_t op, plex_transition* out) {
    plex_transition t{};
    t.mode = PLEX_SWITCH_NONE;
    t.resident_before = resident < 0 ? -1 : resident;
    auto add = [&](int32_t o, int64_t j) { t.ops[t.n_ops] = o; t.op_jobs[t.n_ops] = j; ++t.n_ops; };
    if (resident != incoming) {
        if (resident >= 0) add(PLEX_OP_OFFLOAD, resident);
        if (incoming >= 0) add(PLEX_OP_ONLOAD, incoming);
    }
    if (op == PLEX_OP_SYNC) add(PLEX_OP_SYNC, incoming);
    t.resident_after = incoming >= 0 ? incoming : t.resident_before;
    *out = t;
}

// ---- R3 roles from parameter keys (PLEX_ROLE_AUTO) -----------------------------
// Hugging Face / Qwen key conventions -> (role, fused group name, slot, expert,
// unit).  Plain string parsing (75k keys for Qwen3-30B-A3B).
static bool starts(const std::string& s, const char* p) { return s.compare(0, strlen(p), p) == 0; }
static bool ends(const std::string& s, const char* p) {
    const size_t n = strlen(p);
    return s.size() >= n && s.compare(s.size() - n, n, p) == 0;
}

// "model.layers.<N>." prefix length (0 if the key is not a layer parameter)
static size_t layer_prefix(const std::string& k) {
    static const char* L = "model.layers.";
    if (!starts(k, L)) return 0;
    size_t i = strlen(L), j = i;
    while (j < k.size() && k[j] >= '0' && k[j] <= '9') ++j;
    if (j == i || j >= k.size() || k[j] != '.') return 0;
    return j + 1;
}

struct AutoRole {
    int32_t role, slot, expert, unit;
    std::string group;
};

static AutoRole classify(const std::string& key, int32_t head_dim) {
    AutoRole a{PLEX_ROLE_REPLICATED, 0, -1, 1, key};
    if (ends(key, "embed_tokens.weight") || key == "lm_head.weight") { a.role = PLEX_ROLE_COL; return a; }
    const size_t n = layer_prefix(key);
    if (!n) return a;
    const std::string pre = key.substr(0, n), rest = key.substr(n);
    for (int q = 0; q < 3; ++q) {
        const char* nm[3] = {"self_attn.q_proj.", "self_attn.k_proj.", "self_attn.v_proj."};
        if (starts(rest, nm[q])) {
            const std::string suf = rest.substr(strlen(nm[q]));
            if (suf == "weight" || suf == "bias") {
                a.role = PLEX_ROLE_COL;
                a.slot = q;
                a.unit = head_dim > 0 ? head_dim : 1;
                a.group = pre + "self_attn.qkv_proj." + suf;
            }
            return a;
        }
    }
    if (rest == "self_attn.o_proj.weight" || rest == "mlp.down_proj.weight") { a.role = PLEX_ROLE_ROW; return a; }
    if (rest == "mlp.gate_proj.weight" || rest == "mlp.up_proj.weight") {
        a.role = PLEX_ROLE_COL;
        a.slot = rest == "mlp.gate_proj.weight" ? 0 : 1;
        a.group = pre + "mlp.gate_up_proj.weight";
        return a;
    }
    static const char* E = "mlp.experts.";
    if (starts(rest, E)) {
        size_t i = strlen(E), j = i;
        while (j < rest.size() && rest[j] >= '0' && rest[j] <= '9') ++j;
        if (j == i || j >= rest.size() || rest[j] != '.' || j - i > 9) return a;
        const int32_t e = (int32_t)std::strtol(rest.substr(i, j - i).c_str(), nullptr, 10);
        const std::string w = rest.substr(j + 1);
        if (w == "gate_proj.weight" || w == "up_proj.weight") {
            a.role = PLEX_ROLE_EXPERT; a.expert = e; a.slot = 2 * e + (w == "gate_proj.weight" ? 0 : 1);
            a.group = pre + "mlp.experts.w13_weight";
        } else if (w == "down_proj.weight") {
            a.role = PLEX_ROLE_EXPERT; a.expert = e; a.slot = e;
            a.group = pre + "mlp.experts.w2_weight";
        }
    }
    return a;
}

// R2: FSDP-N dim-0 chunk of rank r: rows [min(d0, r*c), min(d0, (r+1)*c)).
static inline void fsdp_rows(int64_t d0, int32_t world, int32_t r, int64_t* a, int64_t* b) {
    int64_t c = (d0 + world - 1) / world;
    *a = std::min<int64_t>(d0, (int64_t)r * c);
    *b = std::min<int64_t>(d0, (int64_t)(r + 1) * c);
}

// R10 rank map -> (tp rank, dp rank).
static inline void coords(const Plan& p, int32_t g, int32_t* t, int32_t* d) {
    if (p.rank_map == PLEX_RANKMAP_TP_FAST) { *t = g % p.tp; *d = g / p.tp; }
    else { *t = g / p.dp; *d = g % p.dp; }
}

static plex_status build_slab(Plan& p, int32_t r) {
    RankPlan& R = p.ranks[r];
    const int32_t nt = (int32_t)p.tensors.size();
    std::vector<int> kinds;
    for (int k = 0; k < PLEX_NUM_KINDS; ++k)
        if (p.kind_mask & (1u << k)) kinds.push_back(k);
    std::vector<std::pair<int, int32_t>> order;   // (kind, tensor)
    if (p.layout == PLEX_SLAB_KIND_MAJOR) {
        for (int k : kinds) for (int32_t t : p.subset) order.emplace_back(k, t);
    } else {
        for (int32_t t : p.subset) for (int k : kinds) order.emplace_back(k, t);
    }
    uint64_t cur = 0;
    for (auto& kt : order) {
        const Tensor& T = p.tensors[kt.second];
        int64_t a, b;
        fsdp_rows(T.d0, p.world, r, &a, &b);
        const int es = kind_esize(kt.first);
        SegDev s{};
        s.slab_off = align_up(cur, kSegAlign);
        s.bytes = (uint64_t)(b - a) * (uint64_t)T.d1 * es;
        s.index_base = (uint64_t)a * (uint64_t)T.d1;
        s.ptr_slot = (uint32_t)(kt.first * nt + kt.second);
        s.esize = (uint32_t)es;
        R.segs.push_back(s);
        plex_seg_desc d{};
        d.tensor = kt.second; d.kind = kt.first; d.slab_offset = s.slab_off; d.nbytes = s.bytes;
        d.row0 = a; d.row1 = b; d.index_base = s.index_base;
        R.seg_desc.push_back(d);
        R.payload_bytes += s.bytes;
        cur = s.slab_off + s.bytes;
    }
    R.slab_bytes = align_up(cur, kSegAlign);
    // Work items: each segment's slot [off, off + align(bytes)) split at bucket
    // and tile boundaries.  Slots tile the slab exactly (R4), so every slab
    // byte belongs to exactly one item.
    const uint64_t B = p.bucket, TL = p.tile;
    for (uint32_t si = 0; si < R.segs.size(); ++si) {
        const SegDev& s = R.segs[si];
        uint64_t lo = s.slab_off, hi = s.slab_off + align_up(s.bytes, kSegAlign);
        while (lo < hi) {
            uint64_t cut = std::min(hi, std::min((lo / B + 1) * B, lo + TL));
            R.items.push_back(PackItem{lo, (uint32_t)(cut - lo), si});
            lo = cut;
        }
    }
    const int32_t nb = n_buckets(p, R);
    R.bucket_item_start.assign(nb + 1, R.items.size());
    size_t it = 0;
    for (int32_t b = 0; b < nb; ++b) {
        while (it < R.items.size() && R.items[it].slab_lo < (uint64_t)b * B) ++it;
        R.bucket_item_start[b] = it;
    }
    R.bucket_item_start[nb] = R.items.size();
    // NEXT-2: with a KIND_MAJOR slab that also carries MASTER, the leading PARAM
    // region can be derived instead of moved; the remainder gets its own bucket
    // grid starting at the first MASTER byte.
    if ((p.flags & PLEX_PLAN_ELIDE_PARAM) && p.layout == PLEX_SLAB_KIND_MAJOR &&
        (p.kind_mask & (1u << PLEX_KIND_PARAM)) && (p.kind_mask & (1u << PLEX_KIND_MASTER))) {
        uint32_t first = 0;
        while (first < R.seg_desc.size() && R.seg_desc[first].kind == PLEX_KIND_PARAM) ++first;
        if (first > 0 && first < R.seg_desc.size()) {
            const uint64_t e0 = R.segs[first].slab_off;
            R.elide_start = e0;
            while (R.n_param_items < R.items.size() && R.items[R.n_param_items].slab_lo < e0) ++R.n_param_items;
            for (uint32_t si = first; si < R.segs.size(); ++si) {
                const SegDev& sg = R.segs[si];
                uint64_t lo = sg.slab_off, hi = sg.slab_off + align_up(sg.bytes, kSegAlign);
                while (lo < hi) {
                    const uint64_t nb_edge = e0 + ((lo - e0) / B + 1) * B;
                    uint64_t cut = std::min(hi, std::min(nb_edge, lo + TL));
                    R.items_el.push_back(PackItem{lo, (uint32_t)(cut - lo), si});
                    lo = cut;
                }
            }
            const int32_t nbe = (int32_t)((R.slab_bytes - e0 + B - 1) / B);
            R.bstart_el.assign(nbe + 1, R.items_el.size());
            size_t k = 0;
            for (int32_t b = 0; b < nbe; ++b) {
                while (k < R.items_el.size() && R.items_el[k].slab_lo < e0 + (uint64_t)b * B) ++k;
                R.bstart_el[b] = k;
            }
        }
    }
    return PLEX_OK;
}

// R3 destination tensors of rollout rank g.
static plex_status build_dst(Plan& p, int32_t g, const std::vector<int32_t>& group_order,
                             const std::map<int32_t, std::vector<int32_t>>& members,
                             const std::map<int32_t, int32_t>& n_experts) {
    RankPlan& R = p.ranks[g];
    int32_t t, d;
    coords(p, g, &t, &d);
    const int32_t epr = g % p.ep;
    uint64_t cur = 0;
    for (int32_t grp : group_order) {
        const auto& mem = members.at(grp);
        const Tensor& T0 = p.tensors[mem[0]];
        DstTensor D{};
        D.group = grp;
        D.first_tensor = mem[0];
        D.rows = 0;
        D.cols = -1;
        for (int32_t ti : mem) {
            const Tensor& T = p.tensors[ti];
            if (T.role != T0.role) { set_error("group %d mixes roles", grp); return PLEX_E_INVAL; }
            Piece pc{ti, 0, T.d0, 0, T.d1, D.rows};
            switch (T.role) {
                case PLEX_ROLE_REPLICATED: break;
                case PLEX_ROLE_COL: {
                    const int64_t unit = std::max<int32_t>(1, T.unit);
                    if (T.d0 % (p.tp * unit)) {
                        set_error("%s: %lld rows not divisible by TP %d x unit %lld", T.key.c_str(),
                                  (long long)T.d0, p.tp, (long long)unit);
                        return PLEX_E_LAYOUT;
                    }
                    const int64_t n = T.d0 / p.tp;
                    pc.r0 = t * n; pc.r1 = (t + 1) * n;
                    break;
                }
                case PLEX_ROLE_ROW: {
                    if (T.d1 % p.tp) {
                        set_error("%s: %lld cols not divisible by TP %d", T.key.c_str(), (long long)T.d1, p.tp);
                        return PLEX_E_LAYOUT;
                    }
                    if (mem.size() != 1) { set_error("row-parallel group %d has %zu members", grp, mem.size()); return PLEX_E_INVAL; }
                    const int64_t n = T.d1 / p.tp;
                    pc.c0 = t * n; pc.c1 = (t + 1) * n;
                    break;
                }
                case PLEX_ROLE_EXPERT: {
                    const int32_t E = n_experts.at(grp);
                    if (E % p.ep) {
                        set_error("%s: %d experts not divisible by EP %d", T.key.c_str(), E, p.ep);
                        return PLEX_E_LAYOUT;
                    }
                    const int32_t per = E / p.ep;
                    if (T.expert / per != epr) continue;      // not on this EP rank
                    break;
                }
                default: set_error("bad role %d", T.role); return PLEX_E_INVAL;
            }
            const int64_t w = pc.c1 - pc.c0;
            if (D.cols >= 0 && D.cols != w) {
                set_error("group %d: fused pieces have different widths (%lld vs %lld)", grp,
                          (long long)D.cols, (long long)w);
                return PLEX_E_INVAL;
            }
            D.cols = w;
            D.rows += pc.r1 - pc.r0;
            D.pieces.push_back(pc);
        }
        if (D.pieces.empty()) continue;
        D.arena_off = align_up(cur, kSegAlign);
        cur = D.arena_off + (uint64_t)D.rows * (uint64_t)D.cols * 2;
        R.dst.push_back(std::move(D));
    }
    R.arena_bytes = align_up(cur, kSegAlign);
    return PLEX_OK;
}

static void emit_push(Plan& p, std::vector<std::vector<std::vector<PushItem>>>& per_src_dst, int32_t g) {
    const RankPlan& G = p.ranks[g];
    const uint64_t tile_elems = std::max<uint64_t>(8, p.tile / 4);
    for (const DstTensor& D : G.dst) {
        for (const Piece& pc : D.pieces) {
            const Tensor& T = p.tensors[pc.tensor];
            for (int32_t r = 0; r < p.world; ++r) {
                int64_t a, b;
                fsdp_rows(T.d0, p.world, r, &a, &b);
                const int64_t lo = std::max(a, pc.r0), hi = std::min(b, pc.r1);
                if (hi <= lo) continue;
                const uint64_t w = (uint64_t)(pc.c1 - pc.c0);
                const uint64_t rows = (uint64_t)(hi - lo);
                const uint64_t src0 = (uint64_t)(lo - a) * T.d1 + pc.c0;             // in r's shard
                const uint64_t dst0 = D.arena_off / 2 + (uint64_t)(pc.dst_row0 + lo - pc.r0) * D.cols;
                const uint64_t bytes = rows * w * 2;
                p.ledger[(size_t)r * p.world + g] += bytes;
                auto& out = per_src_dst[r][g];
                if (w == (uint64_t)T.d1 && w == (uint64_t)D.cols) {
                    // contiguous run of rows*w elements on both sides
                    const uint64_t n = rows * w;
                    for (uint64_t o = 0; o < n; o += tile_elems) {
                        const uint64_t c = std::min(tile_elems, n - o);
                        out.push_back(PushItem{src0 + o, dst0 + o, (uint32_t)pc.tensor, (uint32_t)g, 1,
                                               (uint32_t)c, (uint32_t)c, (uint32_t)c});
                    }
                } else {
                    const uint64_t rpi = std::max<uint64_t>(1, tile_elems / std::max<uint64_t>(1, w));
                    for (uint64_t o = 0; o < rows; o += rpi) {
                        const uint64_t c = std::min(rpi, rows - o);
                        out.push_back(PushItem{src0 + o * T.d1, dst0 + o * D.cols, (uint32_t)pc.tensor, (uint32_t)g,
                                               (uint32_t)c, (uint32_t)w, (uint32_t)T.d1, (uint32_t)D.cols});
                    }
                }
            }
        }
    }
}

// a9-a11 layout: destination tensors of every rank, the push items of every
// source rank and the ledger, for p.rank_map.
static plex_status build_sync(Plan& p) {
    std::vector<int32_t> order;
    std::map<int32_t, std::vector<int32_t>> members;
    std::map<int32_t, int32_t> n_experts;
    for (int32_t i = 0; i < (int32_t)p.tensors.size(); ++i) {
        const Tensor& T = p.tensors[i];
        if (!members.count(T.group)) order.push_back(T.group);
        members[T.group].push_back(i);
        if (T.role == PLEX_ROLE_EXPERT) n_experts[T.group] = std::max(n_experts[T.group], T.expert + 1);
    }
    for (auto& kv : members)
        std::stable_sort(kv.second.begin(), kv.second.end(),
                         [&](int32_t a, int32_t b) { return p.tensors[a].slot < p.tensors[b].slot; });
    for (int32_t g = 0; g < p.world; ++g) {
        plex_status s = build_dst(p, g, order, members, n_experts);
        if (s) return s;
    }
    std::vector<std::vector<std::vector<PushItem>>> per(p.world, std::vector<std::vector<PushItem>>(p.world));
    for (int32_t g = 0; g < p.world; ++g) emit_push(p, per, g);
    // Interleave each source's items over its destinations in proportion to
    // their sizes (always take the destination least far along its list, ties
    // broken starting at r+1): every sender then spreads its NVLink stores
    // over all peers for the whole kernel -- senders never converge on one
    // receiver, and local (HBM-only) items never bunch up into a tail while
    // the links sit idle.
    for (int32_t r = 0; r < p.world; ++r) {
        RankPlan& R = p.ranks[r];
        std::vector<size_t> pos(p.world, 0);
        size_t left = 0;
        for (int32_t g = 0; g < p.world; ++g) left += per[r][g].size();
        R.push.reserve(left);
        while (left) {
            int32_t best = -1;
            double best_f = 2.0;
            for (int32_t k = 1; k <= p.world; ++k) {
                const int32_t g = (r + k) % p.world;
                const size_t n = per[r][g].size();
                if (pos[g] >= n) continue;
                const double f = (pos[g] + 0.5) / (double)n;
                if (f < best_f) { best_f = f; best = g; }
            }
            R.push.push_back(per[r][best][pos[best]++]);
            --left;
        }
        for (const PushItem& it : R.push) R.src_read_bytes += (uint64_t)it.rows * it.cols * 4;
    }
    for (int32_t r = 0; r < p.world; ++r)
        for (int32_t g = 0; g < p.world; ++g) {
            const uint64_t b = p.ledger[(size_t)r * p.world + g];
            if (r == g) p.ranks[r].local_bytes += b;
            else { p.ranks[r].send_bytes += b; p.ranks[g].recv_bytes += b; }
        }
    return PLEX_OK;
}

// R10: the rollout rank map is a free placement choice; AUTO keeps the map
// whose zero-redundancy ledger has the smaller max over ranks of max(send, recv).
static uint64_t max_link_bytes(const Plan& p) {
    uint64_t m = 0;
    for (const RankPlan& R : p.ranks) m = std::max(m, std::max(R.send_bytes, R.recv_bytes));
    return m;
}

// NEXT-1 host-link balancing: with per-rank host-link weights w_r, the group
// needs T = sum_r S_r / sum_r w_r; ranks above T hand their last whole buckets
// to the ranks with the most spare capacity (deterministic greedy).
static plex_status build_carry(Plan& p, const float* w) {
    const int32_t W = p.world;
    double sw = 0, ss = 0;
    for (int32_t r = 0; r < W; ++r) {
        if (!(w[r] > 0)) { set_error("link weight of rank %d must be > 0", r); return PLEX_E_INVAL; }
        sw += w[r];
        ss += (double)p.ranks[r].slab_bytes;
        p.ranks[r].carried.assign(n_buckets(p, p.ranks[r]), 0);
    }
    const double T = ss / sw;
    std::vector<double> load(W);
    for (int32_t r = 0; r < W; ++r) load[r] = (double)p.ranks[r].slab_bytes;
    std::vector<char> giver(W, 0);
    std::vector<int32_t> next_b(W, 0);                       // next bucket a giver would hand off
    for (int32_t r = 0; r < W; ++r) {
        if (load[r] / w[r] > T * 1.02) giver[r] = 1;
        next_b[r] = n_buckets(p, p.ranks[r]) - 1;
    }
    for (;;) {
        // the most loaded giver hands its last remaining bucket (never bucket 0)
        // to the carrier with the most spare capacity, one bucket at a time
        int32_t r = -1;
        for (int32_t g = 0; g < W; ++g)
            if (giver[g] && next_b[g] >= 1 && load[g] / w[g] > T && (r < 0 || load[g] / w[g] > load[r] / w[r]))
                r = g;
        if (r < 0) break;
        const RankPlan& R = p.ranks[r];
        const int32_t b = next_b[r];
        const uint64_t lo = (uint64_t)b * p.bucket;
        const uint64_t len = std::min<uint64_t>(p.bucket, R.slab_bytes - lo);
        int32_t best = -1;
        double spare = 0;
        for (int32_t c = 0; c < W; ++c) {
            if (giver[c]) continue;
            const double sp = T * w[c] - load[c];
            if (sp > spare) { spare = sp; best = c; }
        }
        // only if it lowers the group's maximum
        if (best < 0 || (load[best] + (double)len) / w[best] >= load[r] / w[r]) { next_b[r] = 0; continue; }
        p.carry.push_back(CarryXfer{r, b, best, lo, len, 0});
        p.ranks[r].carried[b] = 1;
        load[r] -= (double)len;
        load[best] += (double)len;
        next_b[r] = b - 1;
    }
    std::sort(p.carry.begin(), p.carry.end(), [](const CarryXfer& a, const CarryXfer& b) {
        return a.owner != b.owner ? a.owner < b.owner : a.bucket < b.bucket;
    });
    for (CarryXfer& x : p.carry) {
        RankPlan& C = p.ranks[x.carrier];
        x.coff = C.carry_bytes;
        C.carry_bytes += align_up(x.len, kSegAlign);
        C.carried_in += 1;
        p.ranks[x.owner].carried_out += 1;
    }
    return PLEX_OK;
}

// NEXT-2 canonical dedup of the replicated bf16 params (ZeRO-2
// at :587): the slab keeps each rank's FSDP rows only; after onload every rank
// stores its rows of every param into every peer's param arena.  Items are
// contiguous runs of one tile, cycled over the peers so every link is busy for
// the whole kernel.
static plex_status build_replica(Plan& p) {
    if (!(p.kind_mask & (1u << PLEX_KIND_PARAM))) { set_error("REPLICA_PARAM needs the PARAM kind"); return PLEX_E_INVAL; }
    uint64_t cur = 0;
    p.param_off.resize(p.tensors.size());
    for (size_t t = 0; t < p.tensors.size(); ++t) {
        p.param_off[t] = align_up(cur, kSegAlign);
        cur = p.param_off[t] + (uint64_t)p.tensors[t].d0 * (uint64_t)p.tensors[t].d1 * 2;
    }
    p.param_arena_bytes = align_up(cur, kSegAlign);
    const uint64_t tile_elems = std::max<uint64_t>(8, p.tile / 2);
    for (int32_t r = 0; r < p.world; ++r) {
        RankPlan& R = p.ranks[r];
        for (int32_t t : p.subset) {
            const Tensor& T = p.tensors[t];
            int64_t a, b;
            fsdp_rows(T.d0, p.world, r, &a, &b);
            const uint64_t n = (uint64_t)(b - a) * (uint64_t)T.d1;
            const uint64_t e0 = p.param_off[t] / 2 + (uint64_t)a * (uint64_t)T.d1;
            for (uint64_t o = 0; o < n; o += tile_elems) {
                const uint32_t c = (uint32_t)std::min(tile_elems, n - o);
                for (int32_t k = 1; k < p.world; ++k)
                    R.gather.push_back(PushItem{e0 + o, e0 + o, 0, (uint32_t)((r + k) % p.world), 1, c, c, c});
            }
            R.gather_send += n * 2 * (uint64_t)(p.world - 1);
            for (int32_t g = 0; g < p.world; ++g)
                if (g != r) p.ranks[g].gather_recv += n * 2;
        }
    }
    return PLEX_OK;
}

static plex_status build(const plex_plan_req* q, Plan& p) {
    if (!q || q->n_tensors <= 0 || !q->tensors) { set_error("empty manifest"); return PLEX_E_INVAL; }
    if (q->world < 1) { set_error("world must be >= 1"); return PLEX_E_INVAL; }
    p.world = q->world;
    p.tp = q->tp; p.dp = q->dp; p.ep = q->ep > 0 ? q->ep : 1;
    p.rank_map = q->rank_map;
    p.layout = q->slab_layout;
    p.kind_mask = q->kind_mask ? q->kind_mask : PLEX_KINDMASK_ALL;
    p.bucket = q->bucket_bytes ? q->bucket_bytes : kDefaultBucket;
    p.tile = q->tile_bytes ? q->tile_bytes : kDefaultTile;
    p.flags = q->flags;
    if (p.bucket % kSegAlign || p.tile % kSegAlign || p.tile > (1ull << 31)) {
        set_error("bucket/tile must be multiples of 256 B (tile < 2 GiB)"); return PLEX_E_INVAL;
    }
    if (p.kind_mask & ~PLEX_KINDMASK_ALL) { set_error("bad kind mask"); return PLEX_E_INVAL; }
    if (p.flags & ~(PLEX_PLAN_ELIDE_PARAM | PLEX_PLAN_REPLICA_PARAM)) { set_error("bad plan flags"); return PLEX_E_INVAL; }
    if (p.layout != PLEX_SLAB_KIND_MAJOR && p.layout != PLEX_SLAB_KEY_MAJOR) { set_error("bad slab layout"); return PLEX_E_INVAL; }
    if (p.rank_map != PLEX_RANKMAP_TP_FAST && p.rank_map != PLEX_RANKMAP_DP_FAST && p.rank_map != PLEX_RANKMAP_AUTO) {
        set_error("bad rank map");
        return PLEX_E_INVAL;
    }
    const bool sync = !(p.tp == 0 && p.dp == 0);
    if (sync && (p.tp < 1 || p.dp < 1 || p.tp * p.dp != p.world)) {
        set_error("tp*dp (%d*%d) must equal world %d", p.tp, p.dp, p.world); return PLEX_E_INVAL;
    }
    if (sync && p.world % p.ep) { set_error("EP %d must divide world %d", p.ep, p.world); return PLEX_E_LAYOUT; }
    p.tensors.reserve(q->n_tensors);
    uint64_t total = 0;
    const bool autoroles = q->tensors[0].role == PLEX_ROLE_AUTO;
    std::unordered_map<std::string, int32_t> gid;
    for (int32_t i = 0; i < q->n_tensors; ++i) {
        const plex_tensor_desc& d = q->tensors[i];
        if (d.d0 < 0 || d.d1 < 1 || (d.ndim != 1 && d.ndim != 2) || (d.ndim == 1 && d.d1 != 1)) {
            set_error("tensor %d: bad shape", i); return PLEX_E_INVAL;
        }
        if (d.d1 > 0x7FFFFFFF || d.d0 > 0x7FFFFFFF) { set_error("tensor %d: dim too large", i); return PLEX_E_INVAL; }
        if ((d.role == PLEX_ROLE_AUTO) != autoroles) {
            set_error("tensor %d: PLEX_ROLE_AUTO must be used for every tensor or none", i); return PLEX_E_INVAL;
        }
        Tensor T{d.key ? d.key : "", d.d0, d.d1, d.ndim, d.role, d.group, d.slot, d.expert, d.unit};
        if (autoroles) {
            if (!d.key) { set_error("tensor %d: PLEX_ROLE_AUTO needs a key", i); return PLEX_E_INVAL; }
            const AutoRole a = classify(T.key, q->head_dim);
            auto it = gid.find(a.group);
            if (it == gid.end()) {
                it = gid.emplace(a.group, (int32_t)p.group_names.size()).first;
                p.group_names.push_back(a.group);
                p.group_role.push_back(a.role);
                p.group_experts.push_back(0);
            }
            T.role = a.role; T.group = it->second; T.slot = a.slot; T.expert = a.expert; T.unit = a.unit;
            if (a.role == PLEX_ROLE_EXPERT)
                p.group_experts[T.group] = std::max(p.group_experts[T.group], a.expert + 1);
        } else {
            if (d.role < 0 || d.role > PLEX_ROLE_EXPERT) { set_error("tensor %d: bad role", i); return PLEX_E_INVAL; }
            if (d.role == PLEX_ROLE_EXPERT && d.expert < 0) { set_error("tensor %d: expert index", i); return PLEX_E_INVAL; }
            if (d.group < 0) { set_error("tensor %d: negative group", i); return PLEX_E_INVAL; }
            if ((size_t)d.group >= p.group_names.size()) {
                p.group_names.resize(d.group + 1);
                p.group_role.resize(d.group + 1, -1);
                p.group_experts.resize(d.group + 1, 0);
            }
            if (p.group_names[d.group].empty()) { p.group_names[d.group] = T.key; p.group_role[d.group] = d.role; }
            if (d.role == PLEX_ROLE_EXPERT)
                p.group_experts[d.group] = std::max(p.group_experts[d.group], d.expert + 1);
        }
        p.tensors.push_back(std::move(T));
        total += (uint64_t)d.d0 * (uint64_t)d.d1;
    }
    if (q->n_subset > 0 && q->subset) {
        p.subset.assign(q->subset, q->subset + q->n_subset);
        std::sort(p.subset.begin(), p.subset.end());
        p.subset.erase(std::unique(p.subset.begin(), p.subset.end()), p.subset.end());
        for (int32_t t : p.subset)
            if (t < 0 || t >= q->n_tensors) { set_error("subset index %d out of range", t); return PLEX_E_INVAL; }
    } else {
        p.subset.resize(q->n_tensors);
        for (int32_t i = 0; i < q->n_tensors; ++i) p.subset[i] = i;
    }
    // a1: transition ops, the same decision the group executor takes.
    plex_plan_stats& st = p.stats;
    {
        plex_transition t;
        transition_ops(q->resident_job, q->incoming_job, q->op, &t);
        st.n_ops = t.n_ops;
        for (int i = 0; i < 4; ++i) { st.ops[i] = t.ops[i]; st.op_jobs[i] = t.op_jobs[i]; }
    }
    st.n_tensors = q->n_tensors;
    st.world = p.world; st.tp = p.tp; st.dp = p.dp; st.ep = p.ep;
    st.total_params = total;

    p.ranks.resize(p.world);
    for (int32_t r = 0; r < p.world; ++r) {
        plex_status s = build_slab(p, r);
        if (s) return s;
    }
    p.ledger.assign((size_t)p.world * p.world, 0);
    for (RankPlan& R : p.ranks) R.carried.assign(n_buckets(p, R), 0);
    if (p.flags & PLEX_PLAN_REPLICA_PARAM) {
        plex_status s2 = build_replica(p);
        if (s2) return s2;
    }
    if (q->link_weights && p.world > 1) {
        if (p.flags & PLEX_PLAN_ELIDE_PARAM) { set_error("link balancing and param elision are exclusive"); return PLEX_E_INVAL; }
        plex_status s2 = build_carry(p, q->link_weights);
        if (s2) return s2;
    }
    if (sync) {
        if (q->rank_map == PLEX_RANKMAP_AUTO) {
            int32_t best = PLEX_RANKMAP_TP_FAST;
            uint64_t best_bytes = ~0ull;
            for (int32_t m : {PLEX_RANKMAP_TP_FAST, PLEX_RANKMAP_DP_FAST}) {
                Plan t;
                t.tensors = p.tensors;
                t.world = p.world; t.tp = p.tp; t.dp = p.dp; t.ep = p.ep; t.rank_map = m;
                t.tile = p.tile;
                t.ranks.resize(p.world);
                t.ledger.assign((size_t)p.world * p.world, 0);
                plex_status s2 = build_sync(t);
                if (s2) return s2;
                const uint64_t b = max_link_bytes(t);
                if (b < best_bytes) { best_bytes = b; best = m; }
            }
            p.rank_map = best;
        }
        plex_status s2 = build_sync(p);
        if (s2) return s2;
    }
    st.rank_map = p.rank_map;
    p.id = g_plan_ids.fetch_add(1);
    return PLEX_OK;
}

}  // namespace plex

using namespace plex;

extern "C" {

const char* plex_last_error(void) { return plex::g_err; }
const char* plex_version(void) { return "plex-b200 0.1 (sm_100a)"; }

plex_status plex_transition_plan(const plex_plan_req* req, plex_plan_t* out) {
    if (!out) { set_error("out is NULL"); return PLEX_E_INVAL; }
    *out = nullptr;
    try {
        auto* h = new plex_plan_s();
        plex_status s = build(req, h->p);
        if (s) { delete h; return s; }
        *out = h;
        return PLEX_OK;
    } catch (const std::bad_alloc&) {
        set_error("out of host memory building plan");
        return PLEX_E_INVAL;
    } catch (...) {
        set_error("unexpected exception building plan");
        return PLEX_E_INVAL;
    }
}

plex_status plex_plan_query(plex_plan_t plan, plex_plan_stats* out) {
    if (!plan || !out) { set_error("NULL argument"); return PLEX_E_INVAL; }
    *out = plan->p.stats;
    return PLEX_OK;
}

plex_status plex_plan_rank_info(plex_plan_t plan, int32_t rank, plex_rank_info* out) {
    if (!plan || !out || rank < 0 || rank >= plan->p.world) { set_error("bad plan/rank"); return PLEX_E_INVAL; }
    const Plan& p = plan->p;
    const RankPlan& R = p.ranks[rank];
    plex_rank_info o{};
    o.slab_bytes = R.slab_bytes;
    o.payload_bytes = R.payload_bytes;
    o.n_segments = (int32_t)R.segs.size();
    o.n_buckets = n_buckets(p, R);
    o.n_pack_items = R.items.size();
    o.dst_arena_bytes = R.arena_bytes;
    o.n_dst_tensors = (int32_t)R.dst.size();
    o.n_push_items = R.push.size();
    o.send_bytes = R.send_bytes;
    o.recv_bytes = R.recv_bytes;
    o.local_bytes = R.local_bytes;
    o.src_read_bytes = R.src_read_bytes;
    o.elide_buckets = R.elide_start ? (int32_t)R.bstart_el.size() - 1 : 0;
    o.elide_bytes = R.elide_start;
    o.carried_out = R.carried_out;
    o.carried_in = R.carried_in;
    o.carry_bytes = R.carry_bytes;
    o.n_gather_items = R.gather.size();
    o.gather_send_bytes = R.gather_send;
    o.gather_recv_bytes = R.gather_recv;
    *out = o;
    return PLEX_OK;
}

plex_status plex_plan_segment(plex_plan_t plan, int32_t rank, int32_t i, plex_seg_desc* out) {
    if (!plan || !out || rank < 0 || rank >= plan->p.world) { set_error("bad plan/rank"); return PLEX_E_INVAL; }
    const RankPlan& R = plan->p.ranks[rank];
    if (i < 0 || i >= (int32_t)R.seg_desc.size()) { set_error("segment %d out of range", i); return PLEX_E_INVAL; }
    *out = R.seg_desc[i];
    return PLEX_OK;
}

plex_status plex_plan_dst_tensor(plex_plan_t plan, int32_t rank, int32_t i, plex_dst_desc* out) {
    if (!plan || !out || rank < 0 || rank >= plan->p.world) { set_error("bad plan/rank"); return PLEX_E_INVAL; }
    const RankPlan& R = plan->p.ranks[rank];
    if (i < 0 || i >= (int32_t)R.dst.size()) { set_error("dst tensor %d out of range", i); return PLEX_E_INVAL; }
    const DstTensor& D = R.dst[i];
    out->group = D.group;
    out->first_tensor = D.first_tensor;
    out->arena_offset = D.arena_off;
    out->rows = D.rows;
    out->cols = D.cols;
    return PLEX_OK;
}

plex_status plex_plan_group(plex_plan_t plan, int32_t group, char* buf, int32_t cap, int32_t* len, int32_t* role,
                            int32_t* n_experts) {
    if (!plan) { set_error("NULL plan"); return PLEX_E_INVAL; }
    const Plan& p = plan->p;
    if (group < 0 || group >= (int32_t)p.group_names.size() || p.group_role[group] < 0) {
        set_error("group %d out of range", group);
        return PLEX_E_INVAL;
    }
    const std::string& n = p.group_names[group];
    if (len) *len = (int32_t)n.size();
    if (buf && cap > 0) {
        const size_t k = std::min<size_t>((size_t)cap - 1, n.size());
        std::memcpy(buf, n.data(), k);
        buf[k] = '\0';
    }
    if (role) *role = p.group_role[group];
    if (n_experts) *n_experts = p.group_experts[group];
    return PLEX_OK;
}

plex_status plex_transition_decide(int64_t resident, int64_t incoming, int32_t op, plex_transition* out) {
    if (!out) { set_error("NULL out"); return PLEX_E_INVAL; }
    if (op != PLEX_OP_NONE && op != PLEX_OP_SYNC) { set_error("op must be PLEX_OP_NONE or PLEX_OP_SYNC"); return PLEX_E_INVAL; }
    if (op == PLEX_OP_SYNC && incoming < 0) { set_error("SYNC needs an incoming job"); return PLEX_E_INVAL; }
    transition_ops(resident, incoming, op, out);
    return PLEX_OK;
}

plex_status plex_plan_shard_rows(plex_plan_t plan, int32_t rank, int32_t t, int64_t* row0, int64_t* row1) {
    if (!plan || !row0 || !row1 || rank < 0 || rank >= plan->p.world || t < 0 ||
        t >= (int32_t)plan->p.tensors.size()) {
        set_error("bad shard query");
        return PLEX_E_INVAL;
    }
    fsdp_rows(plan->p.tensors[t].d0, plan->p.world, rank, row0, row1);
    return PLEX_OK;
}

plex_status plex_plan_n_carry(plex_plan_t plan, int32_t* n) {
    if (!plan || !n) { set_error("NULL argument"); return PLEX_E_INVAL; }
    *n = (int32_t)plan->p.carry.size();
    return PLEX_OK;
}

plex_status plex_plan_carry(plex_plan_t plan, int32_t i, plex_carry_desc* out) {
    if (!plan || !out || i < 0 || i >= (int32_t)plan->p.carry.size()) { set_error("bad carry index"); return PLEX_E_INVAL; }
    const CarryXfer& x = plan->p.carry[i];
    *out = plex_carry_desc{x.owner, x.bucket, x.carrier, x.lo, x.len, x.coff};
    return PLEX_OK;
}

plex_status plex_plan_ledger(plex_plan_t plan, uint64_t* bytes, int32_t n) {
    if (!plan || !bytes) { set_error("NULL argument"); return PLEX_E_INVAL; }
    const Plan& p = plan->p;
    if (n != p.world * p.world) { set_error("ledger needs world*world = %d entries", p.world * p.world); return PLEX_E_INVAL; }
    std::memcpy(bytes, p.ledger.data(), sizeof(uint64_t) * p.ledger.size());
    return PLEX_OK;
}

plex_status plex_plan_param_arena(plex_plan_t plan, int32_t t, uint64_t* offset, uint64_t* arena_bytes) {
    if (!plan) { set_error("NULL plan"); return PLEX_E_INVAL; }
    const Plan& p = plan->p;
    if (!(p.flags & PLEX_PLAN_REPLICA_PARAM)) { set_error("plan has no replicated params"); return PLEX_E_INVAL; }
    if (t >= (int32_t)p.tensors.size()) { set_error("tensor %d out of range", t); return PLEX_E_INVAL; }
    if (offset) *offset = t >= 0 ? p.param_off[t] : 0;
    if (arena_bytes) *arena_bytes = p.param_arena_bytes;
    return PLEX_OK;
}

}  // extern "C"
