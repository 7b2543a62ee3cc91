// a1 executed: the GPU group's residency authority (pure host; every byte is
// moved by the exported transfer calls of plex_runtime.cu).
//
// PAPER.md:555 (§5.2.2 "Automatic Context Switching"): "the scheduler
// maintains a map (group_executor_gpu_job) tracking the Job ID currently
// resident on each GPU group.  In the _handle_job_transition function, the
// system compares the incoming operation's target Job ID with this map.  If
// they differ, the system automatically prepends offload and load operations".
// PAPER.md:506 (§4.5): the StateManager is the "single node-local authority
// over residency".  R17: one resident job per GPU group.
//
// plex_group_transition takes the op list from transition_ops() (the decision
// plex_transition_plan reports too) and executes it, choosing how each switch
// runs from what fits: an in-place swap for jobs sharing device storage, a
// duplex switch when the incoming job's storage can be acquired beside the
// resident one, a sequential offload -> release -> acquire -> onload otherwise.
#include <cstring>
#include <map>
#include <new>
#include <vector>

#include "plex_internal.h"

namespace plex {

struct GroupJob {
    plex_plan_t plan = nullptr;
    plex_slab_t slab = nullptr;
    int64_t storage = 0;                 // key into Group::storages
};

struct Storage {                         // one set of device tensors
    std::vector<void*> ptrs;             // PLEX_NUM_KINDS x n_tensors
    bool allocated = false;
    bool shared = false;                 // swap partners (storage_id >= 0)
};

}  // namespace plex

using namespace plex;

struct plex_group_s {
    plex_ctx_t ctx = nullptr;
    plex_storage_fn storage = nullptr;
    void* user = nullptr;
    int64_t resident = -1;
    std::map<int64_t, GroupJob> jobs;
    std::map<int64_t, Storage> storages;  // own storage: key -1 - job; shared: storage_id
};

namespace plex {

static size_t table_size(plex_plan_t plan) { return (size_t)PLEX_NUM_KINDS * plan->p.tensors.size(); }

static int32_t residency_of(plex_slab_t s) {
    void* h = nullptr;
    uint64_t n = 0;
    int32_t r = -1;
    if (!s || plex_slab_info(s, &h, &n, &r) != PLEX_OK) return -1;
    return r;
}

static plex_status acquire(plex_group_s* g, int64_t job, Storage& st, bool* ok) {
    *ok = true;
    if (st.allocated) return PLEX_OK;
    if (!g->storage) { set_error("job %lld has no device storage and the group has no storage callback", (long long)job); return PLEX_E_STATE; }
    std::vector<void*> t(st.ptrs.size(), nullptr);
    if (g->storage(g->user, job, 1, t.data(), (int32_t)t.size()) != 0) { *ok = false; return PLEX_OK; }
    st.ptrs.swap(t);
    st.allocated = true;
    return PLEX_OK;
}

static plex_status release(plex_group_s* g, int64_t job, Storage& st) {
    if (!st.allocated || st.shared || !g->storage) return PLEX_OK;      // shared / unmanaged storage stays
    std::vector<void*> t(st.ptrs.size(), nullptr);
    if (g->storage(g->user, job, 0, t.data(), (int32_t)t.size()) != 0) {
        set_error("storage callback failed to release job %lld", (long long)job);
        return PLEX_E_INVAL;
    }
    st.allocated = false;
    return PLEX_OK;
}

// after a failed transfer: the map follows the slabs (a resident job's slab is DEVICE)
static void resync_resident(plex_group_s* g, int64_t a, int64_t b) {
    g->resident = -1;
    for (int64_t j : {a, b}) {
        if (j < 0) continue;
        const GroupJob& J = g->jobs[j];
        if (J.slab && residency_of(J.slab) == PLEX_RES_DEVICE) g->resident = j;
    }
}

}  // namespace plex

extern "C" {

plex_status plex_group_create(plex_ctx_t ctx, plex_storage_fn storage, void* user, plex_group_t* out) {
    if (!ctx || !out) { set_error("NULL ctx/out"); return PLEX_E_INVAL; }
    *out = nullptr;
    try {
        auto* g = new plex_group_s();
        g->ctx = ctx;
        g->storage = storage;
        g->user = user;
        *out = g;
    } catch (const std::bad_alloc&) {
        set_error("out of host memory");
        return PLEX_E_INVAL;
    }
    return PLEX_OK;
}

plex_status plex_group_destroy(plex_group_t g) {
    delete g;
    return PLEX_OK;
}

plex_status plex_group_add_job(plex_group_t g, int64_t job, plex_plan_t plan, plex_slab_t slab, int64_t storage_id,
                               uint32_t flags, void* const* state, int32_t n_state) {
    if (!g || !plan || job < 0) { set_error("NULL group/plan or negative job id"); return PLEX_E_INVAL; }
    if (g->jobs.count(job)) { set_error("job %lld already registered", (long long)job); return PLEX_E_INVAL; }
    if (flags & ~PLEX_GROUP_RESIDENT) { set_error("bad flags"); return PLEX_E_INVAL; }
    CtxInfo ci;
    ctx_query(g->ctx, &ci);
    if (plan->p.world != ci.world) { set_error("plan world %d != ctx world %d", plan->p.world, ci.world); return PLEX_E_INVAL; }
    if ((plan->p.flags & PLEX_PLAN_REPLICA_PARAM) && ci.world > 1 && !ci.has_comm) {
        set_error("replicated-param plans need a ctx with an NCCL communicator (the all-gather after onload)");
        return PLEX_E_INVAL;
    }
    const size_t nt = table_size(plan);
    if (state && (size_t)n_state != nt) { set_error("state table needs %zu pointers, got %d", nt, n_state); return PLEX_E_INVAL; }
    const bool resident = flags & PLEX_GROUP_RESIDENT;
    if (resident && !state) { set_error("a resident job needs its state pointer table"); return PLEX_E_INVAL; }
    if (resident && g->resident >= 0) {
        set_error("job %lld is already resident on this group (one resident job per group, R17)", (long long)g->resident);
        return PLEX_E_STATE;
    }
    if (slab && residency_of(slab) < 0) { set_error("bad slab"); return PLEX_E_INVAL; }
    if (!resident && (!slab || residency_of(slab) != PLEX_RES_HOST)) {
        set_error("a non-resident job needs a slab holding its offloaded (HOST) state");
        return PLEX_E_STATE;
    }
    if (resident && slab && residency_of(slab) == PLEX_RES_HOST) {
        set_error("resident job registered with a slab that holds offloaded state");
        return PLEX_E_STATE;
    }
    const int64_t key = storage_id >= 0 ? storage_id : -1 - job;
    auto sit = g->storages.find(key);
    if (storage_id >= 0 && sit != g->storages.end()) {
        // a swap partner: same plan layout, one set of tensors
        for (auto& kv : g->jobs)
            if (kv.second.storage == key && kv.second.plan->p.id != plan->p.id) {
                set_error("jobs sharing storage %lld must share one plan", (long long)storage_id);
                return PLEX_E_INVAL;
            }
        if (state) {
            for (size_t i = 0; i < nt; ++i)
                if (sit->second.allocated && sit->second.ptrs[i] != state[i]) {
                    set_error("jobs sharing storage %lld were given different tensors", (long long)storage_id);
                    return PLEX_E_INVAL;
                }
        }
    }
    Storage& st = g->storages[key];
    st.shared = storage_id >= 0;
    if (st.ptrs.empty()) st.ptrs.assign(nt, nullptr);
    if (state && !st.allocated) {
        st.ptrs.assign(state, state + nt);
        st.allocated = true;
    }
    g->jobs[job] = GroupJob{plan, slab, key};
    if (resident) g->resident = job;
    return PLEX_OK;
}

plex_status plex_group_resident(plex_group_t g, int64_t* job) {
    if (!g || !job) { set_error("NULL argument"); return PLEX_E_INVAL; }
    *job = g->resident;
    return PLEX_OK;
}

plex_status plex_group_job_slab(plex_group_t g, int64_t job, plex_slab_t* slab) {
    if (!g || !slab) { set_error("NULL argument"); return PLEX_E_INVAL; }
    auto it = g->jobs.find(job);
    if (it == g->jobs.end()) { set_error("job %lld not registered", (long long)job); return PLEX_E_INVAL; }
    *slab = it->second.slab;
    return PLEX_OK;
}

plex_status plex_group_transition(plex_group_t g, int64_t incoming, int32_t op, void* const* dst_arenas,
                                  int32_t n_arenas, void* caller_stream, plex_transition* out) {
    if (!g) { set_error("NULL group"); return PLEX_E_INVAL; }
    auto iit = g->jobs.find(incoming);
    if (iit == g->jobs.end()) { set_error("job %lld not registered", (long long)incoming); return PLEX_E_INVAL; }
    if (op != PLEX_OP_NONE && op != PLEX_OP_SYNC) { set_error("op must be PLEX_OP_NONE or PLEX_OP_SYNC"); return PLEX_E_INVAL; }
    CtxInfo ci;
    ctx_query(g->ctx, &ci);
    GroupJob& I = iit->second;
    if (op == PLEX_OP_SYNC) {
        if (I.plan->p.tp == 0) { set_error("job %lld's plan has no rollout layout", (long long)incoming); return PLEX_E_INVAL; }
        if (!dst_arenas || (n_arenas != 1 && n_arenas != ci.world)) {
            set_error("SYNC needs 1 arena (collective) or world = %d arenas (emulation)", ci.world);
            return PLEX_E_INVAL;
        }
    }
    plex_transition t;
    transition_ops(g->resident, incoming, op, &t);
    const int64_t R = g->resident;
    Storage& SI = g->storages[I.storage];
    plex_status st = PLEX_OK;
    if (R != incoming) {
        if (!I.slab || residency_of(I.slab) != PLEX_RES_HOST) {
            set_error("job %lld's state is not in its slab (HOST)", (long long)incoming);
            return PLEX_E_STATE;
        }
        const bool carry = !I.plan->p.carry.empty();
        if (R < 0) {                                                  // [ONLOAD I]
            bool ok;
            if ((st = acquire(g, incoming, SI, &ok))) return st;
            if (!ok) { set_error("cannot acquire device storage for job %lld", (long long)incoming); return PLEX_E_TIER_FULL; }
            st = plex_state_onload(g->ctx, I.plan, I.slab, SI.ptrs.data(), (int32_t)SI.ptrs.size(), caller_stream);
            t.mode = PLEX_SWITCH_LOAD;
            if (st) { resync_resident(g, -1, incoming); return st; }
        } else {                                                      // [OFFLOAD R, ONLOAD I]
            GroupJob& A = g->jobs[R];
            Storage& SA = g->storages[A.storage];
            if (A.storage == I.storage) {
                // in place: the pair's slab takes the outgoing state, the tensors the incoming one
                t.mode = PLEX_SWITCH_SWAP;
                st = plex_state_swap(g->ctx, I.plan, SI.ptrs.data(), (int32_t)SI.ptrs.size(), I.slab, caller_stream);
                if (st && st != PLEX_E_CHECKSUM) return st;          // validation errors: nothing moved
                std::swap(A.slab, I.slab);                           // the slab now holds R
                g->resident = st ? -1 : incoming;                    // E_CHECKSUM: R safe in the slab
                if (st) return st;
            } else {
                const bool fits_staging =
                    ci.staging_bytes >= (uint64_t)ci.n_slots * (A.plan->p.bucket + I.plan->p.bucket);
                bool duplex = fits_staging && A.slab != nullptr;
                if (!A.slab) { set_error("resident job %lld has no slab to offload into", (long long)R); return PLEX_E_STATE; }
                if (duplex) {
                    bool ok;
                    if ((st = acquire(g, incoming, SI, &ok))) return st;
                    if (!ok && (carry || !A.plan->p.carry.empty())) {
                        set_error("cannot acquire device storage for job %lld beside the resident one (carried-bucket "
                                  "plans need every rank on the same path)", (long long)incoming);
                        return PLEX_E_TIER_FULL;
                    }
                    duplex = ok;
                }
                if (duplex) {
                    t.mode = PLEX_SWITCH_DUPLEX;
                    st = plex_state_switch(g->ctx, A.plan, SA.ptrs.data(), (int32_t)SA.ptrs.size(), A.slab, I.plan,
                                           I.slab, SI.ptrs.data(), (int32_t)SI.ptrs.size(), caller_stream);
                    if (st) { resync_resident(g, R, incoming); if (g->resident != R) (void)release(g, R, SA); return st; }
                    if ((st = release(g, R, SA))) { g->resident = incoming; return st; }
                } else {
                    t.mode = PLEX_SWITCH_SEQUENTIAL;
                    st = plex_state_offload(g->ctx, A.plan, SA.ptrs.data(), (int32_t)SA.ptrs.size(), A.slab, caller_stream);
                    if (st) return st;                                // R still resident, untouched
                    g->resident = -1;
                    if ((st = release(g, R, SA))) return st;
                    bool ok;
                    if ((st = acquire(g, incoming, SI, &ok))) return st;
                    if (!ok) { set_error("cannot acquire device storage for job %lld", (long long)incoming); return PLEX_E_TIER_FULL; }
                    st = plex_state_onload(g->ctx, I.plan, I.slab, SI.ptrs.data(), (int32_t)SI.ptrs.size(), caller_stream);
                    if (st) { resync_resident(g, -1, incoming); return st; }
                }
            }
        }
        g->resident = incoming;
        // NEXT-2 canonical dedup: the other ranks' rows of the replicated params
        if (I.plan->p.flags & PLEX_PLAN_REPLICA_PARAM && (I.plan->p.kind_mask & (1u << PLEX_KIND_PARAM)) && ci.world > 1) {
            void* arena = SI.ptrs[0];                                 // tensor 0's replica sits at arena offset 0
            if (!arena) { set_error("replicated-param job %lld: no param arena pointer", (long long)incoming); return PLEX_E_INVAL; }
            if ((st = plex_param_allgather(g->ctx, I.plan, arena, caller_stream))) return st;
        }
    }
    if (op == PLEX_OP_SYNC) {
        const size_t nt = I.plan->p.tensors.size();
        std::vector<const void*> masters(nt);
        for (size_t k = 0; k < nt; ++k) {
            masters[k] = SI.ptrs[PLEX_KIND_MASTER * nt + k];
            if (!masters[k]) {
                int64_t a = 0, b = 0;
                plex_plan_shard_rows(I.plan, ci.rank, (int32_t)k, &a, &b);
                if (b > a) { set_error("SYNC: job %lld has no master shard of tensor %zu", (long long)incoming, k); return PLEX_E_INVAL; }
            }
        }
        if (n_arenas == 1 && ci.world > 1 && !ci.has_comm) {
            set_error("collective SYNC needs a ctx with an NCCL communicator (pass world arenas to emulate)");
            return PLEX_E_INVAL;
        }
        st = n_arenas == 1 && (ci.world == 1 || ci.has_comm)
                 ? plex_weight_sync(g->ctx, I.plan, masters.data(), (int32_t)nt, dst_arenas[0], caller_stream)
                 : plex_weight_sync_rank(g->ctx, I.plan, ci.rank, masters.data(), (int32_t)nt, dst_arenas, n_arenas,
                                         caller_stream);
        if (st) return st;
    }
    t.resident_after = g->resident;
    if (out) *out = t;
    return PLEX_OK;
}

}  // extern "C"
