// Multi-tenant layerwise transfer pool: epoch admission under a shared budget.
//
// PAPER.md Sec. 3.4: requests whose payload W = N*L*S is below Theta are served
// chunkwise on their own; every layerwise request joins a shared bandwidth pool.  Sec. 3.6
// and Alg. A2: at each scheduling epoch the pool admits the waiting
// layerwise requests under a fixed total budget, gives each a stable target rate for the whole of
// its KV load (Stall-opt / Calibrated Stall-opt or a baseline policy), and bandwidth released by
// a request that finishes early returns to the pool only at the next epoch.  Dispatch:
//   INDEPENDENT  each admitted request is its own fetch, paced byte by byte at its rate (byte b
//                released at t0 + b / r; the minimal layer pacer of a10 would let each layer burst);
//   WDRR         the epoch's admitted requests are one batched launch whose claim order is
//                weighted deficit round robin with weights r_i, each request held at r_i
//                (Alg. A2 lines 6-7; dispatch.cpp), on the first admitted request's stream.
#include <cmath>

#include "oc_internal.h"

namespace oc {

struct Tenant {
    Desc* desc;
    double s, c;          // bytes per layer, compute seconds per layer
    cudaStream_t stream;  // the request's copy stream
    double rate = 0;      // assigned at admission (bytes/s); 0 while waiting or if chunkwise
    int state = 0;        // OC_TENANT_*
    // WDRR members share one launch, whose completion event fires only when the LAST member is
    // done; a member's own completion is its last layer's ready word, turned into an event on a
    // private stream so its bandwidth returns at the next epoch after IT finishes.
    cudaStream_t done_stream = nullptr;
    cudaEvent_t layers_done = nullptr;
};

struct TenantPool {
    int policy;
    double cap, delta;
    uint64_t theta;
    int dispatch = OC_DISPATCH_INDEPENDENT;
    std::mutex mu;
    std::vector<Tenant> tenants;  // ticket = index
    struct EpochBatch {
        oc_batch* batch;
        std::vector<size_t> members;  // tickets
    };
    std::vector<EpochBatch> batches;  // WDRR launches, freed once every member has finished
    uint64_t epochs = 0;
};

}  // namespace oc

extern "C" {

OC_API int oc_pool_create(int policy, double cap_Bps, double delta_Bps, uint64_t theta_bytes, oc_tenant_pool** out) {
    if (!out) return oc::fail(OC_EINVAL, "pool_create: null out");
    *out = nullptr;
    if (policy < OC_POL_EQUAL || policy > OC_POL_CAL_STALL_OPT) return oc::fail(OC_EINVAL, "pool_create: unknown policy");
    if (!(cap_Bps > 0) || !std::isfinite(cap_Bps)) return oc::fail(OC_EINVAL, "pool_create: cap must be > 0");
    if (!(delta_Bps >= 0) || !std::isfinite(delta_Bps)) return oc::fail(OC_EINVAL, "pool_create: delta must be >= 0");
    auto p = new oc::TenantPool;
    p->policy = policy;
    p->cap = cap_Bps;
    p->delta = delta_Bps;
    p->theta = theta_bytes;
    *out = (oc_tenant_pool*)p;
    return OC_OK;
}

OC_API int oc_pool_set_dispatch(oc_tenant_pool* h, int dispatch) {
    if (!h) return oc::fail(OC_EINVAL, "pool_set_dispatch: null pool");
    if (dispatch != OC_DISPATCH_INDEPENDENT && dispatch != OC_DISPATCH_WDRR)
        return oc::fail(OC_EINVAL, "pool_set_dispatch: unknown dispatch");
    oc::TenantPool* p = (oc::TenantPool*)h;
    std::lock_guard<std::mutex> lk(p->mu);
    p->dispatch = dispatch;
    return OC_OK;
}

OC_API int oc_pool_submit(oc_tenant_pool* h, oc_desc* dh, double compute_per_layer_s, void* copy_stream,
                          uint64_t* ticket) {
    if (!h || !dh || !ticket) return oc::fail(OC_EINVAL, "pool_submit: null pointer");
    if (!(compute_per_layer_s > 0) || !std::isfinite(compute_per_layer_s))
        return oc::fail(OC_EINVAL, "pool_submit: compute window must be > 0");
    oc::TenantPool* p = (oc::TenantPool*)h;
    oc::Desc* d = (oc::Desc*)dh;
    oc::Tenant t;
    t.desc = d;
    t.s = (double)d->N * d->geo.S;
    t.c = compute_per_layer_s;
    t.stream = (cudaStream_t)copy_stream;
    const uint64_t W = d->N * d->geo.L * d->geo.S;
    std::lock_guard<std::mutex> lk(p->mu);
    *ticket = p->tenants.size();
    if (oc_select_mode(W, p->theta) == OC_DELIVER_CHUNK_MAJOR) {
        // Eq. 2 chunkwise side: served on its own, outside the shared pool.
        oc_fetch_opts o{};
        o.mode = OC_FETCH_PERSISTENT;
        o.engine = OC_COPY_BULK;
        int rc = oc::launch_fetch(d, o, t.stream);
        if (rc) return rc;
        t.state = OC_TENANT_CHUNKWISE;
    } else {
        t.state = OC_TENANT_WAITING;
    }
    p->tenants.push_back(t);
    return OC_OK;
}

OC_API int oc_pool_epoch(oc_tenant_pool* h, uint64_t* n_admitted) {
    if (!h) return oc::fail(OC_EINVAL, "pool_epoch: null pool");
    oc::TenantPool* p = (oc::TenantPool*)h;
    std::lock_guard<std::mutex> lk(p->mu);
    if (n_admitted) *n_admitted = 0;
    // 1. Requests that finished since the last epoch return their bandwidth now.
    double in_use = 0;
    for (auto& t : p->tenants) {
        if (t.state != OC_TENANT_RUNNING) continue;
        oc::DeviceGuard dg(t.desc->device);
        cudaError_t e = cudaEventQuery(t.layers_done ? t.layers_done : t.desc->done_ev);
        if (e == cudaSuccess) {
            t.state = OC_TENANT_DONE;
        } else if (e == cudaErrorNotReady) {
            in_use += t.rate;
        } else {
            return oc::cuda_fail(e, "pool_epoch: fetch failed");
        }
    }
    for (size_t k = 0; k < p->batches.size();) {  // WDRR launches whose members have all finished
        bool live = false;
        for (size_t i : p->batches[k].members) live |= p->tenants[i].state == OC_TENANT_RUNNING;
        if (live) {
            k++;
        } else {
            oc_batch_free(p->batches[k].batch);
            p->batches.erase(p->batches.begin() + k);
        }
    }
    // 2. Admit every waiting request with rates from the budget the running ones leave.
    std::vector<size_t> waiting;
    for (size_t i = 0; i < p->tenants.size(); i++)
        if (p->tenants[i].state == OC_TENANT_WAITING) waiting.push_back(i);
    p->epochs++;
    const double budget = p->cap - in_use;
    if (waiting.empty() || !(budget > 0)) return OC_OK;
    std::vector<oc_profile> prof(waiting.size());
    for (size_t k = 0; k < waiting.size(); k++)
        prof[k] = {p->tenants[waiting[k]].s, p->tenants[waiting[k]].c};
    std::vector<double> rates(waiting.size());
    int rc = oc_schedule_bandwidth(p->policy, prof.data(), prof.size(), budget, p->delta, rates.data());
    if (rc) return rc;
    // 3. Launch the admitted fetches, each held at its rate for the whole load.
    if (p->dispatch == OC_DISPATCH_WDRR) {  // one launch, WDRR claim order (Alg. A2 lines 6-7)
        std::vector<oc_desc*> ds(waiting.size());
        for (size_t k = 0; k < waiting.size(); k++) ds[k] = (oc_desc*)p->tenants[waiting[k]].desc;
        oc_batch* b = nullptr;
        rc = oc_batch_create(ds.data(), (uint32_t)ds.size(), &b);
        if (rc) return rc;
        oc_fetch_opts o{};
        o.mode = OC_FETCH_PERSISTENT;
        o.engine = OC_COPY_BULK;
        oc_wdrr_opts w{};
        w.weights = rates.data();
        w.hold_rates = 1;
        rc = oc_fetch_batch_wdrr(b, &o, &w, p->tenants[waiting[0]].stream);
        if (rc) {
            oc_batch_free(b);
            return rc;
        }
        p->batches.push_back({b, waiting});
        for (size_t k = 0; k < waiting.size(); k++) {
            oc::Tenant& t = p->tenants[waiting[k]];
            t.rate = rates[k];
            t.state = OC_TENANT_RUNNING;
            oc::DeviceGuard dg(t.desc->device);
            if (!t.done_stream) OC_CUDA(cudaStreamCreateWithFlags(&t.done_stream, cudaStreamNonBlocking));
            if (!t.layers_done) OC_CUDA(cudaEventCreateWithFlags(&t.layers_done, cudaEventDisableTiming));
            rc = oc_wait_layer((oc_desc*)t.desc, t.desc->geo.L - 1, t.done_stream);
            if (rc) return rc;
            OC_CUDA(cudaEventRecord(t.layers_done, t.done_stream));
        }
        if (n_admitted) *n_admitted = waiting.size();
        return OC_OK;
    }
    for (size_t k = 0; k < waiting.size(); k++) {
        oc::Tenant& t = p->tenants[waiting[k]];
        oc_fetch_opts o{};
        o.mode = OC_FETCH_PERSISTENT;
        o.engine = OC_COPY_BULK;
        o.pace_Bps = rates[k];
        o.pace_strict = 1;  // a held rate (Alg. A2 line 6): never above r_i, not only on average
        rc = oc::launch_fetch(t.desc, o, t.stream);
        if (rc) return rc;
        t.rate = rates[k];
        t.state = OC_TENANT_RUNNING;
        if (n_admitted) (*n_admitted)++;
    }
    return OC_OK;
}

OC_API int oc_pool_status(oc_tenant_pool* h, uint64_t ticket, int* state, double* rate_Bps) {
    if (!h) return oc::fail(OC_EINVAL, "pool_status: null pool");
    oc::TenantPool* p = (oc::TenantPool*)h;
    std::lock_guard<std::mutex> lk(p->mu);
    if (ticket >= p->tenants.size()) return oc::fail(OC_ERANGE, "pool_status: unknown ticket");
    const oc::Tenant& t = p->tenants[ticket];
    if (state) *state = t.state;
    if (rate_Bps) *rate_Bps = t.rate;
    return OC_OK;
}

OC_API int oc_pool_destroy(oc_tenant_pool* h) {
    if (!h) return OC_OK;
    for (auto& eb : ((oc::TenantPool*)h)->batches) oc_batch_free(eb.batch);  // waits for its launch
    for (auto& t : ((oc::TenantPool*)h)->tenants) {
        if (t.done_stream) {
            cudaStreamSynchronize(t.done_stream);
            cudaStreamDestroy(t.done_stream);
        }
        if (t.layers_done) cudaEventDestroy(t.layers_done);
    }
    delete (oc::TenantPool*)h;
    return OC_OK;
}

}  // extern "C"
