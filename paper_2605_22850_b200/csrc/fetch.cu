// fetch_layerwise on B200: the storage server's layer aggregation (PAPER.md Alg. A1, P:2565-2581;
// Sec. 3.3) fused with the client's paged-KV placement, as sm_100a kernels.
//
// Alg. A1 for layer l appends RangeGet(H_j, lS, S) of every matched chunk j, in prefix order, to
// B_l, RDMA-writes B_l to the client buffer and notifies "layer ready".  Here no B_l is
// materialised: a work unit is R consecutive token rows of the K (or V) half of one chunk's layer-l
// slice -- contiguous in the chunk object (KV_L2TD) -- and it is copied straight to
// the rows' destination slots (block_table[u / Bs], slot u % Bs).  Every
// matched byte is read once and written once: 2*N*S HBM bytes per layer.
//
// Two copy engines:
//   BULK  one copy warp per CTA drives the TMA: one cp.async.bulk load per unit into a shared-
//         memory ring (mbarrier complete_tx), one bulk store per contiguous destination run.
//   LDST  256 threads per CTA, 16-byte vector loads (all of a round issued before any store).
//
// Completion (Alg. A1 line 7, "NotifyLayerReady"): producers add their finished units to the
// layer's counter with a release reduction (fire and forget); an observer -- thread 0 of CTA 0,
// which copies nothing -- walks the layers in order, acquires each counter once it reaches this
// fetch's target, stamps %globaltimer and stores `ready` = (epoch-1)*L + l + 1 with release
// semantics.  Consumers wait on `ready` with cuStreamWaitValue32 in the GPU front end (no host
// round trip, no kernel), so layer l's compute starts while layer l+1 is still in flight.  In
// PER_LAYER mode each layer is its own launch followed by a CUDA event.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "fetch_kernels.cuh"
#include "oc_internal.h"

namespace oc {

// ---- launch --------------------------------------------------------------------------------------------
namespace {

int occupancy(const void* fn, int threads, size_t smem) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) != cudaSuccess || occ < 1) {
        cudaGetLastError();
        occ = 1;
    }
    return occ;
}

bool force_wait_kernel() {
    const char* e = std::getenv("OC_WAIT_KERNEL");
    return e && e[0] == '1';
}

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e && *e ? std::atoi(e) : dflt;
}

bool env_flag(const char* name, bool dflt) { return env_int(name, dflt ? 1 : 0) != 0; }

// Default unit size (profiles/r01_engine_sweep.txt, r01_corun.json): with the whole GPU, 32 KiB
// units at 3 CTAs per SM reach the copy roofline; with a copy-CTA budget of at most one CTA per
// SM (co-running with prefill) 64 KiB units -- a whole chunk-layer slice at Llama layouts --
// halve the per-unit latency a single copy warp pays (0.85 vs 0.54 TB/s at 16 CTAs).
uint32_t default_unit_bytes(uint32_t max_ctas, int sms) {
    return (max_ctas && max_ctas <= (uint32_t)sms) ? 65536u : 32768u;
}

struct BulkPlan {
    uint32_t copy_ctas, stages, stage_bytes, smem;
};

// Shared-memory ring per CTA: `per_sm` CTAs share the SM's 228 KiB.  Measured on B200
// (profiles/): 3 CTAs per SM with 32 KiB units (2 stages each) reach the copy roofline.
BulkPlan plan_bulk(const DevDesc& dd, int sms, uint32_t max_ctas, uint64_t units) {
    BulkPlan p;
    p.stage_bytes = (uint32_t)(((uint64_t)dd.rows_per_unit * dd.row + 127) & ~127ull);
    int per_sm = std::max(1, env_int("OC_BULK_CTAS_PER_SM", 3));
    const uint32_t sm_bytes = 228 * 1024;
    while (true) {
        uint32_t per_cta = std::min<uint32_t>(sm_bytes / per_sm - 1024 - kBulkStaticSmem, 227 * 1024);
        uint32_t st = per_cta > 128 ? (per_cta - 128) / p.stage_bytes : 0;
        // at most 16: the ring's mbarriers live in the first 128 bytes of the dynamic shared memory
        st = std::min<uint32_t>(st, (uint32_t)std::min(16, std::max(2, env_int("OC_BULK_STAGES", 16))));
        if (st >= 2 || per_sm == 1) {
            p.stages = st >= 2 ? st : 0;  // 0: a unit does not fit twice in shared memory
            break;
        }
        per_sm /= 2;
    }
    p.smem = 128 + p.stages * p.stage_bytes;
    uint64_t grid = (uint64_t)per_sm * sms - 1;  // one CTA slot of the first wave is the observer's
    if (max_ctas) grid = std::min<uint64_t>(grid, max_ctas);
    p.copy_ctas = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(grid, units));
    return p;
}

// Paced launches keep a 2-unit ring: a CTA claims and loads its ring ahead of time, and the
// prologue (or a hold) waits for each claimed unit's release -- with a deep ring a CTA that
// claimed units across a release boundary would hold its earlier units' stores until the later
// release (a paced layer 0 seen ready only after layer 1's release time).
void shallow_ring(BulkPlan* p) {
    if (p->stages > 2) {
        p->stages = 2;
        p->smem = 128 + 2 * p->stage_bytes;
    }
}

// cudaFuncSetAttribute applies to the current device only, so the "already raised" cache is per
// device (a process may hold stores and fetches on several GPUs); racing threads at worst both set it.
constexpr int kMaxDevices = 64;

cudaError_t raise_smem_attr(const void* fn, std::atomic<uint32_t>* per_dev, uint32_t smem) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::atomic<uint32_t>* slot = dev >= 0 && dev < kMaxDevices ? &per_dev[dev] : nullptr;
    if (slot && smem <= slot->load(std::memory_order_acquire)) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<uint32_t>(smem, 48 * 1024));
    if (e == cudaSuccess && slot) {
        uint32_t cur = slot->load(std::memory_order_relaxed);
        while (cur < smem && !slot->compare_exchange_weak(cur, smem, std::memory_order_acq_rel)) {
        }
    }
    return e;
}

template <int MODE>
cudaError_t set_bulk_smem(uint32_t smem) {
    static std::atomic<uint32_t> attr_set[kMaxDevices];
    return raise_smem_attr((const void*)fetch_bulk_kernel<MODE>, attr_set, smem);
}

// Measurement support (OC_TRACE=1, oc_trace_read): one ramp-trace buffer per device.
std::mutex g_trace_mu;
uint64_t* g_trace_buf[kMaxDevices] = {};
uint64_t* g_trace_last = nullptr;

uint64_t* trace_buffer(int device, cudaStream_t s) {
    static const bool on = [] {
        const char* e = std::getenv("OC_TRACE");
        return e && e[0] == '1';
    }();
    if (!on || device < 0 || device >= kMaxDevices) return nullptr;
    std::lock_guard<std::mutex> lk(g_trace_mu);
    uint64_t*& b = g_trace_buf[device];
    const size_t bytes = (size_t)kTraceCtas * kTraceSlots * sizeof(uint64_t);
    if (!b && cudaMalloc((void**)&b, bytes) != cudaSuccess) {
        cudaGetLastError();
        b = nullptr;
        return nullptr;
    }
    if (cudaMemsetAsync(b, 0, bytes, s) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    g_trace_last = b;
    return b;
}

// One launch copies units [g0, g1); it claims them from the descriptor's counter starting at
// d->grab_ctr and advances that counter by (units + copy CTAs) -- see claim_unit.
// Copy CTA b takes unit g0 + b - 1 first (no claim), so the grid never exceeds the units; the
// counter then advances by exactly g1 - g0 (see the kernel's claim).  With `overlap`
// (OC_FETCH_OVERLAP) the launch is a programmatic dependent of the stream's previous kernel: it
// may start once that kernel's CTAs have made their last claims (griddepcontrol.launch_dependents)
// and it does not wait for that kernel's memory -- the caller guarantees independence.
int launch_bulk(Desc* d, const BulkPlan& p, uint32_t g0, uint32_t g1, cudaStream_t s, bool overlap = false) {
    if (p.stages < 2) return fail(OC_ENOTSUP, "bulk engine: two units do not fit in shared memory (use LDST)");
    if (p.copy_ctas == 0 || p.copy_ctas > g1 - g0) return fail(OC_EINVAL, "bulk engine: more copy CTAs than units");
    OC_CUDA(set_bulk_smem<kSingle>(p.smem));
    DevDesc dd = d->dd;
    dd.trace = trace_buffer(d->device, s);
    const uint32_t slot = d->launch_seq++ % kClaimSlots;
    dd.next_unit = d->dd.next_unit + slot * kClaimSlotStride;
    const uint32_t grab = d->grab_ctr[slot];
    static const uint32_t ramp = (env_int("OC_RAMP_STATIC2", 1) ? kRampStatic2 : 0u) |
                                 (env_int("OC_RAMP_FIRST_LAYER", 1) ? kRampFirstLayer : 0u);
    dd.ramp = ramp;
    const uint32_t extra = (ramp & kRampStatic2) ? ramp_extra(g0, g1, dd.units_per_layer, p.copy_ctas) : 0u;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.copy_ctas + 1);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = overlap ? attr : nullptr;
    cfg.numAttrs = overlap ? 1 : 0;
    OC_CUDA(cudaLaunchKernelEx(&cfg, fetch_bulk_kernel<kSingle>, dd, BatchArgs{}, g0, g1, grab, p.stages,
                               p.stage_bytes));
    d->grab_ctr[slot] += g1 - g0 - extra;  // counter claims: units past the static ones + one overshoot per CTA
    return OC_OK;
}

int launch_ldst(Desc* d, int sms, uint32_t max_ctas, uint32_t g0, uint32_t g1, cudaStream_t s,
                bool overlap = false) {
    // one CTA slot of the first wave is the observer's
    static int occ = occupancy((const void*)fetch_ldst_kernel, kThreads, 0);
    uint64_t grid = (uint64_t)occ * sms - 1;
    if (max_ctas) grid = std::min<uint64_t>(grid, max_ctas);
    grid = std::max<uint64_t>(1, std::min<uint64_t>(grid, g1 - g0));
    DevDesc dd = d->dd;
    const uint32_t slot = d->launch_seq++ % kClaimSlots;
    dd.next_unit = d->dd.next_unit + slot * kClaimSlotStride;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid + 1);
    cfg.blockDim = dim3(kThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = overlap ? attr : nullptr;
    cfg.numAttrs = overlap ? 1 : 0;
    OC_CUDA(cudaLaunchKernelEx(&cfg, fetch_ldst_kernel, dd, g0, g1, d->grab_ctr[slot]));
    d->grab_ctr[slot] += (g1 - g0) + (uint32_t)grid;
    return OC_OK;
}

}  // namespace

int launch_offload(const DevDesc& dd, const uint32_t* pos, int device, cudaStream_t s, bool host_dst) {
    const uint64_t total = (uint64_t)dd.units_per_layer * dd.L;
    if (total >= (1ull << 32)) return fail(OC_ERANGE, "put_from_paged: too many units");
    const char* eng = std::getenv("OC_OFFLOAD_ENGINE");
    if (!(eng && std::strcmp(eng, "ldst") == 0)) {
        // Writes into a pinned-host store cross PCIe: a few CTAs saturate it (as for host-tier fetches).
        const uint32_t cap = host_dst ? (uint32_t)std::max(1, env_int("OC_HOST_COPY_CTAS", 8)) : 0;
        const BulkPlan p = plan_bulk(dd, device_sm_count(device), cap, total);
        if (p.stages >= 2) {
            static std::atomic<uint32_t> attr_set[kMaxDevices];
            OC_CUDA(raise_smem_attr((const void*)offload_bulk_kernel, attr_set, p.smem));
            // no observer CTA here: the whole first wave copies
            const uint32_t grid = (uint32_t)std::min<uint64_t>(host_dst ? p.copy_ctas : p.copy_ctas + 1, total);
            offload_bulk_kernel<<<grid, 32, p.smem, s>>>(dd, pos, (uint32_t)total, p.stages, p.stage_bytes);
            OC_CUDA(cudaGetLastError());
            return OC_OK;
        }
    }
    static int occ = occupancy((const void*)offload_kernel, kThreads, 0);
    uint64_t grid = std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)occ * device_sm_count(device), total));
    if (host_dst) grid = std::min<uint64_t>(grid, (uint64_t)std::max(1, env_int("OC_HOST_COPY_CTAS", 8)));
    offload_kernel<<<(unsigned)grid, kThreads, 0, s>>>(dd, pos, (uint32_t)total);
    OC_CUDA(cudaGetLastError());
    return OC_OK;
}

// CE engine for pinned-host chunks: per layer, one strided copy-engine transfer per run of
// consecutive slots (width S, source pitch L*S) lands the layer's N slices contiguously in an HBM
// stage (double-buffered by layer), then the bulk kernel scatters the stage into the paged target
// and announces the layer.  The copy engine reads PCIe at ~55 GB/s where SM zero-copy reads stop
// at ~51 GB/s (profiles/r01_ce_probe.txt, r01_ce2d.txt); the scatter of layer l overlaps the copy
// of layer l+1 (copies on a private stream, events in both directions).
// A copy stream with its per-layer events; kits are recycled per (device, L) because creating a
// stream and 2L+1 events per request cost ~0.2 ms of host time per fetch.
struct CeKit {
    cudaStream_t stream = nullptr;
    cudaEvent_t start = nullptr;
    std::vector<cudaEvent_t> ce_done, scat_done;
};

namespace {
std::mutex g_kit_mu;
std::unordered_map<uint64_t, std::vector<CeKit*>> g_kits;

int ce_kit_get(int device, uint32_t L, CeKit** out) {
    const uint64_t key = ((uint64_t)(uint32_t)device << 32) | L;
    {
        std::lock_guard<std::mutex> lk(g_kit_mu);
        auto& v = g_kits[key];
        if (!v.empty()) {
            *out = v.back();
            v.pop_back();
            return OC_OK;
        }
    }
    auto k = std::make_unique<CeKit>();
    OC_CUDA(cudaStreamCreateWithFlags(&k->stream, cudaStreamNonBlocking));
    OC_CUDA(cudaEventCreateWithFlags(&k->start, cudaEventDisableTiming));
    k->ce_done.resize(L, nullptr);
    k->scat_done.resize(L, nullptr);
    for (uint32_t l = 0; l < L; l++) {
        OC_CUDA(cudaEventCreateWithFlags(&k->ce_done[l], cudaEventDisableTiming));
        OC_CUDA(cudaEventCreateWithFlags(&k->scat_done[l], cudaEventDisableTiming));
    }
    *out = k.release();
    return OC_OK;
}
}  // namespace

// wait_layer relay: a high-priority stream and one event per layer.  Creating them costs ~50 us of
// host time, so they are pooled per (device, L) like the CE kits.
struct RelayKit {
    cudaStream_t stream = nullptr;
    std::vector<cudaEvent_t> ev;
};

namespace {
std::mutex g_relay_mu;
std::unordered_map<uint64_t, std::vector<RelayKit*>> g_relays;

int relay_get(int device, uint32_t L, RelayKit** out) {
    const uint64_t key = ((uint64_t)(uint32_t)device << 32) | L;
    {
        std::lock_guard<std::mutex> lk(g_relay_mu);
        auto& v = g_relays[key];
        if (!v.empty()) {
            *out = v.back();
            v.pop_back();
            return OC_OK;
        }
    }
    auto k = std::make_unique<RelayKit>();
    int lo = 0, hi = 0;
    OC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    OC_CUDA(cudaStreamCreateWithPriority(&k->stream, cudaStreamNonBlocking, hi));
    k->ev.resize(L, nullptr);
    for (auto& e : k->ev) OC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    *out = k.release();
    return OC_OK;
}
}  // namespace

// PER_LAYER mode's per-layer events, pooled per (device, L) as well (a serving loop builds a
// descriptor per request; creating L events costs tens of us of host time).
namespace {
std::unordered_map<uint64_t, std::vector<std::vector<cudaEvent_t>>> g_layer_evs;  // under g_relay_mu
}  // namespace

int per_layer_events_get(int device, uint32_t L, std::vector<cudaEvent_t>* out) {
    {
        std::lock_guard<std::mutex> lk(g_relay_mu);
        auto& v = g_layer_evs[((uint64_t)(uint32_t)device << 32) | L];
        if (!v.empty()) {
            *out = std::move(v.back());
            v.pop_back();
            return OC_OK;
        }
    }
    out->assign(L, nullptr);
    for (auto& e : *out) OC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return OC_OK;
}

// Called by oc_desc_free after the descriptor's last fetch has completed (every recorded event is).
void per_layer_events_release(Desc* d) {
    if (d->events.empty()) return;
    std::lock_guard<std::mutex> lk(g_relay_mu);
    g_layer_evs[((uint64_t)(uint32_t)d->device << 32) | d->geo.L].push_back(std::move(d->events));
    d->events.clear();
}

// Called by oc_desc_free after the descriptor's last fetch has completed.  A relay still waiting
// (a consumer waited on a layer that was never announced) is not reused: it is destroyed, and the
// runtime releases it when its work ends.
void relay_release(Desc* d) {
    RelayKit* k = d->relay;
    d->relay = nullptr;
    if (!k) return;
    if (cudaStreamQuery(k->stream) == cudaSuccess) {
        std::lock_guard<std::mutex> lk(g_relay_mu);
        g_relays[((uint64_t)(uint32_t)d->device << 32) | d->geo.L].push_back(k);
        return;
    }
    cudaGetLastError();
    for (auto e : k->ev) cudaEventDestroy(e);
    cudaStreamDestroy(k->stream);
    delete k;
}

// Called by oc_desc_free after the descriptor's last fetch has completed.
void ce_release(Desc* d) {
    if (d->ce_kit) {
        std::lock_guard<std::mutex> lk(g_kit_mu);
        g_kits[((uint64_t)(uint32_t)d->device << 32) | d->geo.L].push_back(d->ce_kit);
        d->ce_kit = nullptr;
    }
    dev_pool_free(d->device, d->stage_mem, d->stage_class);
    d->stage_mem = nullptr;
}

int launch_fetch_ce(Desc* d, const oc_fetch_opts& o, cudaStream_t s) {
    if (o.mode != OC_FETCH_PERSISTENT) return fail(OC_ENOTSUP, "fetch_layerwise: the CE engine uses PERSISTENT mode");
    if (o.pace_Bps != 0) return fail(OC_ENOTSUP, "fetch_layerwise: the CE engine is unpaced");
    if (d->host_chunks != d->N || d->run_first.empty())
        return fail(OC_ENOTSUP, "fetch_layerwise: the CE engine needs every chunk in the pinned host tier");
    if (d->poisoned) return fail(OC_ECUDA, "fetch_layerwise: descriptor unusable after a failed launch");
    DeviceGuard dg(d->device);
    int urc = upload_order(&d->up, s);
    if (urc) return urc;
    const uint32_t L = d->geo.L;
    const uint64_t NS = d->N * d->geo.S;
    if (!d->done_ev) OC_CUDA(cudaEventCreateWithFlags(&d->done_ev, cudaEventDisableTiming));
    if (!d->ce_kit) {
        int krc = ce_kit_get(d->device, L, &d->ce_kit);
        if (krc) return krc;
    }
    CeKit& kit = *d->ce_kit;
    if (d->flat_base) {
        // FLAT target (the paper's client buffer): layer l of a run of consecutive slots is one
        // strided transfer straight into B_l = flat + l*N*S (chunk j at + j*S) -- no stage, no
        // scatter kernel; a one-thread kernel after each layer's copies announces it.
        uint32_t epoch = d->epoch + 1;
        if (epoch == 0) epoch = 1;
        d->dd.epoch = epoch;
        d->epoch = epoch;  // the unit counters are untouched: cnt_base stays
        d->poisoned = true;
        OC_CUDA(cudaEventRecord(kit.start, s));
        OC_CUDA(cudaStreamWaitEvent(kit.stream, kit.start, 0));
        stamp_kernel<<<1, 1, 0, kit.stream>>>(d->dd.ts);
        OC_CUDA(cudaGetLastError());
        for (uint32_t l = 0; l < L; l++) {
            uint8_t* dst = (uint8_t*)d->flat_base + (uint64_t)l * NS;
            const bool hot = l < d->hot_layers;  // from the HBM mirror (the run's store's pitch)
            for (size_t r = 0; r < d->run_first.size(); r++)
                OC_CUDA(cudaMemcpy2DAsync(dst + d->run_first[r] * d->geo.S, d->geo.S,
                                          (const void*)((hot ? d->run_hot[r] : d->run_src[r]) + (uint64_t)l * d->geo.S),
                                          hot ? d->run_hot_pitch[r] : d->geo.chunk, d->geo.S,
                                          d->run_len[r], cudaMemcpyDefault, kit.stream));
            announce_kernel<<<1, 1, 0, kit.stream>>>(d->dd.ts + 1 + l, d->dd.ready, d->dd.ready_host,
                                                     (epoch - 1u) * L + l + 1u);
            OC_CUDA(cudaGetLastError());
        }
        OC_CUDA(cudaEventRecord(kit.ce_done[L - 1], kit.stream));
        OC_CUDA(cudaStreamWaitEvent(s, kit.ce_done[L - 1], 0));  // the caller's stream sees the fetch end
        OC_CUDA(cudaEventRecord(d->done_ev, s));
        d->poisoned = false;
        d->last_mode = OC_FETCH_PERSISTENT;
        d->last_stream = s;
        d->fetched = true;
        return OC_OK;
    }
    if (!d->stage_mem) {
        d->stage_mem = dev_pool_alloc(d->device, 2 * NS, &d->stage_class);
        if (!d->stage_mem) return fail(OC_ENOMEM, "fetch_layerwise: CE stage allocation failed");
    }
    plan_units(d, o.unit_bytes ? o.unit_bytes : default_unit_bytes(o.max_ctas, device_sm_count(d->device)));
    DevDesc& dd = d->dd;
    const uint64_t total_units = (uint64_t)dd.units_per_layer * L;
    if (total_units >= (1ull << 32)) return fail(OC_ERANGE, "fetch_layerwise: too many units");
    uint32_t epoch = d->epoch + 1;
    if (epoch == 0) epoch = 1;
    dd.epoch = epoch;
    dd.cnt_target = d->cnt_base + dd.units_per_layer;
    dd.pace_ns = 0;
    dd.pace_ns_per_byte = 0.0;
    dd.staged = 1;
    dd.stage_base[0] = (uint64_t)d->stage_mem;
    dd.stage_base[1] = (uint64_t)d->stage_mem + NS;
    const BulkPlan p = plan_bulk(dd, device_sm_count(d->device), o.max_ctas, dd.units_per_layer);
    d->epoch = epoch;
    d->cnt_base = dd.cnt_target;
    d->poisoned = true;
    const uint32_t upl = dd.units_per_layer;
    OC_CUDA(cudaEventRecord(kit.start, s));  // the copies follow the caller's earlier work
    OC_CUDA(cudaStreamWaitEvent(kit.stream, kit.start, 0));
    stamp_kernel<<<1, 1, 0, kit.stream>>>(dd.ts);  // layer_times()[0] = the start of the copies
    OC_CUDA(cudaGetLastError());
    for (uint32_t l = 0; l < L; l++) {
        if (l >= 2) OC_CUDA(cudaStreamWaitEvent(kit.stream, kit.scat_done[l - 2], 0));  // stage l&1 free
        uint8_t* stage = (uint8_t*)d->stage_mem + (l & 1) * NS;
        const bool hot = l < d->hot_layers;  // from the HBM mirror (the run's store's pitch)
        for (size_t r = 0; r < d->run_first.size(); r++)
            OC_CUDA(cudaMemcpy2DAsync(stage + d->run_first[r] * d->geo.S, d->geo.S,
                                      (const void*)((hot ? d->run_hot[r] : d->run_src[r]) + (uint64_t)l * d->geo.S),
                                      hot ? d->run_hot_pitch[r] : d->geo.chunk, d->geo.S,
                                      d->run_len[r], cudaMemcpyDefault, kit.stream));
        OC_CUDA(cudaEventRecord(kit.ce_done[l], kit.stream));
        OC_CUDA(cudaStreamWaitEvent(s, kit.ce_done[l], 0));
        int rc = launch_bulk(d, p, l * upl, (l + 1) * upl, s);
        if (rc) return rc;
        OC_CUDA(cudaEventRecord(kit.scat_done[l], s));
    }
    OC_CUDA(cudaEventRecord(d->done_ev, s));
    d->poisoned = false;
    d->last_mode = OC_FETCH_PERSISTENT;
    d->last_stream = s;
    d->fetched = true;
    return OC_OK;
}

// The client half of the paper's unfused flow (Alg. A1 writes B_l into the client buffer, the
// client then copies it into its paged cache, iffalse): a layer-major payload
// [L][N][S] already in device memory is scattered into the descriptor's target by the bulk
// kernel, with the descriptor's per-layer completion.  2*N*S bytes per layer, like a fetch.
int launch_scatter_flat(Desc* d, uint64_t flat, uint64_t cap, const oc_fetch_opts& o, cudaStream_t s) {
    if (o.mode != OC_FETCH_PERSISTENT || o.pace_Bps != 0)
        return fail(OC_ENOTSUP, "scatter_flat: PERSISTENT mode, unpaced");
    if (cap < d->N * d->geo.L * d->geo.S) return fail(OC_ERANGE, "scatter_flat: flat payload smaller than N*L*S");
    if (flat % 16) return fail(OC_EALIGN, "scatter_flat: flat base not 16-byte aligned");
    if (d->poisoned) return fail(OC_ECUDA, "scatter_flat: descriptor unusable after a failed launch");
    if (d->range_open) return fail(OC_EINVAL, "scatter_flat: the previous fetch_layers fetch is incomplete");
    DeviceGuard dg(d->device);
    int urc = upload_order(&d->up, s);
    if (urc) return urc;
    if (!d->done_ev) OC_CUDA(cudaEventCreateWithFlags(&d->done_ev, cudaEventDisableTiming));
    plan_units(d, o.unit_bytes ? o.unit_bytes : default_unit_bytes(o.max_ctas, device_sm_count(d->device)));
    DevDesc& dd = d->dd;
    const uint64_t total_units = (uint64_t)dd.units_per_layer * dd.L;
    if (total_units >= (1ull << 32)) return fail(OC_ERANGE, "scatter_flat: too many units");
    uint32_t epoch = d->epoch + 1;
    if (epoch == 0) epoch = 1;
    dd.epoch = epoch;
    dd.cnt_target = d->cnt_base + dd.units_per_layer;
    dd.pace_ns = 0;
    dd.pace_ns_per_byte = 0.0;
    dd.staged = 2;
    dd.stage_base[0] = flat;
    d->epoch = epoch;
    d->cnt_base = dd.cnt_target;
    d->poisoned = true;
    const BulkPlan p = plan_bulk(dd, device_sm_count(d->device), o.max_ctas, total_units);
    int rc = launch_bulk(d, p, 0, (uint32_t)total_units, s);
    if (rc) return rc;
    OC_CUDA(cudaEventRecord(d->done_ev, s));
    d->poisoned = false;
    d->last_mode = OC_FETCH_PERSISTENT;
    d->last_stream = s;
    d->fetched = true;
    return OC_OK;
}

// oc_fetch_layers: the ranges of one fetch may be on different streams, so each records its own
// completion event, and the final range's stream waits for all of them before done_ev -- done_ev
// (which desc_free, layer_times and the next fetch rely on) then covers the whole fetch.
int record_range(Desc* d, cudaStream_t s, bool last) {
    if (d->n_ranges >= d->range_evs.size()) {
        cudaEvent_t ev = nullptr;
        OC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        d->range_evs.push_back(ev);
    }
    OC_CUDA(cudaEventRecord(d->range_evs[d->n_ranges++], s));
    if (last) {
        for (uint32_t k = 0; k + 1 < d->n_ranges; k++) OC_CUDA(cudaStreamWaitEvent(s, d->range_evs[k], 0));
        d->n_ranges = 0;
    }
    OC_CUDA(cudaEventRecord(d->done_ev, s));
    return OC_OK;
}

// Layers [l0, l1) of the descriptor's current fetch (oc_fetch_layers): l0 == 0 opens a new fetch
// like fetch_layerwise and launches only its first layers; l0 > 0 continues it where the previous
// call stopped.  One launch per call over the range's units, announced by its observer CTA.
int launch_fetch_range(Desc* d, const oc_fetch_opts& oin, uint32_t l0, uint32_t l1, cudaStream_t s) {
    const uint32_t L = d->geo.L;
    if (l0 >= l1 || l1 > L) return fail(OC_ERANGE, "fetch_layers: need l0 < l1 <= L");
    if (l0 == 0) return launch_fetch(d, oin, s, l1);
    if (!d->fetched || d->range_open != l0)
        return fail(OC_EINVAL, "fetch_layers: layers must follow the previous call's range (l0 = its l1)");
    oc_fetch_opts o = oin;
    if (o.engine == OC_COPY_AUTO) o.engine = d->dd.nhd ? OC_COPY_BULK : OC_COPY_LDST;
    if (o.mode != OC_FETCH_PERSISTENT || o.pace_Bps != 0 || (o.engine != OC_COPY_BULK && o.engine != OC_COPY_LDST))
        return fail(OC_ENOTSUP, "fetch_layers: PERSISTENT mode, BULK or LDST engine, unpaced");
    if (o.unit_bytes && o.unit_bytes != d->range_unit_bytes)
        return fail(OC_EINVAL, "fetch_layers: the unit size is fixed by the call with l0 = 0");
    if (d->poisoned) return fail(OC_ECUDA, "fetch_layers: descriptor unusable after a failed launch");
    DeviceGuard dg(d->device);
    int urc = upload_order(&d->up, s);  // the kernel reads the descriptor block
    if (urc) return urc;
    const int sms = device_sm_count(d->device);
    const uint32_t upl = d->dd.units_per_layer;
    d->poisoned = true;
    int rc;
    d->dd.wait_prev_layers = 1;  // this launch's copy of the descriptor (launches take it by value)
    if (o.engine == OC_COPY_BULK) {
        BulkPlan p = plan_bulk(d->dd, sms, o.max_ctas, (uint64_t)(l1 - l0) * upl);
        if (o.flags & OC_FETCH_LEAN) shallow_ring(&p);
        if (o.flags & OC_FETCH_YIELD) {  // one unit per CTA, as the yield launch's later layers
            p.copy_ctas = (l1 - l0) * upl;
            shallow_ring(&p);
        }
        rc = launch_bulk(d, p, l0 * upl, l1 * upl, s);
    } else {
        rc = launch_ldst(d, sms, o.max_ctas, l0 * upl, l1 * upl, s);
    }
    d->dd.wait_prev_layers = 0;
    if (rc) return rc;
    rc = record_range(d, s, l1 == L);
    if (rc) return rc;
    d->poisoned = false;
    d->range_open = l1 < L ? l1 : 0;
    d->last_stream = s;
    return OC_OK;
}

int launch_fetch(Desc* d, const oc_fetch_opts& oin, cudaStream_t s, uint32_t l_end) {
    oc_fetch_opts o = oin;
    if (d->range_open)
        return fail(OC_EINVAL, "fetch: the previous fetch_layers fetch is incomplete (fetch its remaining layers)");
    const bool ranged = l_end < d->geo.L;
    if (o.mode != OC_FETCH_PERSISTENT && o.mode != OC_FETCH_PER_LAYER)
        return fail(OC_EINVAL, "fetch_layerwise: unknown mode");
    if (ranged && (o.mode != OC_FETCH_PERSISTENT || o.pace_Bps != 0 || o.engine == OC_COPY_CE ||
                   (o.flags & (OC_FETCH_YIELD | OC_FETCH_FIRST_LAYER_FULL))))
        return fail(OC_ENOTSUP, "fetch_layers: PERSISTENT mode, BULK or LDST engine, unpaced");
    // AUTO: the TMA engine where destination rows are contiguous (NHD, flat); with a head-split
    // target (HND) every row becomes n_kv stores of d*p bytes, which holds the TMA engine to
    // 4.2 TB/s at 4K while 16-byte LD/ST streams at 6.3 (profiles/r01_hnd_probe.txt).  Strict
    // pacing exists only in the TMA engine.
    if (o.engine == OC_COPY_AUTO) {
        // A FLAT target fed from pinned host memory in a few slot runs: the copy engine writes
        // B_l directly (no stage, no SMs): 53.3 GB/s of PCIe reads at 1 run, 51.5 at 4, against
        // 51.4 for SM zero-copy reads (profiles/r01_flat_auto.txt); with many runs per layer its
        // per-transfer cost wins (45.6 GB/s at 16 runs; profiles/r01_ce2d.txt).
        // A PAGED target fed that way with large layers (>= 32 MiB: a 64K hit) too: one strided
        // transfer per layer into an HBM stage, then the scatter kernel -- 55.5 GB/s of PCIe reads
        // against 51.2 for zero-copy (config 3, profiles/r02_bench.json legs.config3), X0 4.9 vs
        // 5.3 ms; at 4K (14-16 MiB layers) the per-layer stage/scatter/announce steps cost more than
        // they gain (spin-window added TTFT 0.74 vs 0.59 ms), so zero-copy stays.
        const bool few_runs = !ranged && d->host_chunks == d->N && !d->run_first.empty() &&
                              d->run_first.size() <= 4 && o.pace_Bps == 0 && o.mode == OC_FETCH_PERSISTENT;
        const bool ce = few_runs && (d->flat_base || (d->hot_layers == 0 && d->N * d->geo.S >= (32ull << 20)));
        o.engine = ce ? OC_COPY_CE
                      : (d->dd.nhd || (o.pace_Bps > 0 && o.pace_strict)) ? OC_COPY_BULK : OC_COPY_LDST;
    }
    if (o.engine == OC_COPY_CE) return launch_fetch_ce(d, o, s);
    if (o.engine != OC_COPY_LDST && o.engine != OC_COPY_BULK) return fail(OC_EINVAL, "fetch_layerwise: unknown engine");
    d->dd.staged = 0;
    if (o.pace_Bps < 0) return fail(OC_EINVAL, "fetch_layerwise: pace must be >= 0");
    if (o.pace_Bps > 0 && o.mode != OC_FETCH_PERSISTENT)
        return fail(OC_ENOTSUP, "fetch_layerwise: pacing needs PERSISTENT mode");
    if (o.pace_Bps > 0 && o.pace_strict && o.engine != OC_COPY_BULK)
        return fail(OC_ENOTSUP, "fetch_layerwise: strict pacing needs the BULK engine");
    if (d->poisoned) return fail(OC_ECUDA, "fetch_layerwise: descriptor unusable after a failed launch");
    DeviceGuard dg(d->device);
    int urc = upload_order(&d->up, s);  // the kernel reads the descriptor block
    if (urc) return urc;
    if (!d->done_ev) OC_CUDA(cudaEventCreateWithFlags(&d->done_ev, cudaEventDisableTiming));
    if (o.mode == OC_FETCH_PER_LAYER && d->events.empty()) {
        int erc = per_layer_events_get(d->device, d->geo.L, &d->events);
        if (erc) return erc;
    }
    // PCIe-bound sources (pinned host tier) saturate the link from a handful of CTAs.  More CTAs
    // only lengthen the PCIe read queue, and every other GPU read of host memory -- the command
    // fetches of the consumer's stream -- waits behind it: 16 CTAs add ~30 us to each consumer
    // launch, 8 CTAs x 32 KiB units ~4 us at the same 51.4 GB/s; 6 CTAs lose bandwidth on large
    // slabs (profiles/r01_pcie_latency*.txt).
    const bool host_src = d->host_chunks * 2 > d->N;
    uint32_t max_ctas = o.max_ctas;
    if (!max_ctas && host_src) max_ctas = (uint32_t)std::max(1, env_int("OC_HOST_COPY_CTAS", 8));
    // PCIe-bound fetches keep 32 KiB units: finer units finish layer 0 sooner on a slow link.
    d->range_unit_bytes = o.unit_bytes ? o.unit_bytes : default_unit_bytes(host_src ? 0 : max_ctas, device_sm_count(d->device));
    plan_units(d, d->range_unit_bytes);
    DevDesc& dd = d->dd;
    const uint64_t total_units = (uint64_t)dd.units_per_layer * dd.L;
    if (total_units >= (1ull << 32)) return fail(OC_ERANGE, "fetch_layerwise: too many units");
    uint32_t epoch = d->epoch + 1;
    if (epoch == 0) epoch = 1;  // epochs count from 1: layer l of epoch e is ready at (e-1)*L + l + 1
    dd.epoch = epoch;
    dd.cnt_target = d->cnt_base + dd.units_per_layer;  // the unit size may change between fetches
    dd.pace_ns = o.pace_Bps > 0 && !o.pace_strict ? (uint64_t)((double)d->N * d->geo.S / o.pace_Bps * 1e9) : 0;
    dd.pace_ns_per_byte = o.pace_Bps > 0 && o.pace_strict ? 1e9 / o.pace_Bps : 0.0;
    const int sms = device_sm_count(d->device);
    // From the first launch on, the device counters belong to this epoch.
    d->epoch = epoch;
    d->cnt_base = dd.cnt_target;
    d->poisoned = true;
    const uint32_t upl = dd.units_per_layer;
    const bool paced = dd.pace_ns || dd.pace_ns_per_byte > 0.0;
    if (ranged) {
        BulkPlan p = plan_bulk(dd, sms, max_ctas, (uint64_t)l_end * upl);
        if (o.flags & OC_FETCH_LEAN) shallow_ring(&p);
        int rc = o.engine == OC_COPY_BULK ? launch_bulk(d, p, 0, l_end * upl, s)
                                          : launch_ldst(d, sms, max_ctas, 0, l_end * upl, s);
        if (rc) return rc;
    } else if (o.mode == OC_FETCH_PERSISTENT && dd.hot_layers && host_src && !paced) {
        // Hot layers mirrored in HBM: they go first with an HBM-sized grid (X0 at HBM speed), the
        // rest follows from host memory with the PCIe-sized grid; each launch announces its layers.
        const uint32_t k_units = std::min(dd.hot_layers, dd.L) * upl;
        const uint32_t ranges[2][2] = {{0, k_units}, {k_units, (uint32_t)total_units}};
        const uint32_t caps[2] = {o.max_ctas, max_ctas};
        for (int part = 0; part < 2; part++) {
            const uint32_t g0 = ranges[part][0], g1 = ranges[part][1];
            if (g1 <= g0) continue;
            int rc = o.engine == OC_COPY_BULK ? launch_bulk(d, plan_bulk(dd, sms, caps[part], g1 - g0), g0, g1, s)
                                              : launch_ldst(d, sms, caps[part], g0, g1, s);
            if (rc) return rc;
        }
    } else if (o.mode == OC_FETCH_PERSISTENT && (o.flags & OC_FETCH_YIELD) && o.engine == OC_COPY_BULK && !paced &&
               !host_src) {
        // Co-running with prefill: layer 0 with the whole GPU (persistent grid), then layers
        // 1..L-1 with one unit per CTA -- CTAs retire as they finish, so kernels of a higher-priority
        // stream take their SMs as soon as they are launched and the fetch fills what is left.
        int rc = launch_bulk(d, plan_bulk(dd, sms, 0, upl), 0, upl, s);
        if (rc) return rc;
        if (dd.L > 1) {
            BulkPlan p = plan_bulk(dd, sms, 0, (uint64_t)total_units - upl);
            p.copy_ctas = (uint32_t)(total_units - upl);
            shallow_ring(&p);  // one unit per CTA: the smallest ring (2 stages) is the smallest footprint
            // OC_YIELD_CTAS_PER_SM=k (measurement knob): pad the CTA's shared memory so that at most
            // k copy CTAs share an SM (less HBM pressure in the consumer's kernel tails)
            if (const int k = env_int("OC_YIELD_CTAS_PER_SM", 0); k > 0) {
                const uint32_t f = (228u * 1024u) / (uint32_t)k;  // per-CTA footprint: k fit, k + 1 do not
                const uint32_t dyn = std::min<uint32_t>(f - 1024u - kBulkStaticSmem, 227u * 1024u);
                p.smem = std::max(p.smem, dyn);
            }
            rc = launch_bulk(d, p, upl, (uint32_t)total_units, s);
            if (rc) return rc;
        }
    } else if (o.mode == OC_FETCH_PERSISTENT && (o.flags & OC_FETCH_FIRST_LAYER_FULL) && max_ctas && !paced &&
               dd.L > 1) {
        // Layer 0 with the whole GPU (its transfer is exposed before any compute can start), the
        // rest with the caller's copy-CTA budget (they only have to keep ahead of the compute).
        const uint32_t ranges[2][2] = {{0, upl}, {upl, (uint32_t)total_units}};
        const uint32_t caps[2] = {0, max_ctas};
        for (int part = 0; part < 2; part++) {
            const uint32_t g0 = ranges[part][0], g1 = ranges[part][1];
            int rc = o.engine == OC_COPY_BULK ? launch_bulk(d, plan_bulk(dd, sms, caps[part], g1 - g0), g0, g1, s)
                                              : launch_ldst(d, sms, caps[part], g0, g1, s);
            if (rc) return rc;
        }
    } else if (o.mode == OC_FETCH_PERSISTENT) {
        BulkPlan p = plan_bulk(dd, sms, max_ctas, total_units);
        if (paced || (o.flags & OC_FETCH_LEAN)) shallow_ring(&p);
        const bool overlap = (o.flags & OC_FETCH_OVERLAP) != 0;
        int rc = o.engine == OC_COPY_BULK ? launch_bulk(d, p, 0, (uint32_t)total_units, s, overlap)
                                          : launch_ldst(d, sms, max_ctas, 0, (uint32_t)total_units, s, overlap);
        if (rc) return rc;
    } else {
        // PER_LAYER: one launch + one CUDA event per layer.  The layers' launches are independent
        // (disjoint units, sources and destinations), so layer l+1's launch is a programmatic
        // dependent of layer l's and fills the SMs as layer l's CTAs drain; event l still records
        // the completion of layer l's launch.  Layer 0 follows the stream's earlier work unless the
        // caller set OC_FETCH_OVERLAP.
        // Default grid: 3/4 of the SMs' worth of copy CTAs per layer, so the CTAs of two to three
        // consecutive layers' launches are resident together -- the next layer's loads are in flight
        // while this layer's stores drain (profiles/r02_per_layer_sweep.json: 6.69 TB/s at 111 CTAs
        // vs 5.0 with a full grid per layer, 6.77 for the single persistent launch).
        const uint32_t pl_ctas = max_ctas ? max_ctas : std::max<uint32_t>(1, (uint32_t)sms * 3 / 4);
        const BulkPlan p = plan_bulk(dd, sms, pl_ctas, upl);
        // the layers' launches overlap, so each observer first waits for the earlier layers'
        // announcement: `ready` and the layer stamps stay in layer order
        dd.wait_prev_layers = 1;
        for (uint32_t l = 0; l < dd.L; l++) {
            const bool ov = l > 0 || (o.flags & OC_FETCH_OVERLAP);
            int rc = o.engine == OC_COPY_BULK ? launch_bulk(d, p, l * upl, (l + 1) * upl, s, ov)
                                              : launch_ldst(d, sms, max_ctas, l * upl, (l + 1) * upl, s, ov);
            if (rc) {
                dd.wait_prev_layers = 0;
                return rc;
            }
            OC_CUDA(cudaEventRecord(d->events[l], s));
        }
        dd.wait_prev_layers = 0;
    }
    if (ranged) {
        d->n_ranges = 0;
        int rrc = record_range(d, s, false);
        if (rrc) return rrc;
    } else {
        OC_CUDA(cudaEventRecord(d->done_ev, s));
    }
    d->poisoned = false;
    d->last_mode = o.mode;
    d->last_stream = s;
    d->fetched = true;
    d->range_open = ranged ? l_end : 0;
    return OC_OK;
}

// ---- batches --------------------------------------------------------------------------------------
struct Batch {
    std::vector<Desc*> descs;
    int device = 0;
    uint32_t n = 0;
    size_t upload_bytes = 0;   // DevDesc[n] | cum[n+1] | seg_cum[n+1] | seg_pos[n] | seg_cnt[n] | memb[n] (uint2)
    int order = OC_BATCH_BY_REQUEST;
    void* dev = nullptr;       // upload area + claim counter
    uint64_t dev_class = 0;
    void* stage = nullptr;     // pinned staging of the upload area
    uint64_t stage_class = 0;
    cudaEvent_t staged = nullptr;  // the last upload has finished reading `stage` (and `ent_stage`)
    uint32_t grab_ctr = 0;
    uint32_t* claim = nullptr;
    // WDRR claim table: [t0 slot (16 B)][entries], device block and pinned stage, grown on demand
    void* ent_dev = nullptr;
    uint64_t ent_dev_class = 0;
    void* ent_stage = nullptr;
    uint64_t ent_stage_class = 0;
    size_t ent_cap = 0;  // bytes of both blocks
};

// Grow the WDRR table blocks to `bytes`.  The old device block may still be read by this batch's
// previous launch, so it is released only after every member's last fetch has completed.
int ensure_ent_capacity(Batch* b, size_t bytes) {
    if (bytes <= b->ent_cap) return OC_OK;
    for (Desc* d : b->descs)
        if (d->fetched && d->done_ev) OC_CUDA(cudaEventSynchronize(d->done_ev));
    dev_pool_free(b->device, b->ent_dev, b->ent_dev_class);
    dev_pool_free(-1, b->ent_stage, b->ent_stage_class);
    b->ent_dev = dev_pool_alloc(b->device, bytes, &b->ent_dev_class);
    b->ent_stage = dev_pool_alloc(-1, bytes, &b->ent_stage_class);
    if (!b->ent_dev || !b->ent_stage) {
        dev_pool_free(b->device, b->ent_dev, b->ent_dev_class);
        dev_pool_free(-1, b->ent_stage, b->ent_stage_class);
        b->ent_dev = b->ent_stage = nullptr;
        b->ent_cap = 0;
        return fail(OC_ENOMEM, "fetch_batch_wdrr: claim table allocation failed");
    }
    b->ent_cap = bytes;
    return OC_OK;
}

int fetch_batch(Batch* b, const oc_fetch_opts& o, const oc_wdrr_opts* wdrr, cudaStream_t s) {
    if (o.mode != OC_FETCH_PERSISTENT) return fail(OC_ENOTSUP, "fetch_batch: batches use PERSISTENT mode");
    if (o.engine != OC_COPY_BULK && o.engine != OC_COPY_LDST && o.engine != OC_COPY_AUTO)
        return fail(OC_ENOTSUP, "fetch_batch: batches use the BULK or LDST engine");
    if (o.pace_Bps != 0)
        return fail(OC_ENOTSUP, "fetch_batch: pace_Bps is per request (fetch_layerwise); WDRR batches use hold_rates");
    for (Desc* d : b->descs) {
        if (d->poisoned) return fail(OC_ECUDA, "fetch_batch: a descriptor is unusable after a failed launch");
        if (d->range_open) return fail(OC_EINVAL, "fetch_batch: a member's fetch_layers fetch is incomplete");
    }
    DeviceGuard dg(b->device);
    OC_CUDA(cudaEventSynchronize(b->staged));  // previous upload done with the staging buffers
    DevDesc* st = (DevDesc*)b->stage;
    uint32_t* cum = (uint32_t*)((uint8_t*)b->stage + sizeof(DevDesc) * b->n);
    uint32_t* seg_cum = cum + (b->n + 1);
    uint32_t* seg_pos = seg_cum + (b->n + 1);
    uint32_t* seg_cnt = seg_pos + b->n;
    uint32_t* memb = seg_cnt + b->n;  // [n] x {member, units per layer}
    std::vector<uint32_t> sorted(b->n);
    uint64_t host_chunks = 0, chunks = 0, total = 0;
    cum[0] = 0;
    for (uint32_t i = 0; i < b->n; i++) {
        Desc* d = b->descs[i];
        int urc = upload_order(&d->up, s);  // the kernel reads every descriptor's block
        if (urc) return urc;
        if (!d->done_ev) OC_CUDA(cudaEventCreateWithFlags(&d->done_ev, cudaEventDisableTiming));
        plan_units(d, o.unit_bytes ? o.unit_bytes : default_unit_bytes(o.max_ctas, device_sm_count(b->device)));
        DevDesc& dd = d->dd;
        uint32_t epoch = d->epoch + 1;
        if (epoch == 0) epoch = 1;
        dd.epoch = epoch;
        dd.cnt_target = d->cnt_base + dd.units_per_layer;
        dd.pace_ns = 0;
        dd.pace_ns_per_byte = 0.0;
        dd.staged = 0;
        st[i] = dd;
        total += dd.units_per_layer;
        cum[i + 1] = (uint32_t)total;
        host_chunks += d->host_chunks;
        chunks += d->N;
    }
    const uint32_t L = b->descs[0]->geo.L;
    if (total * L >= (1ull << 32)) return fail(OC_ERANGE, "fetch_batch: too many units in one batch");
    // By position: members sorted by N descending; run k holds the positions where exactly
    // seg_cnt[k] members still have a chunk
    uint32_t nseg = 0;
    const bool by_pos = !wdrr && b->order == OC_BATCH_BY_POSITION;
    if (by_pos) {
        for (uint32_t i = 0; i < b->n; i++) sorted[i] = i;
        std::stable_sort(sorted.begin(), sorted.end(),
                         [&](uint32_t x, uint32_t y) { return b->descs[x]->N > b->descs[y]->N; });
        const uint32_t tiles = b->descs[0]->dd.tiles;
        seg_cum[0] = 0;
        for (uint32_t cnt = b->n; cnt >= 1; cnt--) {
            const uint64_t p0 = cnt == b->n ? 0 : b->descs[sorted[cnt]]->N;
            const uint64_t p1 = b->descs[sorted[cnt - 1]]->N;
            if (p1 <= p0) continue;
            seg_pos[nseg] = (uint32_t)p0;
            seg_cnt[nseg] = cnt;
            seg_cum[nseg + 1] = seg_cum[nseg] + (uint32_t)((p1 - p0) * cnt * tiles);
            nseg++;
        }
        for (Desc* d : b->descs)
            if (d->dd.tiles != tiles) return fail(OC_EINVAL, "fetch_batch: members planned with different units");
        for (uint32_t i = 0; i < b->n; i++) {  // units_per_layer was set by plan_units above
            memb[2 * i] = sorted[i];
            memb[2 * i + 1] = b->descs[sorted[i]]->dd.units_per_layer;
        }
    }
    // WDRR: the claim order (Alg. A2 line 7), uploaded behind a zeroed start-time slot
    // claim items of the launch: units, WDRR entries, or by-position claims of pos_claim units
    const uint32_t pos_claim = by_pos ? (uint32_t)std::max(1, env_int("OC_BYPOS_CLAIM", 8)) : 1u;
    uint64_t n_claims = (total * L + pos_claim - 1) / pos_claim;
    if (wdrr) {
        const DevDesc& d0 = b->descs[0]->dd;
        std::vector<uint64_t> n_units(b->n);
        for (uint32_t i = 0; i < b->n; i++) {
            if (b->descs[i]->dd.tiles != d0.tiles || b->descs[i]->dd.rows_per_unit != d0.rows_per_unit)
                return fail(OC_EINVAL, "fetch_batch_wdrr: members planned with different units");
            n_units[i] = (uint64_t)b->descs[i]->dd.units_per_layer * L;
        }
        std::vector<uint32_t> tile_bytes(d0.tiles);
        for (uint32_t t = 0; t < d0.tiles; t++)
            tile_bytes[t] = (uint32_t)(std::min(d0.rows_per_unit, 2 * d0.G - t * d0.rows_per_unit) * d0.row);
        // layers a member reads from the store's HBM mirror are not paced (reading c24)
        std::vector<uint64_t> free_units(b->n);
        oc_wdrr_opts wo = *wdrr;
        if (!wo.free_units) {
            for (uint32_t i = 0; i < b->n; i++)
                free_units[i] = (uint64_t)b->descs[i]->dd.units_per_layer * b->descs[i]->dd.hot_layers;
            wo.free_units = free_units.data();
        }
        std::vector<WdrrEntry> ents;
        int rc = wdrr_plan(n_units.data(), b->n, tile_bytes.data(), d0.tiles, wo, &ents);
        if (rc) return rc;
        rc = ensure_ent_capacity(b, 16 + ents.size() * sizeof(WdrrEntry));
        if (rc) return rc;
        std::memset(b->ent_stage, 0, 16);
        std::memcpy((uint8_t*)b->ent_stage + 16, ents.data(), ents.size() * sizeof(WdrrEntry));
        OC_CUDA(cudaMemcpyAsync(b->ent_dev, b->ent_stage, 16 + ents.size() * sizeof(WdrrEntry),
                                cudaMemcpyHostToDevice, s));
        n_claims = ents.size();
    }
    uint32_t max_ctas = o.max_ctas;
    if (!max_ctas && host_chunks * 2 > chunks) max_ctas = (uint32_t)std::max(1, env_int("OC_HOST_COPY_CTAS", 8));
    const int sms = device_sm_count(b->device);
    BulkPlan p = plan_bulk(b->descs[0]->dd, sms, max_ctas, n_claims);
    if (wdrr && wdrr->hold_rates) shallow_ring(&p);
    OC_CUDA(cudaMemcpyAsync(b->dev, b->stage, b->upload_bytes, cudaMemcpyHostToDevice, s));
    OC_CUDA(cudaEventRecord(b->staged, s));
    for (Desc* d : b->descs) {  // from the launch on, the device counters belong to the new epoch
        d->epoch = d->dd.epoch;
        d->cnt_base = d->dd.cnt_target;
        d->poisoned = true;
    }
    BatchArgs ba;
    ba.descs = (const DevDesc*)b->dev;
    ba.cum = (const uint32_t*)((uint8_t*)b->dev + sizeof(DevDesc) * b->n);
    ba.claim = b->claim;
    ba.n = b->n;
    ba.upl_total = (uint32_t)total;
    ba.div_upl_total = make_fastdiv((uint32_t)total);
    ba.ents = wdrr ? (const uint4*)((uint8_t*)b->ent_dev + 16) : nullptr;
    ba.t0_slot = wdrr ? (unsigned long long*)b->ent_dev : nullptr;
    ba.paced = wdrr && wdrr->hold_rates ? 1u : 0u;
    {
        const uint32_t* dcum = ba.cum + (b->n + 1);
        ba.seg_cum = dcum;
        ba.seg_pos = dcum + (b->n + 1);
        ba.seg_cnt = ba.seg_pos + b->n;
        ba.memb = (const uint2*)(ba.seg_cnt + b->n);
        ba.nseg = nseg;
        ba.tiles = b->descs[0]->dd.tiles;
        // B = ~4 MiB of one request's slices per block (profiles/r01_batch_dram.json)
        const uint64_t blk_bytes = (uint64_t)std::max(1, env_int("OC_BYPOS_BLOCK_KIB", 4096)) << 10;
        ba.pos_block = (uint32_t)std::max<uint64_t>(1, blk_bytes / b->descs[0]->geo.S);
        ba.pos_claim = pos_claim;
        ba.n_units = (uint32_t)(total * L);
    }
    // AUTO: the LD/ST engine as soon as one member's target is head-split (see launch_fetch)
    bool ldst = o.engine == OC_COPY_LDST;
    if (o.engine == OC_COPY_AUTO)
        for (Desc* d : b->descs) ldst |= !d->dd.nhd;
    if (ldst) {
        static int occ = occupancy((const void*)fetch_ldst_batch_kernel<kBatch>, kThreads, 0);
        uint64_t grid = (uint64_t)occ * sms - 1;  // one CTA slot of the first wave is the observer's
        if (max_ctas) grid = std::min<uint64_t>(grid, max_ctas);
        grid = std::max<uint64_t>(1, std::min<uint64_t>(grid, n_claims));
        const unsigned gb = (unsigned)grid + 1;
        if (wdrr) fetch_ldst_batch_kernel<kWdrr><<<gb, kThreads, 0, s>>>(ba, 0u, (uint32_t)n_claims, b->grab_ctr);
        else if (by_pos) fetch_ldst_batch_kernel<kByPos><<<gb, kThreads, 0, s>>>(ba, 0u, (uint32_t)n_claims, b->grab_ctr);
        else fetch_ldst_batch_kernel<kBatch><<<gb, kThreads, 0, s>>>(ba, 0u, (uint32_t)n_claims, b->grab_ctr);
        OC_CUDA(cudaGetLastError());
        b->grab_ctr += (uint32_t)n_claims + (uint32_t)grid;
    } else {
        if (p.stages < 2) return fail(OC_ENOTSUP, "fetch_batch: two units do not fit in shared memory");
        if (wdrr) {
            OC_CUDA(set_bulk_smem<kWdrr>(p.smem));
            fetch_bulk_kernel<kWdrr><<<p.copy_ctas + 1, 64, p.smem, s>>>(DevDesc{}, ba, 0u, (uint32_t)n_claims,
                                                                         b->grab_ctr, p.stages, p.stage_bytes);
        } else if (by_pos) {
            OC_CUDA(set_bulk_smem<kByPos>(p.smem));
            fetch_bulk_kernel<kByPos><<<p.copy_ctas + 1, 64, p.smem, s>>>(DevDesc{}, ba, 0u, (uint32_t)n_claims,
                                                                          b->grab_ctr, p.stages, p.stage_bytes);
        } else {
            OC_CUDA(set_bulk_smem<kBatch>(p.smem));
            fetch_bulk_kernel<kBatch><<<p.copy_ctas + 1, 64, p.smem, s>>>(DevDesc{}, ba, 0u, (uint32_t)n_claims,
                                                                          b->grab_ctr, p.stages, p.stage_bytes);
        }
        OC_CUDA(cudaGetLastError());
        b->grab_ctr += (uint32_t)n_claims + p.copy_ctas;
    }
    for (Desc* d : b->descs) {
        OC_CUDA(cudaEventRecord(d->done_ev, s));
        d->poisoned = false;
        d->last_mode = OC_FETCH_PERSISTENT;
        d->last_stream = s;
        d->fetched = true;
    }
    return OC_OK;
}

}  // namespace oc

using oc::Desc;

extern "C" {

OC_API int oc_fetch_layerwise(oc_desc* h, const oc_fetch_opts* opts, void* stream) {
    if (!h) return oc::fail(OC_EINVAL, "fetch_layerwise: null descriptor");
    oc_fetch_opts o{};
    o.mode = OC_FETCH_PERSISTENT;
    o.engine = OC_COPY_AUTO;
    if (opts) o = *opts;
    return oc::launch_fetch((Desc*)h, o, (cudaStream_t)stream);
}

OC_API int oc_fetch_layers(oc_desc* h, uint32_t l0, uint32_t l1, const oc_fetch_opts* opts, void* stream) {
    if (!h) return oc::fail(OC_EINVAL, "fetch_layers: null descriptor");
    oc_fetch_opts o{};
    o.mode = OC_FETCH_PERSISTENT;
    o.engine = OC_COPY_AUTO;
    if (opts) o = *opts;
    return oc::launch_fetch_range((Desc*)h, o, l0, l1, (cudaStream_t)stream);
}

OC_API int oc_batch_create(oc_desc* const* descs, uint32_t n, oc_batch** out) {
    if (!out || !descs || n == 0) return oc::fail(OC_EINVAL, "batch_create: need n >= 1 descriptors");
    *out = nullptr;
    auto b = std::make_unique<oc::Batch>();
    for (uint32_t i = 0; i < n; i++) {
        Desc* d = (Desc*)descs[i];
        if (!d) return oc::fail(OC_EINVAL, "batch_create: null descriptor");
        if (!oc::same_layout(d->layout, ((Desc*)descs[0])->layout) || d->device != ((Desc*)descs[0])->device)
            return oc::fail(OC_EINVAL, "batch_create: descriptors must share layout and device");
        for (uint32_t k = 0; k < i; k++)
            if (descs[k] == descs[i]) return oc::fail(OC_EINVAL, "batch_create: duplicate descriptor");
        b->descs.push_back(d);
    }
    b->n = n;
    b->device = b->descs[0]->device;
    b->upload_bytes = sizeof(oc::DevDesc) * n + 4 * (n + 1) * 2 + 4 * n * 4;
    const size_t dev_bytes = ((b->upload_bytes + 15) & ~size_t(15)) + 16;
    oc::DeviceGuard dg(b->device);
    b->dev = oc::dev_pool_alloc(b->device, dev_bytes, &b->dev_class);
    b->stage = oc::dev_pool_alloc(-1, b->upload_bytes, &b->stage_class);
    if (!b->dev || !b->stage) {
        oc::dev_pool_free(b->device, b->dev, b->dev_class);
        oc::dev_pool_free(-1, b->stage, b->stage_class);
        return oc::fail(OC_ENOMEM, "batch_create: allocation failed");
    }
    b->claim = (uint32_t*)((uint8_t*)b->dev + ((b->upload_bytes + 15) & ~size_t(15)));
    {  // zero the (possibly recycled) claim counter before any stream can launch on it
        cudaStream_t us = oc::upload_stream(b->device);
        if (!us) return oc::fail(OC_ECUDA, "batch_create: no upload stream");
        OC_CUDA(cudaMemsetAsync(b->claim, 0, 16, us));
        OC_CUDA(cudaStreamSynchronize(us));
    }
    OC_CUDA(cudaEventCreateWithFlags(&b->staged, cudaEventDisableTiming));
    *out = (oc_batch*)b.release();
    return OC_OK;
}

OC_API int oc_fetch_batch(oc_batch* h, const oc_fetch_opts* opts, void* stream) {
    if (!h) return oc::fail(OC_EINVAL, "fetch_batch: null batch");
    oc_fetch_opts o{};
    o.mode = OC_FETCH_PERSISTENT;
    o.engine = OC_COPY_BULK;
    if (opts) o = *opts;
    return oc::fetch_batch((oc::Batch*)h, o, nullptr, (cudaStream_t)stream);
}

OC_API int oc_scatter_flat(oc_desc* h, uint64_t flat_base, uint64_t flat_capacity, const oc_fetch_opts* opts,
                           void* stream) {
    if (!h) return oc::fail(OC_EINVAL, "scatter_flat: null descriptor");
    oc_fetch_opts o{};
    o.mode = OC_FETCH_PERSISTENT;
    o.engine = OC_COPY_BULK;
    if (opts) o = *opts;
    return oc::launch_scatter_flat((Desc*)h, flat_base, flat_capacity, o, (cudaStream_t)stream);
}

OC_API int oc_batch_set_order(oc_batch* h, int order) {
    if (!h) return oc::fail(OC_EINVAL, "batch_set_order: null batch");
    if (order != OC_BATCH_BY_REQUEST && order != OC_BATCH_BY_POSITION)
        return oc::fail(OC_EINVAL, "batch_set_order: unknown order");
    ((oc::Batch*)h)->order = order;
    return OC_OK;
}

OC_API int oc_fetch_batch_wdrr(oc_batch* h, const oc_fetch_opts* opts, const oc_wdrr_opts* wdrr, void* stream) {
    if (!h || !wdrr) return oc::fail(OC_EINVAL, "fetch_batch_wdrr: null pointer");
    oc_fetch_opts o{};
    o.mode = OC_FETCH_PERSISTENT;
    o.engine = OC_COPY_BULK;
    if (opts) o = *opts;
    return oc::fetch_batch((oc::Batch*)h, o, wdrr, (cudaStream_t)stream);
}

OC_API int oc_batch_free(oc_batch* h) {
    if (!h) return OC_OK;
    oc::Batch* b = (oc::Batch*)h;
    {
        oc::DeviceGuard dg(b->device);
        for (Desc* d : b->descs)  // the batch's device copy is read until its launches finish
            if (d->fetched && d->done_ev) cudaEventSynchronize(d->done_ev);
        if (b->staged) {
            cudaEventSynchronize(b->staged);
            cudaEventDestroy(b->staged);
        }
        oc::dev_pool_free(b->device, b->dev, b->dev_class);
        oc::dev_pool_free(-1, b->stage, b->stage_class);
        oc::dev_pool_free(b->device, b->ent_dev, b->ent_dev_class);
        oc::dev_pool_free(-1, b->ent_stage, b->ent_stage_class);
        cudaGetLastError();
    }
    delete b;
    return OC_OK;
}

OC_API int oc_wait_layer(oc_desc* h, uint32_t layer, void* stream) {
    if (!h) return oc::fail(OC_EINVAL, "wait_layer: null descriptor");
    Desc* d = (Desc*)h;
    if (layer >= d->geo.L) return oc::fail(OC_ERANGE, "wait_layer: layer >= L");
    if (!d->fetched) return oc::fail(OC_EINVAL, "wait_layer: no fetch has been issued");
    const uint32_t L = d->geo.L;
    const uint32_t want_layer = d->delivery == OC_DELIVER_CHUNK_MAJOR ? L - 1 : layer;
    oc::DeviceGuard dg(d->device);
    cudaStream_t s = (cudaStream_t)stream;
    if (d->last_mode == OC_FETCH_PER_LAYER) {
        OC_CUDA(cudaStreamWaitEvent(s, d->events[want_layer], 0));
        return OC_OK;
    }
    const uint32_t target = (d->epoch - 1u) * L + want_layer + 1u;
    // Already announced (the host mirror is written after the device word, once the layer's bytes
    // are in device memory): nothing needs to be enqueued -- a stream wait costs the consumer
    // 1-4 us of launch pipelining even when its condition already holds.
    if (d->ready_host && (int32_t)(__atomic_load_n(d->ready_host, __ATOMIC_ACQUIRE) - target) >= 0) return OC_OK;
    // The default wait is a one-thread kernel on the consumer stream that spins on the ready word:
    // it holds one CTA slot, never the stream's hardware queue.  A stream value wait
    // (cuStreamWaitValue32) stalls the hardware queue its stream is mapped to, and streams share
    // queues (CUDA_DEVICE_MAX_CONNECTIONS, 8 by default): a producer stream mapped behind a blocked
    // consumer waits too.  Measured (profiles/r02_wait_queue_hazard.json): the headline's next fetch
    // queued behind the consumer's wait for the previous one (overlap lost, 6.31 instead of 6.72 TB/s
    // with one connection, and once with the default 8); with relay streams (value wait on a
    // per-descriptor relay stream + event) workload C's requests all ended after the largest one
    // (2.4-4.2x Eq. 3 instead of 1.00; profiles/r02_sched_relay_hazard.json).
    // OC_WAIT_VALUE=1: the value wait on the consumer stream (2.3 us of consumer-stream time per
    // wait); OC_WAIT_RELAY=1: the relay (0.7 us; profiles/r02_wait_kinds.txt).  Both opt-in.
    const bool relay_on = oc::env_flag("OC_WAIT_RELAY", false);
    const bool value_on = oc::env_flag("OC_WAIT_VALUE", false);
    if (relay_on && !oc::force_wait_kernel()) {
        std::lock_guard<std::mutex> lk(d->relay_mu);
        if (!d->relay) {
            int krc = oc::relay_get(d->device, L, &d->relay);
            if (krc) return krc;
        }
        cudaStream_t rs = d->relay->stream;
        int urc = oc::upload_order(&d->up, rs);  // the ready word lives in the uploaded block
        if (urc) return urc;
        int rc = oc::stream_wait_geq(rs, d->dd.ready, target);
        if (rc == OC_OK) {
            OC_CUDA(cudaEventRecord(d->relay->ev[want_layer], rs));
            OC_CUDA(cudaStreamWaitEvent(s, d->relay->ev[want_layer], 0));
            return OC_OK;
        }
    }
    int urc = oc::upload_order(&d->up, s);  // the ready word lives in the uploaded block
    if (urc) return urc;
    if (value_on && !oc::force_wait_kernel()) {
        int rc = oc::stream_wait_geq(s, d->dd.ready, target);
        if (rc == OC_OK) return OC_OK;
    }
    oc::wait_geq_kernel<<<1, 1, 0, s>>>(d->dd.ready, target);
    OC_CUDA(cudaGetLastError());
    return OC_OK;
}

OC_API int oc_sync_layer(oc_desc* h, uint32_t layer) {
    if (!h) return oc::fail(OC_EINVAL, "sync_layer: null descriptor");
    Desc* d = (Desc*)h;
    if (layer >= d->geo.L) return oc::fail(OC_ERANGE, "sync_layer: layer >= L");
    if (!d->fetched) return oc::fail(OC_EINVAL, "sync_layer: no fetch has been issued");
    oc::DeviceGuard dg(d->device);
    const uint32_t want_layer = d->delivery == OC_DELIVER_CHUNK_MAJOR ? d->geo.L - 1 : layer;
    if (d->last_mode == OC_FETCH_PER_LAYER) {
        OC_CUDA(cudaEventSynchronize(d->events[want_layer]));
        return OC_OK;
    }
    // Persistent mode: already announced per the host mirror, else a private stream waits on the
    // ready word and the host blocks on an event after it.
    const uint32_t target = (d->epoch - 1u) * d->geo.L + want_layer + 1u;
    if (d->ready_host && (int32_t)(__atomic_load_n(d->ready_host, __ATOMIC_ACQUIRE) - target) >= 0) return OC_OK;
    if (!d->sync_stream) OC_CUDA(cudaStreamCreateWithFlags(&d->sync_stream, cudaStreamNonBlocking));
    if (!d->sync_ev) OC_CUDA(cudaEventCreateWithFlags(&d->sync_ev, cudaEventDisableTiming | cudaEventBlockingSync));
    int rc = oc_wait_layer(h, layer, d->sync_stream);
    if (rc) return rc;
    OC_CUDA(cudaEventRecord(d->sync_ev, d->sync_stream));
    OC_CUDA(cudaEventSynchronize(d->sync_ev));
    return OC_OK;
}

OC_API int oc_layers_ready(oc_desc* h, uint32_t* n) {
    if (!h || !n) return oc::fail(OC_EINVAL, "layers_ready: null pointer");
    Desc* d = (Desc*)h;
    if (!d->fetched) return oc::fail(OC_EINVAL, "layers_ready: no fetch has been issued");
    const uint32_t L = d->geo.L;
    uint32_t k = 0;
    if (d->last_mode == OC_FETCH_PER_LAYER) {
        oc::DeviceGuard dg(d->device);
        while (k < L && cudaEventQuery(d->events[k]) == cudaSuccess) k++;
        cudaGetLastError();
    } else {
        if (!d->ready_host) return oc::fail(OC_ENOTSUP, "layers_ready: descriptor has no host mirror");
        const int32_t a = (int32_t)(__atomic_load_n(d->ready_host, __ATOMIC_ACQUIRE) - (d->epoch - 1u) * L);
        k = a <= 0 ? 0u : std::min<uint32_t>((uint32_t)a, L);
    }
    if (d->delivery == OC_DELIVER_CHUNK_MAJOR && k < L) k = 0;
    *n = k;
    return OC_OK;
}

OC_API int oc_layer_times(oc_desc* h, uint64_t* out) {
    if (!h || !out) return oc::fail(OC_EINVAL, "layer_times: null pointer");
    Desc* d = (Desc*)h;
    if (!d->fetched) return oc::fail(OC_EINVAL, "layer_times: no fetch has been issued");
    oc::DeviceGuard dg(d->device);
    OC_CUDA(cudaEventSynchronize(d->done_ev));
    OC_CUDA(cudaMemcpy(out, d->dd.ts, (d->geo.L + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return OC_OK;
}

OC_API int oc_layer_times_async(oc_desc* h, uint64_t* out, void* stream) {
    if (!h || !out) return oc::fail(OC_EINVAL, "layer_times_async: null pointer");
    Desc* d = (Desc*)h;
    if (!d->fetched) return oc::fail(OC_EINVAL, "layer_times_async: no fetch has been issued");
    oc::DeviceGuard dg(d->device);
    cudaStream_t s = (cudaStream_t)stream;
    OC_CUDA(cudaStreamWaitEvent(s, d->done_ev, 0));
    OC_CUDA(cudaMemcpyAsync(out, d->dd.ts, (d->geo.L + 1) * sizeof(uint64_t), cudaMemcpyDefault, s));
    return OC_OK;
}

OC_API int oc_trace_read(uint64_t* out, uint64_t n) {
    if (!out) return oc::fail(OC_EINVAL, "trace_read: null out");
    std::lock_guard<std::mutex> lk(oc::g_trace_mu);
    if (!oc::g_trace_last) return oc::fail(OC_EINVAL, "trace_read: no traced launch (set OC_TRACE=1)");
    OC_CUDA(cudaDeviceSynchronize());
    const uint64_t m = std::min<uint64_t>(n, (uint64_t)oc::kTraceCtas * oc::kTraceSlots);
    OC_CUDA(cudaMemcpy(out, oc::g_trace_last, m * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return OC_OK;
}

OC_API int oc_emulate_compute(uint64_t ns, uint64_t* stamps, void* stream) {
    if (ns > 60ull * 1000000000ull) return oc::fail(OC_ERANGE, "emulate_compute: window > 60 s");
    if (stamps && ((uintptr_t)stamps & 7)) return oc::fail(OC_EALIGN, "emulate_compute: stamps not 8-byte aligned");
    oc::emulate_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(ns, stamps);
    OC_CUDA(cudaGetLastError());
    return OC_OK;
}

}  // extern "C"
