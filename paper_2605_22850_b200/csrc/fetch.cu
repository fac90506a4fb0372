// fetch_layerwise on B200: the storage server's layer aggregation (PAPER.md Alg. A1, P:2565-2581;
// Sec. 3.3) fused with the client's paged-KV placement, as one sm_100a kernel.
//
// Alg. A1 for layer l appends RangeGet(H_j, lS, S) for every matched chunk j in prefix order to
// B_l, RDMA-writes B_l to the client buffer and notifies "layer ready".  Here no B_l is
// materialised: each CTA copies one unit -- R consecutive token rows of the K (or V) half of one
// chunk's layer-l slice, contiguous in the chunk object -- straight to the rows' destination
// slots (block_table[u / Bs], slot u % Bs), with 16-byte vector loads
// and stores, all loads of a round issued before any store.  Every HBM byte of the matched
// prefix is read once and written once (2*N*S bytes per layer).
//
// Completion (Alg. A1 line 7, "NotifyLayerReady"): after each unit the CTA bumps the layer's
// unit counter; the CTA that completes a layer marks it done, and whichever CTA finds layers
// 0..l all done advances the monotone `ready` word past l (so layers are announced strictly in
// order), stamps %globaltimer and mirrors the epoch into pinned host memory.  Consumers wait on
// `ready` with cuStreamWaitValue32 (no host round trip) or, in PER_LAYER mode, on a CUDA event
// recorded after the layer's own launch.
#include <algorithm>
#include <cstdlib>

#include "oc_internal.h"

namespace oc {

constexpr int kThreads = 256;   // threads per CTA
constexpr int kVec = 8;         // 16-byte vectors in flight per thread per round
constexpr int kMaxRows = 1024;  // rows per unit (plan_units caps R)

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ void st_global(uint64_t addr, const uint4& v) {
    asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Copy one unit: rows [r0, r0 + nrows) of matrix kv of chunk j at `layer`.
__device__ __forceinline__ void copy_unit(const DevDesc& d, uint32_t layer, uint32_t unit, uint64_t* s_dst) {
    const uint32_t j = fdiv(unit, d.div_units_per_chunk);
    const uint32_t rem = unit - j * 2u * d.tiles;
    const uint32_t kv = rem >= d.tiles ? 1u : 0u;
    const uint32_t tile = rem - kv * d.tiles;
    const uint32_t r0 = tile * d.rows_per_unit;
    const uint32_t nrows = min(d.rows_per_unit, d.G - r0);
    // KV_L2TD: layer l of chunk j at [lS, (l+1)S); K rows then V rows, row-major (reading c2).
    const uint8_t* src = (const uint8_t*)d.src[j] + (uint64_t)layer * d.S + ((uint64_t)kv * d.G + r0) * d.row;
    const uint64_t base = kv ? d.v_base[layer] : d.k_base[layer];
    const uint32_t u0 = d.first_token + j * d.G + r0;  // request token of row r0
    for (uint32_t r = threadIdx.x; r < nrows; r += kThreads) {
        const uint32_t u = u0 + r;
        const uint32_t b = fdiv(u, d.div_Bs);
        const uint32_t slot = u - b * d.Bs;
        s_dst[r] = base + (uint64_t)d.bt[b] * d.block_stride + (uint64_t)slot * d.token_stride;
    }
    __syncthreads();
    const uint32_t nvec = nrows * d.vpr;
    for (uint32_t v0 = 0; v0 < nvec; v0 += kThreads * kVec) {
        uint4 buf[kVec];
#pragma unroll
        for (int k = 0; k < kVec; k++) {
            const uint32_t v = v0 + threadIdx.x + k * kThreads;
            if (v < nvec) buf[k] = ld_stream(src + (uint64_t)v * 16);
        }
#pragma unroll
        for (int k = 0; k < kVec; k++) {
            const uint32_t v = v0 + threadIdx.x + k * kThreads;
            if (v < nvec) {
                const uint32_t r = fdiv(v, d.div_vpr);
                const uint32_t c = v - r * d.vpr;
                uint64_t off;
                if (d.nhd) {
                    off = (uint64_t)c * 16;
                } else {  // head-split destination (e.g. HND): head h, 16-byte piece e of that head
                    const uint32_t h = fdiv(c, d.div_hdv);
                    const uint32_t e = c - h * d.div_hdv.d;
                    off = (uint64_t)h * d.head_stride + (uint64_t)e * 16;
                }
                st_global(s_dst[r] + off, buf[k]);
            }
        }
    }
}

// Thread 0 of a CTA that completed layer l's work: publish layers in increasing order.
__device__ void advance_ready(const DevDesc& d) {
    const uint32_t base = (d.epoch - 1u) * d.L;
    while (true) {
        const uint32_t r = ld_acquire(d.ready);
        const uint32_t rel = r - base;
        if (rel >= d.L) return;
        if (ld_acquire(&d.done_epoch[rel]) != d.epoch) return;
        if (atomicCAS(d.ready, r, r + 1u) == r) {
            d.ts[1 + rel] = globaltimer();
            __threadfence_system();
            ((volatile uint32_t*)d.host_ready)[rel] = d.epoch;
        }
        __threadfence();
    }
}

__device__ __forceinline__ void complete_unit(const DevDesc& d, uint32_t layer) {
    // Called by thread 0 after a __syncthreads(): the CTA's stores happen-before this fence
    // (cumulativity), so they are visible GPU-wide before the counter moves.
    __threadfence();
    const uint32_t target = d.epoch * d.units_per_layer;
    const uint32_t old = atomicAdd(&d.unit_cnt[layer], 1u);
    if (old + 1u == target) {
        atomicExch(&d.done_epoch[layer], d.epoch);
        __threadfence();
        advance_ready(d);
    }
}

__global__ void __launch_bounds__(kThreads) fetch_persistent_kernel(const DevDesc d) {
    __shared__ uint64_t s_dst[kMaxRows];
    const uint64_t t0 = globaltimer();
    if (blockIdx.x == 0 && threadIdx.x == 0) d.ts[0] = t0;
    const uint32_t total = d.L * d.units_per_layer;
    uint32_t layer = blockIdx.x / d.units_per_layer;
    uint32_t unit = blockIdx.x - layer * d.units_per_layer;
    for (uint32_t g = blockIdx.x; g < total; g += gridDim.x) {
        if (d.pace_ns) {  // minimal pacer: layer l released at t0 + l * pace
            const uint64_t rel = t0 + (uint64_t)layer * d.pace_ns;
            while (globaltimer() < rel) __nanosleep(2000);
        }
        copy_unit(d, layer, unit, s_dst);
        __syncthreads();
        if (threadIdx.x == 0) complete_unit(d, layer);
        // advance (layer, unit) by gridDim.x units without a division
        unit += gridDim.x;
        while (unit >= d.units_per_layer) {
            unit -= d.units_per_layer;
            layer++;
        }
    }
}

__global__ void __launch_bounds__(kThreads) fetch_layer_kernel(const DevDesc d, uint32_t layer) {
    __shared__ uint64_t s_dst[kMaxRows];
    if (layer == 0 && blockIdx.x == 0 && threadIdx.x == 0) d.ts[0] = globaltimer();
    for (uint32_t unit = blockIdx.x; unit < d.units_per_layer; unit += gridDim.x) {
        copy_unit(d, layer, unit, s_dst);
        __syncthreads();
        if (threadIdx.x == 0) complete_unit(d, layer);
    }
}

__global__ void wait_geq_kernel(const uint32_t* addr, uint32_t value) {
    while ((int32_t)(ld_acquire(addr) - value) < 0) __nanosleep(256);
}

namespace {

int occupancy(const void* fn) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, 0) != cudaSuccess || occ < 1) {
        cudaGetLastError();
        occ = 1;
    }
    return occ;
}

bool force_wait_kernel() {
    const char* e = std::getenv("OC_WAIT_KERNEL");
    return e && e[0] == '1';
}

}  // namespace

int launch_fetch(Desc* d, const oc_fetch_opts& o, cudaStream_t s) {
    if (o.mode != OC_FETCH_PERSISTENT && o.mode != OC_FETCH_PER_LAYER)
        return fail(OC_EINVAL, "fetch_layerwise: unknown mode");
    if (o.engine != OC_COPY_LDST) return fail(OC_ENOTSUP, "fetch_layerwise: copy engine not available yet");
    if (o.pace_Bps < 0) return fail(OC_EINVAL, "fetch_layerwise: pace must be >= 0");
    if (o.pace_Bps > 0 && o.mode != OC_FETCH_PERSISTENT)
        return fail(OC_ENOTSUP, "fetch_layerwise: pacing needs PERSISTENT mode");
    DeviceGuard dg(d->device);
    if (!d->done_ev) OC_CUDA(cudaEventCreateWithFlags(&d->done_ev, cudaEventDisableTiming));
    plan_units(d, o.unit_bytes);
    DevDesc& dd = d->dd;
    if ((uint64_t)dd.units_per_layer * dd.L >= (1ull << 32)) return fail(OC_ERANGE, "fetch_layerwise: too many units");
    d->epoch++;
    if (d->epoch == 0) d->epoch = 1;  // never 0: done_epoch starts at 0
    dd.epoch = d->epoch;
    dd.pace_ns = o.pace_Bps > 0 ? (uint64_t)((double)d->N * d->geo.S / o.pace_Bps * 1e9) : 0;
    const int sms = device_sm_count(d->device);
    if (o.mode == OC_FETCH_PERSISTENT) {
        static int occ = occupancy((const void*)fetch_persistent_kernel);
        uint64_t grid = (uint64_t)occ * sms;
        if (o.max_ctas) grid = std::min<uint64_t>(grid, o.max_ctas);
        grid = std::min<uint64_t>(grid, (uint64_t)dd.units_per_layer * dd.L);
        fetch_persistent_kernel<<<(unsigned)grid, kThreads, 0, s>>>(dd);
        OC_CUDA(cudaGetLastError());
    } else {
        if (d->events.empty()) {
            d->events.resize(dd.L, nullptr);
            for (auto& ev : d->events) OC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        }
        static int occ = occupancy((const void*)fetch_layer_kernel);
        uint64_t grid = (uint64_t)occ * sms;
        if (o.max_ctas) grid = std::min<uint64_t>(grid, o.max_ctas);
        grid = std::min<uint64_t>(grid, dd.units_per_layer);
        for (uint32_t l = 0; l < dd.L; l++) {
            fetch_layer_kernel<<<(unsigned)grid, kThreads, 0, s>>>(dd, l);
            OC_CUDA(cudaGetLastError());
            OC_CUDA(cudaEventRecord(d->events[l], s));
        }
    }
    OC_CUDA(cudaEventRecord(d->done_ev, s));
    d->last_mode = o.mode;
    d->last_stream = s;
    d->fetched = true;
    return OC_OK;
}

}  // namespace oc

using oc::Desc;

extern "C" {

OC_API int oc_fetch_layerwise(oc_desc* h, const oc_fetch_opts* opts, void* stream) {
    if (!h) return oc::fail(OC_EINVAL, "fetch_layerwise: null descriptor");
    oc_fetch_opts o{};
    o.mode = OC_FETCH_PERSISTENT;
    o.engine = OC_COPY_LDST;
    if (opts) o = *opts;
    return oc::launch_fetch((Desc*)h, o, (cudaStream_t)stream);
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
    if (!oc::force_wait_kernel()) {
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
    volatile uint32_t* flag = d->host_ready + want_layer;
    for (uint64_t spins = 0;; spins++) {
        if (*flag == d->epoch) return OC_OK;
        if ((spins & 255) == 255) {
            cudaError_t e = cudaEventQuery(d->done_ev);
            if (e == cudaSuccess) {
                if (*flag == d->epoch) return OC_OK;
                return oc::fail(OC_ECUDA, "sync_layer: fetch finished without announcing the layer");
            }
            if (e != cudaErrorNotReady) return oc::cuda_fail(e, "sync_layer: fetch failed");
        }
    }
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

}  // extern "C"
