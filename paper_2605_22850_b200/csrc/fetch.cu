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

// Stream nrows contiguous source rows to the destination rows in `tab` (16-byte vectors, kVec
// loads in flight per thread before the matching stores).
__device__ __forceinline__ void copy_rows(const DevDesc& d, const uint8_t* src, uint32_t nrows, const uint64_t* tab) {
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
                st_global(tab[r] + off, buf[k]);
            }
        }
    }
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
    copy_rows(d, src, nrows, s_dst);
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

// Persistent LD/ST engine.  The destination-row table is double-buffered so one barrier per unit
// suffices: the barrier that publishes unit k's table also orders every thread's unit k-1 stores
// before thread 0 announces unit k-1, while the other warps already stream unit k.
__global__ void __launch_bounds__(kThreads, 4) fetch_persistent_kernel(const DevDesc d) {
    __shared__ uint64_t s_dst[2][kMaxRows];
    const uint64_t t0 = globaltimer();
    if (blockIdx.x == 0 && threadIdx.x == 0) d.ts[0] = t0;
    const uint32_t total = d.L * d.units_per_layer;
    uint32_t layer = blockIdx.x / d.units_per_layer;
    uint32_t unit = blockIdx.x - layer * d.units_per_layer;
    uint32_t pending_layer = 0;
    bool pending = false;
    uint32_t k = 0;
    for (uint32_t g = blockIdx.x; g < total; g += gridDim.x, k++) {
        if (d.pace_ns) {  // minimal pacer: layer l released at t0 + l * pace
            const uint64_t rel = t0 + (uint64_t)layer * d.pace_ns;
            // CTA-uniform decision (also the barrier that orders unit k-1's stores)
            if (__syncthreads_or(threadIdx.x == 0 && globaltimer() < rel)) {  // announce, then idle
                if (threadIdx.x == 0 && pending) complete_unit(d, pending_layer);
                pending = false;
                while (globaltimer() < rel) __nanosleep(2000);
            }
        }
        uint64_t* tab = s_dst[k & 1];
        const uint32_t j = fdiv(unit, d.div_units_per_chunk);
        const uint32_t rem = unit - j * 2u * d.tiles;
        const uint32_t kv = rem >= d.tiles ? 1u : 0u;
        const uint32_t r0 = (rem - kv * d.tiles) * d.rows_per_unit;
        const uint32_t nrows = min(d.rows_per_unit, d.G - r0);
        const uint64_t base = kv ? d.v_base[layer] : d.k_base[layer];
        const uint32_t u0 = d.first_token + j * d.G + r0;
        for (uint32_t r = threadIdx.x; r < nrows; r += kThreads) {
            const uint32_t u = u0 + r;
            const uint32_t b = fdiv(u, d.div_Bs);
            tab[r] = base + (uint64_t)d.bt[b] * d.block_stride + (uint64_t)(u - b * d.Bs) * d.token_stride;
        }
        __syncthreads();
        if (threadIdx.x == 0 && pending) complete_unit(d, pending_layer);
        const uint8_t* src = (const uint8_t*)d.src[j] + (uint64_t)layer * d.S + ((uint64_t)kv * d.G + r0) * d.row;
        copy_rows(d, src, nrows, tab);
        pending = true;
        pending_layer = layer;
        unit += gridDim.x;  // advance (layer, unit) by gridDim.x units without a division
        while (unit >= d.units_per_layer) {
            unit -= d.units_per_layer;
            layer++;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && pending) complete_unit(d, pending_layer);
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

// ---- TMA bulk engine ------------------------------------------------------------------------------
// One warp per CTA drives the copy engine: a unit (contiguous source rows) is pulled into a
// shared-memory stage with one cp.async.bulk load (mbarrier complete_tx), then pushed to its
// destination with one bulk store per contiguous destination run (a run of rows inside one
// block for NHD, one head of one row otherwise), lanes splitting the runs.  `stages` units are
// in flight per CTA; a unit is announced once its stores are complete (bulk wait_group with a
// lag of two units, so stores stay in flight).  Register and instruction cost per byte is
// near zero; the SM's load/store units are free for a co-running prefill.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "OC_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra OC_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sdst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void bulk_store(uint64_t gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

struct UnitGeo {
    uint32_t layer, j, kv, r0, nrows;
};

__device__ __forceinline__ UnitGeo unit_geo(const DevDesc& d, uint32_t g) {
    UnitGeo u;
    u.layer = fdiv(g, d.div_upl);
    const uint32_t unit = g - u.layer * d.units_per_layer;
    u.j = fdiv(unit, d.div_units_per_chunk);
    const uint32_t rem = unit - u.j * 2u * d.tiles;
    u.kv = rem >= d.tiles ? 1u : 0u;
    const uint32_t tile = rem - u.kv * d.tiles;
    u.r0 = tile * d.rows_per_unit;
    u.nrows = min(d.rows_per_unit, d.G - u.r0);
    return u;
}

// Units g in [g0, g1) are processed by this kernel; CTA b takes g0 + b, g0 + b + grid, ...
__global__ void __launch_bounds__(32) fetch_bulk_kernel(const DevDesc d, uint32_t g0, uint32_t g1,
                                                        uint32_t stages, uint32_t stage_bytes) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* bars = (uint64_t*)smem;
    uint8_t* buf = smem + 128;
    const uint32_t lane = threadIdx.x;
    const uint64_t t0 = globaltimer();
    if (g0 == 0 && blockIdx.x == 0 && lane == 0) d.ts[0] = t0;
    if (lane == 0) {
        for (uint32_t s = 0; s < stages; s++) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const uint32_t first = g0 + blockIdx.x;
    const uint32_t n_my = first < g1 ? (g1 - first + gridDim.x - 1) / gridDim.x : 0;

    auto release_time = [&](uint32_t k) {  // minimal pacer: layer l released at t0 + l * pace
        return t0 + (uint64_t)fdiv(first + k * gridDim.x, d.div_upl) * d.pace_ns;
    };
    auto issue_load = [&](uint32_t k) {
        const uint32_t g = first + k * gridDim.x;
        const UnitGeo u = unit_geo(d, g);
        const uint8_t* src = (const uint8_t*)d.src[u.j] + (uint64_t)u.layer * d.S + ((uint64_t)u.kv * d.G + u.r0) * d.row;
        const uint32_t bytes = (uint32_t)(u.nrows * d.row);
        const uint32_t s = k % stages;
        mbar_expect_tx(&bars[s], bytes);
        bulk_load(buf + (size_t)s * stage_bytes, src, bytes, &bars[s]);
    };

    // Completion of units is batched per layer: one release-add per layer change.
    uint32_t pend_layer = 0, pend_cnt = 0;
    auto flush = [&]() {
        if (pend_cnt) {
            __threadfence();
            const uint32_t target = d.epoch * d.units_per_layer;
            const uint32_t old = atomicAdd(&d.unit_cnt[pend_layer], pend_cnt);
            if (old + pend_cnt == target) {
                atomicExch(&d.done_epoch[pend_layer], d.epoch);
                __threadfence();
                advance_ready(d);
            }
            pend_cnt = 0;
        }
    };
    auto retire = [&](uint32_t k) {  // unit k's stores are complete (all lanes waited)
        const uint32_t layer = fdiv(first + k * gridDim.x, d.div_upl);
        if (pend_cnt && layer != pend_layer) flush();
        pend_layer = layer;
        pend_cnt++;
    };

    if (lane == 0)
        for (uint32_t k = 0; k + 1 < stages && k < n_my; k++) {
            if (d.pace_ns)
                while (globaltimer() < release_time(k)) __nanosleep(2000);
            issue_load(k);
        }

    uint32_t next_retire = 0;  // first unit not yet announced (same value in every lane)
    for (uint32_t k = 0; k < n_my; k++) {
        const uint32_t s = k % stages;
        const UnitGeo u = unit_geo(d, first + k * gridDim.x);
        mbar_wait(&bars[s], (k / stages) & 1u);
        const uint8_t* sbuf = buf + (size_t)s * stage_bytes;
        const uint64_t base = u.kv ? d.v_base[u.layer] : d.k_base[u.layer];
        const uint32_t u0 = d.first_token + u.j * d.G + u.r0;
        if (d.nhd) {
            // Lane r owns row r if row r starts a run: the first row, or the first slot of a block.
            for (uint32_t r = lane; r < u.nrows; r += 32) {
                const uint32_t tok = u0 + r;
                const uint32_t b = fdiv(tok, d.div_Bs);
                const uint32_t slot = tok - b * d.Bs;
                if (r == 0 || slot == 0) {
                    const uint32_t len = min(u.nrows - r, d.Bs - slot);
                    const uint64_t dst = base + (uint64_t)d.bt[b] * d.block_stride + (uint64_t)slot * d.token_stride;
                    bulk_store(dst, sbuf + (size_t)r * d.row, (uint32_t)(len * d.row));
                }
            }
        } else {
            const uint32_t hdv = d.div_hdv.d;  // 16-byte pieces per head
            const uint32_t heads = d.vpr / hdv;
            const uint32_t hbytes = hdv * 16;
            for (uint32_t p = lane; p < u.nrows * heads; p += 32) {
                const uint32_t r = p / heads;
                const uint32_t h = p - r * heads;
                const uint32_t tok = u0 + r;
                const uint32_t b = fdiv(tok, d.div_Bs);
                const uint32_t slot = tok - b * d.Bs;
                const uint64_t dst = base + (uint64_t)d.bt[b] * d.block_stride + (uint64_t)slot * d.token_stride +
                                     (uint64_t)h * d.head_stride;
                bulk_store(dst, sbuf + (size_t)r * d.row + (size_t)h * hbytes, hbytes);
            }
        }
        bulk_commit();
        // stage of unit k-1 is free once its stores have read shared memory
        bulk_wait_read<1>();
        __syncwarp();
        const uint32_t kl = k + stages - 1;  // next unit to load, into unit k-1's stage
        if (kl < n_my) {
            if (d.pace_ns) {
                uint32_t hold = lane == 0 ? (globaltimer() < release_time(kl) ? 1u : 0u) : 0u;
                hold = __shfl_sync(0xffffffffu, hold, 0);
                if (hold) {  // announce everything copied so far before idling until the release
                    bulk_wait<0>();
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        for (uint32_t r = next_retire; r <= k; r++) retire(r);
                        flush();
                        while (globaltimer() < release_time(kl)) __nanosleep(2000);
                    }
                    next_retire = k + 1;
                    __syncwarp();
                }
            }
            if (lane == 0) issue_load(kl);
        }
        if (k >= 2 && next_retire + 2 <= k) {
            bulk_wait<2>();                                   // unit k-2's stores are complete
            asm volatile("fence.proxy.async.global;" ::: "memory");
            __syncwarp();
            if (lane == 0)
                for (uint32_t r = next_retire; r + 2 <= k; r++) retire(r);
            next_retire = k - 1;
        }
    }
    bulk_wait<0>();
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
        for (uint32_t r = next_retire; r < n_my; r++) retire(r);
        flush();
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

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e && *e ? std::atoi(e) : dflt;
}

struct BulkPlan {
    uint32_t grid, stages, stage_bytes, smem;
};

// Shared-memory ring per CTA: `ctas_per_sm` CTAs share the SM's 228 KiB.
BulkPlan plan_bulk(const DevDesc& dd, int sms, uint32_t max_ctas, uint64_t units) {
    BulkPlan p;
    p.stage_bytes = (uint32_t)(((uint64_t)dd.rows_per_unit * dd.row + 127) & ~127ull);
    int per_sm = std::max(1, env_int("OC_BULK_CTAS_PER_SM", 3));
    const uint32_t sm_bytes = 228 * 1024;
    while (true) {
        uint32_t per_cta = std::min<uint32_t>(sm_bytes / per_sm - 1024, 227 * 1024);
        uint32_t st = (per_cta - 128) / p.stage_bytes;
        st = std::min<uint32_t>(st, (uint32_t)std::max(2, env_int("OC_BULK_STAGES", 16)));
        if (st >= 2 || per_sm == 1) {
            p.stages = std::max<uint32_t>(st, 1);
            break;
        }
        per_sm /= 2;
    }
    p.smem = 128 + p.stages * p.stage_bytes;
    uint64_t grid = (uint64_t)per_sm * sms;
    if (max_ctas) grid = std::min<uint64_t>(grid, max_ctas);
    p.grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(grid, units));
    return p;
}

int launch_bulk(const DevDesc& dd, const BulkPlan& p, uint32_t g0, uint32_t g1, cudaStream_t s) {
    static uint32_t attr_set = 0;
    if (p.smem > attr_set) {
        OC_CUDA(cudaFuncSetAttribute((const void*)fetch_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)std::max<uint32_t>(p.smem, 48 * 1024)));
        attr_set = p.smem;
    }
    fetch_bulk_kernel<<<p.grid, 32, p.smem, s>>>(dd, g0, g1, p.stages, p.stage_bytes);
    OC_CUDA(cudaGetLastError());
    return OC_OK;
}

}  // namespace

int launch_fetch(Desc* d, const oc_fetch_opts& o, cudaStream_t s) {
    if (o.mode != OC_FETCH_PERSISTENT && o.mode != OC_FETCH_PER_LAYER)
        return fail(OC_EINVAL, "fetch_layerwise: unknown mode");
    if (o.engine != OC_COPY_LDST && o.engine != OC_COPY_BULK) return fail(OC_EINVAL, "fetch_layerwise: unknown engine");
    if (o.pace_Bps < 0) return fail(OC_EINVAL, "fetch_layerwise: pace must be >= 0");
    if (o.pace_Bps > 0 && o.mode != OC_FETCH_PERSISTENT)
        return fail(OC_ENOTSUP, "fetch_layerwise: pacing needs PERSISTENT mode");
    DeviceGuard dg(d->device);
    if (!d->done_ev) OC_CUDA(cudaEventCreateWithFlags(&d->done_ev, cudaEventDisableTiming));
    // Measured on B200 (profiles/): bulk engine best with 16 KiB units at 3 CTAs/SM, LD/ST with 32 KiB.
    plan_units(d, o.unit_bytes ? o.unit_bytes : (o.engine == OC_COPY_BULK ? 16384u : 32768u));
    DevDesc& dd = d->dd;
    if ((uint64_t)dd.units_per_layer * dd.L >= (1ull << 32)) return fail(OC_ERANGE, "fetch_layerwise: too many units");
    d->epoch++;
    if (d->epoch == 0) d->epoch = 1;  // never 0: done_epoch starts at 0
    dd.epoch = d->epoch;
    dd.pace_ns = o.pace_Bps > 0 ? (uint64_t)((double)d->N * d->geo.S / o.pace_Bps * 1e9) : 0;
    const int sms = device_sm_count(d->device);
    const uint64_t total_units = (uint64_t)dd.units_per_layer * dd.L;
    if (o.engine == OC_COPY_BULK) {
        if (o.mode == OC_FETCH_PERSISTENT) {
            BulkPlan p = plan_bulk(dd, sms, o.max_ctas, total_units);
            int rc = launch_bulk(dd, p, 0, (uint32_t)total_units, s);
            if (rc) return rc;
        } else {
            if (d->events.empty()) {
                d->events.resize(dd.L, nullptr);
                for (auto& ev : d->events) OC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            }
            BulkPlan p = plan_bulk(dd, sms, o.max_ctas, dd.units_per_layer);
            for (uint32_t l = 0; l < dd.L; l++) {
                int rc = launch_bulk(dd, p, l * dd.units_per_layer, (l + 1) * dd.units_per_layer, s);
                if (rc) return rc;
                OC_CUDA(cudaEventRecord(d->events[l], s));
            }
        }
    } else if (o.mode == OC_FETCH_PERSISTENT) {
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
    o.engine = OC_COPY_BULK;
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
