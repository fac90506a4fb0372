// Device code of the fetch path (included by fetch.cu only: one translation unit, so the kernel
// templates and their launchers see each other).  Sections: small device helpers, unit geometry,
// completion (release reductions + in-order observer), the LD/ST engine, the offload kernels, the
// BULK (TMA) engine with its batch claim orders.  The design notes are at the top of fetch.cu.
#pragma once
#include "oc_internal.h"

namespace oc {


constexpr int kThreads = 256;   // LDST: threads per CTA
constexpr int kVec = 8;         // LDST: 16-byte vectors in flight per thread per round
constexpr int kMaxRows = 1024;  // rows per unit (plan_units caps R)
constexpr uint32_t kFifo = 16;  // BULK: copy-warp -> signaler-warp retire FIFO (mbarrier slots)
constexpr uint32_t kBulkStaticSmem = 1280;  // BULK: FIFO + claim ring (static shared memory, rounded up)

// ---- small device helpers ------------------------------------------------------------------------
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

__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Release reduction: every write that happens-before it (this thread's, and other threads' ordered
// before it by a barrier -- PTX release is cumulative) is visible before the counter moves.
__device__ __forceinline__ void red_add_release(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void red_max_release(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.max.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// The host's copy of a ready word (pinned, mapped), stored after the device word, so a host thread
// that reads `v` there may skip its stream wait for any layer <= v: the store is executed only
// after the observer's acquire has seen every unit of those layers complete, i.e. after their bytes
// are visible at GPU scope, where the consumer's later kernels read them.  A relaxed (posted)
// store: a system-scope release fence here drains the SM's outstanding writes -- the copy CTAs'
// bulk stores beside the observer -- and made a stream-ordered 4K fetch 25 us slower (168 -> 193
// us).  Not monotone under overlapped fetches of one descriptor (a lower value may land last); the
// host then merely enqueues a wait it could have skipped.
__device__ __forceinline__ void mirror_ready(uint32_t* host_word, uint32_t v) {
    if (host_word) asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(host_word), "r"(v) : "memory");
}

// Programmatic dependent launch: this CTA will issue no more claims, so a dependent launch (the
// stream's next fetch, OC_FETCH_OVERLAP) may start claiming from the counter.  No-op otherwise.
__device__ __forceinline__ void allow_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Release pattern in two parts: one fence for a group of relaxed reductions.
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void red_add_relaxed(uint32_t* p, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Measurement support (OC_TRACE=1): stamp slot i of this CTA's ramp trace.
__device__ __forceinline__ void trace_stamp(const DevDesc& d, uint32_t i) {
    if (d.trace && blockIdx.x < kTraceCtas) d.trace[blockIdx.x * kTraceSlots + i] = globaltimer();
}

// ---- unit geometry -------------------------------------------------------------------------------
// Layer l of chunk j is 2G rows at [lS, (l+1)S) of the slot: K rows 0..G-1, then V rows G..2G-1
// (KV_L2TD, reading c2).  A unit is R consecutive rows q0 .. q0+R-1 of that slice -- contiguous
// in the source; it may cover part of K, part of V, or both.
struct UnitGeo {
    uint32_t layer, j, q0, nrows;
};

// Global unit g (layer-major): layer = g / units_per_layer; inside a layer chunk j, then tile.
__device__ __forceinline__ UnitGeo unit_geo(const DevDesc& d, uint32_t g) {
    UnitGeo u;
    u.layer = fdiv(g, d.div_upl);
    const uint32_t unit = g - u.layer * d.units_per_layer;
    u.j = fdiv(unit, d.div_tiles);
    u.q0 = (unit - u.j * d.tiles) * d.rows_per_unit;
    u.nrows = min(d.rows_per_unit, 2u * d.G - u.q0);
    return u;
}

__device__ __forceinline__ const uint8_t* unit_src(const DevDesc& d, const UnitGeo& u) {
    if (d.staged == 1)  // CE engine: layer l of chunk j was staged at stage_base[l & 1] + j*S
        return (const uint8_t*)d.stage_base[u.layer & 1] + (uint64_t)u.j * d.S + (uint64_t)u.q0 * d.row;
    if (d.staged == 2)  // flat payload [L][N][S]
        return (const uint8_t*)d.stage_base[0] + ((uint64_t)u.layer * d.N + u.j) * d.S + (uint64_t)u.q0 * d.row;
    const uint64_t base = u.layer < d.hot_layers ? d.src_hot[u.j] : d.src[u.j];  // hot layers: HBM mirror
    return (const uint8_t*)base + (uint64_t)u.layer * d.S + (uint64_t)u.q0 * d.row;
}

// Destination of row q of chunk `pos`'s layer-l slice: matrix kv = q >= G, token t = q - kv*G,
// request token u = first_token + pos*G + t, at {k,v}_base[l] + block_table[u / Bs]*block_stride
// + (u % Bs)*token_stride.
__device__ __forceinline__ uint64_t row_addr(const DevDesc& d, uint32_t layer, uint32_t pos, uint32_t q,
                                             uint32_t* slot_out) {
    const uint32_t kv = q >= d.G ? 1u : 0u;
    const uint32_t tok = d.first_token + pos * d.G + (q - kv * d.G);
    const uint32_t b = fdiv(tok, d.div_Bs);
    const uint32_t slot = tok - b * d.Bs;
    if (slot_out) *slot_out = slot;
    const uint64_t base = kv ? d.v_base[layer] : d.k_base[layer];
    return base + (uint64_t)d.bt[b] * d.block_stride + (uint64_t)slot * d.token_stride;
}

// ---- completion --------------------------------------------------------------------------------------
// Account n finished units of `layer`; the caller's writes of those units happen-before this call.
__device__ __forceinline__ void complete_units(const DevDesc& d, uint32_t layer, uint32_t n) {
    red_add_release(&d.unit_cnt[layer], n);
}

// Observer: announce layers [l0, l1) in order.  The counters are monotone across fetches; this
// fetch's units of a layer are all done when the counter reaches cnt_target (an acquire load of
// the last reduction synchronises with every release reduction before it).
__device__ void observe_layers(const DevDesc& d, uint32_t l0, uint32_t l1) {
    const uint32_t base = (d.epoch - 1u) * d.L;
    // oc_fetch_layers ranges and PER_LAYER launches may run beside the launch covering the earlier
    // layers (another stream; programmatic dependent launches): announce nothing before those are
    // announced, so `ready`, its host copy and the layer stamps only ever move through the layers
    // in order.  (The other split launches are stream-ordered.)
    if (d.wait_prev_layers && l0 > 0) {
        uint32_t ns = 64;
        while ((int32_t)(ld_acquire(d.ready) - (base + l0)) < 0) {
            __nanosleep(ns);
            ns = min(ns * 2, 1024u);
        }
    }
    for (uint32_t l = l0; l < l1; l++) {
        uint32_t ns = 32;
        while ((int32_t)(ld_acquire(&d.unit_cnt[l]) - d.cnt_target) < 0) {
            __nanosleep(ns);
            ns = min(ns * 2, 256u);
        }
        d.ts[1 + l] = globaltimer();
        // max, not a plain store: with OC_FETCH_OVERLAP the next fetch of this descriptor may
        // already announce its early layers while this one announces its last ones
        red_max_release(d.ready, base + l + 1u);
        mirror_ready(d.ready_host, base + l + 1u);
    }
}

// ---- LDST engine ---------------------------------------------------------------------------------------
// Stream nrows contiguous source rows to the destination rows listed in `tab`.
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

// Dynamic unit scheduling: units are claimed in global (layer-major) order from a monotone
// per-descriptor counter, so whichever CTAs are resident finish the layers in order -- a CTA
// that starts late (SMs busy with a co-running prefill) cannot hold back layer 0.
// Each copy CTA stops claiming after its first claim past g1, so one launch advances the counter
// by exactly (units + copy CTAs) and the host knows the next launch's grab_base.
__device__ __forceinline__ uint32_t claim_unit(const DevDesc& d, uint32_t g0, uint32_t grab_base) {
    return g0 + (atomicAdd(d.next_unit, 1u) - grab_base);
}

// Units g0 .. g1-1; CTA 0 observes layers [g0/upl, g1/upl), the other CTAs claim and copy units.
// The destination-row table is double-buffered so one barrier per unit suffices: the barrier that
// publishes unit k's table also orders every thread's unit k-1 stores before thread 0 releases
// unit k-1, while the other warps already stream unit k.
__global__ void __launch_bounds__(kThreads, 4) fetch_ldst_kernel(const DevDesc d, uint32_t g0, uint32_t g1,
                                                                 uint32_t grab_base) {
    __shared__ uint64_t s_dst[2][kMaxRows];
    __shared__ uint32_t s_g[2];
    const uint64_t t0 = globaltimer();
    // a dependent launch (OC_FETCH_OVERLAP: the stream's next fetch) may be scheduled at once; it
    // claims from another counter slot and first waits for that slot's previous user (below)
    allow_dependents();
    if (blockIdx.x == 0) {
        if (threadIdx.x == 0) {
            if (g0 == 0) d.ts[0] = t0;
            observe_layers(d, g0 / d.units_per_layer, g1 / d.units_per_layer);
        }
        return;
    }
    uint32_t pending_layer = 0;
    bool pending = false;
    uint32_t next_g = 0;
    if (threadIdx.x == 0) {  // claims stop after the first one past g1: exactly one per CTA overshoots
        // the slot's previous user (a launch kClaimSlots launches ago, possibly still running under a
        // dependent launch) has made all its claims once the counter reaches this launch's base
        while ((int32_t)(*(volatile uint32_t*)d.next_unit - grab_base) < 0) __nanosleep(64);
        s_g[0] = claim_unit(d, g0, grab_base);
        next_g = s_g[0] < g1 ? claim_unit(d, g0, grab_base) : s_g[0];  // one ahead hides the latency
    }
    __syncthreads();
    for (uint32_t k = 0;; k++) {
        const uint32_t g = s_g[k & 1];
        if (g >= g1) break;  // uniform: every thread read the same slot after the last barrier
        const UnitGeo u = unit_geo(d, g);
        if (d.pace_ns) {  // minimal pacer: layer l released at t0 + l * pace
            // mirrored (hot) layers do not cross the paced link: the schedule starts after them
            const uint64_t rel = t0 + (uint64_t)(u.layer < d.hot_layers ? 0u : u.layer - d.hot_layers) * d.pace_ns;
            // CTA-uniform decision (also the barrier that orders unit k-1's stores)
            if (__syncthreads_or(threadIdx.x == 0 && globaltimer() < rel)) {  // announce, then idle
                if (threadIdx.x == 0 && pending) complete_units(d, pending_layer, 1);
                pending = false;
                while (globaltimer() < rel) __nanosleep(2000);
            }
        }
        uint64_t* tab = s_dst[k & 1];
        for (uint32_t r = threadIdx.x; r < u.nrows; r += kThreads) tab[r] = row_addr(d, u.layer, u.j, u.q0 + r, nullptr);
        if (threadIdx.x == 0) {  // publish unit k+1 (read after the barrier below), claim k+2
            s_g[(k + 1) & 1] = next_g;
            if (next_g < g1) next_g = claim_unit(d, g0, grab_base);
        }
        __syncthreads();
        if (threadIdx.x == 0 && pending) complete_units(d, pending_layer, 1);
        copy_rows(d, unit_src(d, u), u.nrows, tab);
        pending = true;
        pending_layer = u.layer;
    }
    __syncthreads();
    if (threadIdx.x == 0 && pending) complete_units(d, pending_layer, 1);
}

// ---- offload (paged cache -> chunk slots) ----------------------------------------------------------
// The inverse of copy_rows: nrows scattered source rows (listed in `tab`) to contiguous `dst`.
__device__ __forceinline__ void gather_rows(const DevDesc& d, uint8_t* dst, uint32_t nrows, const uint64_t* tab) {
    const uint32_t nvec = nrows * d.vpr;
    for (uint32_t v0 = 0; v0 < nvec; v0 += kThreads * kVec) {
        uint4 buf[kVec];
#pragma unroll
        for (int k = 0; k < kVec; k++) {
            const uint32_t v = v0 + threadIdx.x + k * kThreads;
            if (v < nvec) {
                const uint32_t r = fdiv(v, d.div_vpr);
                const uint32_t c = v - r * d.vpr;
                uint64_t off;
                if (d.nhd) {
                    off = (uint64_t)c * 16;
                } else {
                    const uint32_t h = fdiv(c, d.div_hdv);
                    off = (uint64_t)h * d.head_stride + (uint64_t)(c - h * d.div_hdv.d) * 16;
                }
                buf[k] = ld_stream((const void*)(tab[r] + off));
            }
        }
#pragma unroll
        for (int k = 0; k < kVec; k++) {
            const uint32_t v = v0 + threadIdx.x + k * kThreads;
            if (v < nvec) st_global((uint64_t)(dst + (uint64_t)v * 16), buf[k]);
        }
    }
}

// Unit g of the offload job: chunk j (new slot d.src[j], request chunk pos[j]), matrix, row tile.
__global__ void __launch_bounds__(kThreads, 4) offload_kernel(const DevDesc d, const uint32_t* __restrict__ pos,
                                                              uint32_t total) {
    __shared__ uint64_t tab[kMaxRows];
    for (uint32_t g = blockIdx.x; g < total; g += gridDim.x) {
        const UnitGeo u = unit_geo(d, g);
        const uint32_t p = pos[u.j];
        __syncthreads();  // the previous unit is done with tab
        for (uint32_t r = threadIdx.x; r < u.nrows; r += kThreads) tab[r] = row_addr(d, u.layer, p, u.q0 + r, nullptr);
        __syncthreads();
        gather_rows(d, (uint8_t*)unit_src(d, u), u.nrows, tab);
    }
}

// ---- BULK engine ---------------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

// Non-blocking: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
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

__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Launch flavours of fetch_bulk_kernel.
//   kSingle  one descriptor; units claimed in its layer-major order.
//   kBatch   several descriptors (same L) in one launch, claimed layer-major across the batch:
//            layer l of request 0, of request 1, ..., then layer l+1 -- every request sees its
//            layers in order and all requests' early layers go first.
//   kWdrr    several descriptors; the claim order is a table of entries (request, first unit,
//            count, release us) built by weighted deficit round robin (dispatch.cpp; Alg. A2
//            lines 6-7), each request's units still in its own layer-major order.
//   kByPos   several descriptors, layer-major, and inside a layer position-major in blocks: a
//            block of B consecutive chunk positions of every request holding them (request by
//            request, each request's B positions tile by tile) before the next block.  Requests that
//            share a prefix (same chunk at the same position) then re-read each shared slice about
//            B*S bytes after the first read -- close enough that L2 still holds it, far enough
//            that the readers do not collide on the same L2 lines at once -- so HBM serves it once.
enum { kSingle = 0, kBatch = 1, kWdrr = 2, kByPos = 3 };

struct BatchArgs {
    const DevDesc* descs;  // [n] device copies of the requests' descriptors
    const uint32_t* cum;   // [n + 1] prefix sums of units_per_layer (kBatch)
    uint32_t* claim;       // batch claim counter (monotone across launches)
    const uint4* ents;     // kWdrr: claim entries {request, first unit, count, release us}
    unsigned long long* t0_slot;  // kWdrr: the launch's common start time (0 before the launch)
    uint32_t n;
    uint32_t upl_total;    // cum[n]
    uint32_t paced;        // kWdrr: entries carry release times
    FastDiv div_upl_total;
    // kByPos: members sorted by N (descending) into runs of positions with a constant number of
    // members: seg_cum[k] = units of a layer before run k, seg_pos[k] = its first position,
    // seg_cnt[k] = members holding those positions (the first seg_cnt[k] of `sorted`)
    const uint32_t* seg_cum;  // [nseg + 1]
    const uint32_t* seg_pos;  // [nseg]
    const uint32_t* seg_cnt;  // [nseg]
    const uint2* memb;        // [n] {member index, its units per layer}, N descending
    uint32_t nseg;
    uint32_t tiles;           // units per chunk-layer slice (the same for every member)
    uint32_t pos_block;       // B: positions per block
    uint32_t pos_claim;       // kByPos: units per claim
    uint32_t n_units;         // kByPos: units of the launch
};

struct Resolved {
    const DevDesc* d;
    uint32_t g;    // unit index within the request
    uint32_t req;  // request index within the batch (0 without a batch)
};

// The batch segment the previous claim fell in -- kByPos: a run of positions; kBatch: a member's
// units of a layer (cnt = member, len = its units per layer).  A CTA's consecutive claims are ~one
// grid apart, so they usually stay in one segment: lane-0 registers, refreshed by a binary search
// only on a miss.
struct SegCache {
    uint32_t c0 = 1, c1 = 0;  // units [c0, c1) of a layer (empty until the first search)
    uint32_t cnt = 0, pos0 = 0, len = 0;
};

template <int MODE>
__device__ __forceinline__ Resolved resolve(const DevDesc& d0, const BatchArgs& ba, uint32_t g, SegCache& sc) {
    if (MODE == kSingle) return {&d0, g, 0u};
    const uint32_t layer = fdiv(g, ba.div_upl_total);
    const uint32_t rem = g - layer * ba.upl_total;
    if (MODE == kByPos) {
        if (rem < sc.c0 || rem >= sc.c1) {
            uint32_t lo = 0, hi = ba.nseg;  // largest k with seg_cum[k] <= rem
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (__ldg(&ba.seg_cum[mid]) <= rem) lo = mid;
                else hi = mid;
            }
            sc.c0 = __ldg(&ba.seg_cum[lo]);
            sc.c1 = __ldg(&ba.seg_cum[lo + 1]);
            sc.cnt = __ldg(&ba.seg_cnt[lo]);
            sc.pos0 = __ldg(&ba.seg_pos[lo]);
            sc.len = (sc.c1 - sc.c0) / (sc.cnt * ba.tiles);  // positions in the run
        }
        const uint32_t per_pos = sc.cnt * ba.tiles;   // units of one position across its members
        const uint32_t o = rem - sc.c0;
        const uint32_t per_blk = ba.pos_block * per_pos;
        const uint32_t bi = o / per_blk;              // block of positions
        const uint32_t r1 = o - bi * per_blk;
        const uint32_t blen = min(ba.pos_block, sc.len - bi * ba.pos_block);
        const uint32_t m = r1 / (blen * ba.tiles);    // member, then its positions, then tiles
        const uint32_t r2 = r1 - m * blen * ba.tiles;
        const uint32_t pos = sc.pos0 + bi * ba.pos_block + r2 / ba.tiles;
        const uint2 mb = __ldg(&ba.memb[m]);          // {member, units per layer}
        return {&ba.descs[mb.x], layer * mb.y + pos * ba.tiles + (r2 % ba.tiles), mb.x};
    }
    if (rem < sc.c0 || rem >= sc.c1) {  // kBatch: the cache holds the member of the last claim
        uint32_t lo = 0, hi = ba.n;  // largest r with cum[r] <= rem
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(&ba.cum[mid]) <= rem) lo = mid;
            else hi = mid;
        }
        sc.c0 = __ldg(&ba.cum[lo]);
        sc.c1 = __ldg(&ba.cum[lo + 1]);
        sc.cnt = lo;
        sc.len = sc.c1 - sc.c0;  // the member's units per layer
    }
    return {&ba.descs[sc.cnt], layer * sc.len + (rem - sc.c0), sc.cnt};
}

// Batch observer: lane i announces the layers of requests i, i+32, ...; each request's layers go
// out in order (same protocol as observe_layers).  The lane polls its requests round-robin without
// blocking on any one of them -- under WDRR a light request may be many layers behind a heavy one.
// A request's next layer is read back from its ready word, which only this lane writes during the
// fetch (it holds (epoch-1)*L when the fetch starts: the previous fetch announced all L layers).
__device__ void observe_batch(const BatchArgs& ba, uint64_t t0) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t left = 0;
    for (uint32_t r = lane; r < ba.n; r += 32) {
        ba.descs[r].ts[0] = t0;
        left++;
    }
    uint32_t ns = 32;
    while (left) {
        bool moved = false;
        for (uint32_t r = lane; r < ba.n; r += 32) {
            const DevDesc& d = ba.descs[r];
            const uint32_t base = (d.epoch - 1u) * d.L;
            uint32_t l = *(volatile uint32_t*)d.ready - base;
            if (l >= d.L) continue;
            while (l < d.L && (int32_t)(ld_acquire(&d.unit_cnt[l]) - d.cnt_target) >= 0) {
                d.ts[1 + l] = globaltimer();
                st_release(d.ready, base + l + 1u);
                mirror_ready(d.ready_host, base + l + 1u);
                l++;
                moved = true;
            }
            if (l == d.L) left--;
        }
        if (moved) {
            ns = 32;
        } else {
            __nanosleep(ns);
            ns = min(ns * 2, 256u);
        }
    }
}

// CTA 0: observer.  CTA b >= 1: warp 0 claims units and copies them through a `stages`-deep
// shared-memory ring; warp 1 (lane 0) turns the copy warp's retire records -- handed over through
// an mbarrier-guarded shared-memory FIFO -- into release reductions, so the copy pipeline never
// waits on a GPU-scope fence.  A unit is retired once its bulk stores
// are complete (wait_group with a lag of two units, so stores stay in flight).
template <int MODE>
__global__ void __launch_bounds__(64) fetch_bulk_kernel(const __grid_constant__ DevDesc d0,
                                                        const __grid_constant__ BatchArgs ba, uint32_t g0,
                                                        uint32_t g1, uint32_t grab_base, uint32_t stages,
                                                        uint32_t stage_bytes) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint32_t fifo_req[kFifo], fifo_layer[kFifo], fifo_n[kFifo];
    __shared__ uint32_t s_unit[32], s_req[32], s_rel[32];
    constexpr bool BATCH = MODE != kSingle;
    __shared__ __align__(8) uint64_t fifo_full[kFifo], fifo_empty[kFifo];
    const uint64_t t0 = globaltimer();
    // kSingle: a dependent launch (OC_FETCH_OVERLAP, or the next layer's launch in PER_LAYER mode)
    // may start at once: it claims from another counter slot and waits for its slot's earlier user
    if (!BATCH) allow_dependents();
    if (blockIdx.x == 0) {
        if (BATCH) {
            if (threadIdx.x < 32) observe_batch(ba, t0);
        } else {
            if (threadIdx.x == 0) {
                if (g0 == 0 && d0.staged != 1) d0.ts[0] = t0;  // CE engine: stamped when the copies start
                observe_layers(d0, g0 / d0.units_per_layer, g1 / d0.units_per_layer);
            }
        }
        return;
    }
    uint64_t* bars = (uint64_t*)smem;
    uint8_t* buf = smem + 128;
    const uint32_t lane = threadIdx.x & 31;
    const bool tr = !BATCH && d0.trace != nullptr;  // ramp trace (measurement support)
    if (tr && threadIdx.x == 0) d0.trace[blockIdx.x * kTraceSlots + 0] = t0;
    // kSingle: the first unit is static (below); start the load of its source address now, so its
    // latency overlaps the barrier set-up
    const uint8_t* src0 = (MODE == kSingle && threadIdx.x == 0) ? unit_src(d0, unit_geo(d0, g0 + blockIdx.x - 1))
                                                                 : nullptr;
    // barriers: one per thread (stages <= 16 ring slots, 2 * kFifo FIFO slots)
    if (threadIdx.x < stages) mbar_init(&bars[threadIdx.x], 1);
    if (threadIdx.x < kFifo) {
        mbar_init(&fifo_full[threadIdx.x], 1);
        mbar_init(&fifo_empty[threadIdx.x], 1);
    }
    // the inits (generic proxy) before the TMA's complete_tx (async proxy); no cluster peers
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x >= 32) {  // ---- signaler warp
        if (threadIdx.x != 32) return;
        // Each round takes every record already in the FIFO (waiting only for the first), merges
        // records of the same (request, layer), then publishes them with ONE GPU-scope release
        // fence followed by relaxed reductions (a PTX release pattern) -- a fence per record
        // (MEMBAR.GPU + ERRBAR) throttled batches that change request at every unit.
        constexpr int kBatchRec = 8;
        uint32_t h = 0;  // slot h % kFifo, round h / kFifo
        bool done = false;
        while (!done) {
            uint32_t rq[kBatchRec], ly[kBatchRec], nn[kBatchRec];
            int m = 0;
            for (int taken = 0; taken < kBatchRec; taken++, h++) {
                const uint32_t f = h % kFifo;
                if (taken == 0) mbar_wait(&fifo_full[f], (h / kFifo) & 1u);  // acquire: the record is visible
                else if (!mbar_test(&fifo_full[f], (h / kFifo) & 1u)) break;
                const uint32_t req = fifo_req[f], layer = fifo_layer[f], n = fifo_n[f];
                mbar_arrive(&fifo_empty[f]);                 // release: the slot may be reused
                if (layer == 0xffffffffu) {
                    done = true;
                    h++;
                    break;
                }
                int e = 0;
                while (e < m && !(rq[e] == req && ly[e] == layer)) e++;
                if (e == m) {
                    rq[m] = req;
                    ly[m] = layer;
                    nn[m++] = n;
                } else {
                    nn[e] += n;
                }
            }
            if (m) {
                fence_acq_rel_gpu();
                for (int e = 0; e < m; e++) red_add_relaxed(&(BATCH ? ba.descs[rq[e]] : d0).unit_cnt[ly[e]], nn[e]);
                if (tr && d0.trace[blockIdx.x * kTraceSlots + 7] == 0) trace_stamp(d0, 7);
            }
        }
        return;
    }
    // ---- copy warp
    constexpr uint32_t kEnd = 0xffffffffu;
    uint32_t* claim_ctr = BATCH ? ba.claim : d0.next_unit;
    uint32_t tail = 0;
    auto push = [&](uint32_t req, uint32_t layer, uint32_t n) {  // lane 0 only
        const uint32_t f = tail % kFifo;
        mbar_wait(&fifo_empty[f], ((tail / kFifo) & 1u) ^ 1u);  // round 0 passes on the fresh barrier
        fifo_req[f] = req;
        fifo_layer[f] = layer;
        fifo_n[f] = n;
        mbar_arrive(&fifo_full[f]);
        tail++;
    };
    // s_unit/s_req[k % 32] = the k-th unit this CTA claimed (kEnd once the launch's units run out).
    bool exhausted = false;  // lane 0 only
    // The claim for the next unit is issued one claim ahead, so the atomic's round trip (~1 us)
    // overlaps a unit's copy instead of stalling the issue loop -- with a small copy-CTA budget
    // that latency would otherwise cap each CTA at one unit per round trip.
    // kSingle: copy CTA b's first unit is g0 + b - 1 (the host sizes the grid to at most the
    // launch's units), so the first load goes out without a claim round trip; later claims come
    // from the counter, which maps value c to unit g0 + copy CTAs + (c - grab_base).
    // kRampStatic2: the first layer's remainder goes to CTAs 1..extra as static second units, and
    // the counter then starts after them.
    const uint32_t copy_ctas = gridDim.x - 1;
    const uint32_t cta_i = blockIdx.x - 1u;
    const uint32_t extra = (MODE == kSingle && (d0.ramp & kRampStatic2))
                               ? ramp_extra(g0, g1, d0.units_per_layer, copy_ctas) : 0u;
    const bool static2 = extra != 0 && cta_i < extra;
    uint32_t next_raw = (lane == 0 && MODE != kSingle) ? atomicAdd(claim_ctr, 1u) : 0u;
    if (tr && lane == 0) trace_stamp(d0, 2);
    // kWdrr: the entry being consumed (lane 0) and the launch's common start time
    uint32_t cur_req = 0, cur_next = 0, cur_left = 0, cur_rel = 0;
    SegCache seg_cache;  // kByPos (lane 0)
    uint64_t t_start = t0;
    if (MODE == kWdrr && ba.paced && lane == 0) {
        const unsigned long long old = atomicCAS(ba.t0_slot, 0ull, (unsigned long long)t0);
        t_start = old ? old : t0;
    }
    auto claim = [&](uint32_t k) {  // lane 0 only: claim unit k, returns false at the end
        uint32_t g = kEnd, req = 0;
        if (MODE == kWdrr) {
            if (!exhausted && cur_left == 0) {  // take the next entry (claims stop past g1 as below)
                const uint32_t e = g0 + (next_raw - grab_base);
                if (e >= g1) {
                    exhausted = true;
                } else {
                    next_raw = atomicAdd(claim_ctr, 1u);
                    const uint4 en = ba.ents[e];
                    cur_req = en.x;
                    cur_next = en.y;
                    cur_left = en.z;
                    cur_rel = en.w;
                }
            }
            if (!exhausted) {
                g = cur_next++;
                cur_left--;
                req = cur_req;
                s_rel[k % 32] = cur_rel;
            }
        } else if (MODE == kByPos) {
            // claims of pos_claim consecutive units of the position-major order: one atomic per
            // claim, and a CTA streams one member's run of positions
            if (!exhausted && cur_left == 0) {
                const uint32_t c = g0 + (next_raw - grab_base);
                if (c >= g1) {
                    exhausted = true;
                } else {
                    next_raw = atomicAdd(claim_ctr, 1u);
                    cur_next = c * ba.pos_claim;
                    cur_left = min(ba.pos_claim, ba.n_units - cur_next);
                }
            }
            if (!exhausted) {
                const Resolved rs = resolve<MODE>(d0, ba, cur_next++, seg_cache);
                cur_left--;
                g = rs.g;
                req = rs.req;
            }
        } else if (!exhausted) {
            // Each copy CTA stops after its first counter claim past g1.  kSingle: the static first
            // units plus one overshoot per CTA -- the counter advances by exactly the launch's
            // units; batches: by (units + copy CTAs).  The host knows the next launch's grab_base.
            uint32_t gg;
            bool take_next = true;  // issue the next counter claim (one ahead)
            if (MODE == kSingle) {
                if (k == 0) {
                    gg = g0 + cta_i;
                } else if (k == 1 && static2) {
                    gg = g0 + copy_ctas + cta_i;
                    take_next = false;  // the claim issued at k = 0 is still ahead
                } else {
                    gg = g0 + copy_ctas + extra + (next_raw - grab_base);
                }
                if (k == 0) {
                    // the slot's previous user (a launch kSlots launches ago, possibly still running
                    // under a dependent launch) has made all its claims once the counter reaches
                    // this launch's base; in stream order it has long finished
                    while ((int32_t)(*(volatile uint32_t*)claim_ctr - grab_base) < 0) __nanosleep(64);
                }
            } else {
                gg = g0 + (next_raw - grab_base);
            }
            if (gg >= g1) {
                exhausted = true;
            } else {
                if (take_next) next_raw = atomicAdd(claim_ctr, 1u);
                const Resolved rs = resolve<MODE>(d0, ba, gg, seg_cache);
                g = rs.g;
                req = rs.req;
            }
        }
        s_unit[k % 32] = g;
        s_req[k % 32] = req;
        return g != kEnd;
    };
    auto desc_of = [&](uint32_t k) -> const DevDesc& { return BATCH ? ba.descs[s_req[k % 32]] : d0; };
    auto issue_load = [&](uint32_t k) {  // lane 0 only, after a successful claim(k)
        const DevDesc& d = desc_of(k);
        const UnitGeo u = unit_geo(d, s_unit[k % 32]);
        const uint32_t bytes = (uint32_t)(u.nrows * d.row);
        const uint32_t s = k % stages;
        mbar_expect_tx(&bars[s], bytes);
        bulk_load(buf + (size_t)s * stage_bytes, (MODE == kSingle && k == 0) ? src0 : unit_src(d, u), bytes, &bars[s]);
    };
    // kSingle: minimal pacer, layer l released at t0 + l * pace.  kWdrr: the entry's
    // release time after the launch's start (Alg. A2 line 6, reading c22).
    const bool paced = MODE == kSingle ? (d0.pace_ns != 0 || d0.pace_ns_per_byte > 0.0)
                                       : (MODE == kWdrr && ba.paced != 0);
    auto release_time = [&](uint32_t k) -> uint64_t {
        if (MODE == kWdrr) return t_start + (uint64_t)s_rel[k % 32] * 1000ull;
        const DevDesc& d = desc_of(k);
        // Mirrored (hot) layers do not cross the paced link: they go at once, and the link's
        // schedule counts only the layers after them.
        if (d.pace_ns_per_byte > 0.0) {  // strict: the unit's first byte among the link's bytes
            const UnitGeo u = unit_geo(d, s_unit[k % 32]);
            if (u.layer < d.hot_layers) return t0;
            const double b = (double)(u.layer - d.hot_layers) * d.N * d.S + (double)u.j * d.S + (double)u.q0 * d.row;
            return t0 + (uint64_t)(b * d.pace_ns_per_byte);
        }
        const uint32_t layer = fdiv(s_unit[k % 32], d.div_upl);
        return t0 + (uint64_t)(layer < d.hot_layers ? 0u : layer - d.hot_layers) * d.pace_ns;
    };
    // Retired units are batched per (request, layer): one record per change.
    uint32_t pend_req = 0, pend_layer = 0, pend_cnt = 0;
    auto flush = [&]() {
        if (pend_cnt) {
            push(pend_req, pend_layer, pend_cnt);
            pend_cnt = 0;
        }
    };
    auto retire = [&](uint32_t k) {  // unit k's stores are complete (every lane waited)
        const uint32_t req = s_req[k % 32];
        const uint32_t layer = fdiv(s_unit[k % 32], desc_of(k).div_upl);
        if (pend_cnt && (layer != pend_layer || req != pend_req)) flush();
        pend_req = req;
        pend_layer = layer;
        pend_cnt++;
    };

    // Prologue: units 0 .. stages-2 (plus a static second unit with a 2-stage ring).
    const uint32_t prologue = max(stages - 1u, static2 ? 2u : 1u);
    uint32_t issued = 0;  // units claimed and loaded so far (warp-uniform after the shuffle)
    if (lane == 0)
        for (uint32_t k = 0; k < prologue; k++) {
            if (!claim(k)) break;
            if (paced)
                while (globaltimer() < release_time(k)) __nanosleep(2000);
            issue_load(k);
            issued++;
            if (tr && k == 0) trace_stamp(d0, 3);
        }
    issued = __shfl_sync(0xffffffffu, issued, 0);
    __syncwarp();
    // kRampFirstLayer: the launch's first layer (kSingle)
    const uint32_t first_layer = MODE == kSingle ? fdiv(g0, d0.div_upl) : 0u;
    const bool first_layer_hold = MODE == kSingle && !paced && (d0.ramp & kRampFirstLayer);

    uint32_t next_retire = 0;  // first unit not yet retired (same value in every lane)
    uint32_t k = 0;
    for (;; k++) {
        const uint32_t g = s_unit[k % 32];
        if (g == kEnd) break;
        const DevDesc& d = desc_of(k);
        const uint32_t s = k % stages;
        const UnitGeo u = unit_geo(d, g);
        // Row-contiguous targets with units of <= 32 rows (32 KiB at Llama layouts): lane r's
        // destination run is computed while the unit's load is still in flight, so the block-table
        // and base loads do not delay the stores.  Lane r owns row r if row r starts a run: the
        // unit's first row, a block's first slot, or the first V row; a run ends at the next one.
        const bool lane_rows = d.nhd && u.nrows <= 32;
        uint64_t run_dst = 0;
        uint32_t run_bytes = 0;
        if (lane_rows && lane < u.nrows) {
            const uint32_t q = u.q0 + lane;
            uint32_t slot;
            const uint64_t dst = row_addr(d, u.layer, u.j, q, &slot);
            if (lane == 0 || slot == 0 || q == d.G) {
                uint32_t len = min(u.nrows - lane, d.Bs - slot);
                if (q < d.G) len = min(len, d.G - q);
                run_dst = dst;
                run_bytes = (uint32_t)(len * d.row);
            }
        }
        mbar_wait(&bars[s], (k / stages) & 1u);
        if (tr && k == 0 && lane == 0) trace_stamp(d0, 4);
        const uint8_t* sbuf = buf + (size_t)s * stage_bytes;
        if (lane_rows) {
            if (run_bytes) bulk_store(run_dst, sbuf + (size_t)lane * d.row, run_bytes);
        } else if (d.nhd) {
            for (uint32_t r = lane; r < u.nrows; r += 32) {
                const uint32_t q = u.q0 + r;
                uint32_t slot;
                const uint64_t dst = row_addr(d, u.layer, u.j, q, &slot);
                if (r == 0 || slot == 0 || q == d.G) {
                    uint32_t len = min(u.nrows - r, d.Bs - slot);
                    if (q < d.G) len = min(len, d.G - q);
                    bulk_store(dst, sbuf + (size_t)r * d.row, (uint32_t)(len * d.row));
                }
            }
        } else {  // one store per (row, head)
            const uint32_t hdv = d.div_hdv.d;  // 16-byte pieces per head
            const uint32_t heads = d.vpr / hdv;
            const uint32_t hbytes = hdv * 16;
            for (uint32_t p = lane; p < u.nrows * heads; p += 32) {
                const uint32_t r = p / heads;
                const uint32_t h = p - r * heads;
                const uint64_t dst = row_addr(d, u.layer, u.j, u.q0 + r, nullptr) + (uint64_t)h * d.head_stride;
                bulk_store(dst, sbuf + (size_t)r * d.row + (size_t)h * hbytes, hbytes);
            }
        }
        bulk_commit();
        if (tr && k == 0 && lane == 0) trace_stamp(d0, 5);
        bulk_wait_read<1>();  // unit k-1's stage is free once its stores have read shared memory
        __syncwarp();
        const uint32_t kl = k + stages - 1;  // next unit to load, into unit k-1's stage
        const bool need = kl >= issued;      // not already loaded by the prologue
        uint32_t got = 0;
        if (need && lane == 0) got = claim(kl) ? 1u : 0u;
        got = __shfl_sync(0xffffffffu, got, 0);
        if (need && got) {
            issued++;
            if (first_layer_hold && u.layer == first_layer) {
                // the first layer is complete in this CTA before any later layer's load goes out
                const uint32_t ln = lane == 0 ? fdiv(s_unit[kl % 32], d.div_upl) : 0u;
                if (__shfl_sync(0xffffffffu, ln, 0) != first_layer) {
                    bulk_wait<0>();
                    fence_proxy_async_global();
                    __syncwarp();
                    if (lane == 0) {
                        for (uint32_t r = next_retire; r <= k; r++) retire(r);
                        // Publish the first layer's units from this warp, not through the signaler:
                        // no loads or stores of this CTA are in flight now (and the other CTAs of
                        // the SM are at the same point), so the GPU-scope release is cheap; the
                        // signaler's fence would queue behind the next layer's traffic.
                        if (tr) trace_stamp(d0, 1);
                        if (pend_cnt) {
                            red_add_release(&d0.unit_cnt[pend_layer], pend_cnt);
                            pend_cnt = 0;
                        }
                        if (tr) trace_stamp(d0, 6);
                    }
                    next_retire = k + 1;
                }
            }
            if (paced) {
                uint32_t hold = lane == 0 ? (globaltimer() < release_time(kl) ? 1u : 0u) : 0u;
                hold = __shfl_sync(0xffffffffu, hold, 0);
                if (hold) {  // retire everything copied so far before idling until the release
                    bulk_wait<0>();
                    fence_proxy_async_global();
                    __syncwarp();
                    if (lane == 0) {
                        for (uint32_t r = next_retire; r <= k; r++) retire(r);
                        flush();
                        while (globaltimer() < release_time(kl)) __nanosleep(2000);
                    }
                    next_retire = k + 1;
                }
            }
            if (lane == 0) issue_load(kl);
        }
        __syncwarp();
        // Retire policy.  Units of one (request, layer) keep their stores in flight together; when
        // the next unit starts another layer (or the CTA's work ends) every outstanding unit is
        // retired as soon as its stores complete, so the layer is announced promptly.  Inside a
        // layer at most 8 units stay unretired -- a small copy-CTA budget (a CTA owning many
        // units per layer) keeps 4-8 units of stores in flight instead of waiting on each.
        // kByPos changes request at every unit, but a member's layer completes only at the end of
        // the layer: there only a layer change is a boundary.
        const uint32_t gn = s_unit[(k + 1) % 32];  // claimed already: claims run stages-1 ahead
        bool boundary = gn == kEnd || (MODE != kByPos && s_req[(k + 1) % 32] != s_req[k % 32]);
        if (!boundary)
            boundary = fdiv(gn, desc_of(k + 1).div_upl) != fdiv(g, d.div_upl);
        if (boundary) {
            bulk_wait<0>();
            fence_proxy_async_global();
            __syncwarp();
            if (lane == 0) {
                for (uint32_t r = next_retire; r <= k; r++) retire(r);
                flush();
                if (tr && next_retire == 0) trace_stamp(d0, 6);
            }
            next_retire = k + 1;
        } else if (k + 1 - next_retire >= 8) {
            bulk_wait<4>();  // units up to k-4 have completed stores
            fence_proxy_async_global();
            __syncwarp();
            if (lane == 0)
                for (uint32_t r = next_retire; r + 4 <= k; r++) retire(r);
            next_retire = k - 3;
        }
    }
    bulk_wait<0>();
    fence_proxy_async_global();
    __syncwarp();
    if (lane == 0) {
        for (uint32_t r = next_retire; r < k; r++) retire(r);
        flush();
        push(0, 0xffffffffu, 0);
    }
}

// Batched claims for the LD/ST engine: the same three orders as fetch_bulk_kernel (layer-major
// by request, by position in claims of pos_claim units, WDRR entries), produced one unit at a
// time by thread 0.
template <int MODE>
struct BatchClaimer {
    uint32_t next_raw = 0, cur_req = 0, cur_next = 0, cur_left = 0, cur_rel = 0;
    bool exhausted = false;
    SegCache sc;
    // the next unit (request, unit within it, release us); false once the launch's claims are out
    __device__ bool next(const BatchArgs& ba, uint32_t g0, uint32_t g1, uint32_t grab_base, uint32_t& req,
                         uint32_t& g, uint32_t& rel) {
        rel = 0;
        if (MODE == kBatch) {
            if (exhausted) return false;
            const uint32_t gg = g0 + (next_raw - grab_base);
            if (gg >= g1) {
                exhausted = true;
                return false;
            }
            next_raw = atomicAdd(ba.claim, 1u);
            const Resolved rs = resolve<MODE>(DevDesc{}, ba, gg, sc);
            req = rs.req;
            g = rs.g;
            return true;
        }
        if (!exhausted && cur_left == 0) {
            const uint32_t c = g0 + (next_raw - grab_base);
            if (c >= g1) {
                exhausted = true;
            } else {
                next_raw = atomicAdd(ba.claim, 1u);
                if (MODE == kWdrr) {
                    const uint4 en = ba.ents[c];
                    cur_req = en.x;
                    cur_next = en.y;
                    cur_left = en.z;
                    cur_rel = en.w;
                } else {
                    cur_next = c * ba.pos_claim;
                    cur_left = min(ba.pos_claim, ba.n_units - cur_next);
                }
            }
        }
        if (exhausted) return false;
        cur_left--;
        if (MODE == kWdrr) {
            req = cur_req;
            g = cur_next++;
            rel = cur_rel;
        } else {
            const Resolved rs = resolve<MODE>(DevDesc{}, ba, cur_next++, sc);
            req = rs.req;
            g = rs.g;
        }
        return true;
    }
};

// LD/ST engine for batches (head-split targets, where per-piece TMA stores are slow): the loop of
// fetch_ldst_kernel with units from a BatchClaimer; CTA 0's first warp is the batch observer.
template <int MODE>
__global__ void __launch_bounds__(kThreads, 4) fetch_ldst_batch_kernel(const __grid_constant__ BatchArgs ba,
                                                                        uint32_t g0, uint32_t g1, uint32_t grab_base) {
    __shared__ uint64_t s_dst[2][kMaxRows];
    __shared__ uint32_t s_g[2], s_req[2], s_rel[2], s_ok[2];
    const uint64_t t0 = globaltimer();
    if (blockIdx.x == 0) {
        if (threadIdx.x < 32) observe_batch(ba, t0);
        return;
    }
    uint64_t t_start = t0;
    BatchClaimer<MODE> cl;
    if (threadIdx.x == 0) {
        if (MODE == kWdrr && ba.paced) {
            const unsigned long long old = atomicCAS(ba.t0_slot, 0ull, (unsigned long long)t0);
            t_start = old ? old : t0;
        }
        cl.next_raw = atomicAdd(ba.claim, 1u);
        uint32_t rq = 0, g = 0, rel = 0;
        s_ok[0] = cl.next(ba, g0, g1, grab_base, rq, g, rel) ? 1u : 0u;
        s_req[0] = rq;
        s_g[0] = g;
        s_rel[0] = rel;
    }
    __syncthreads();
    uint32_t pending_req = 0, pending_layer = 0;
    bool pending = false;
    for (uint32_t k = 0;; k++) {
        const uint32_t b = k & 1;
        if (!s_ok[b]) break;  // uniform: every thread read the same slot after the last barrier
        const DevDesc& d = ba.descs[s_req[b]];
        const UnitGeo u = unit_geo(d, s_g[b]);
        if (MODE == kWdrr && ba.paced) {  // held rate (c22): wait for the entry's release time
            const uint64_t rel = t_start + (uint64_t)s_rel[b] * 1000ull;
            if (__syncthreads_or(threadIdx.x == 0 && globaltimer() < rel)) {
                if (threadIdx.x == 0 && pending) complete_units(ba.descs[pending_req], pending_layer, 1);
                pending = false;
                while (globaltimer() < rel) __nanosleep(2000);
            }
        }
        uint64_t* tab = s_dst[b];
        for (uint32_t r = threadIdx.x; r < u.nrows; r += kThreads) tab[r] = row_addr(d, u.layer, u.j, u.q0 + r, nullptr);
        if (threadIdx.x == 0) {  // publish unit k+1 (read after the barrier below)
            uint32_t rq = 0, g = 0, rel = 0;
            s_ok[b ^ 1] = cl.next(ba, g0, g1, grab_base, rq, g, rel) ? 1u : 0u;
            s_req[b ^ 1] = rq;
            s_g[b ^ 1] = g;
            s_rel[b ^ 1] = rel;
        }
        __syncthreads();
        if (threadIdx.x == 0 && pending) complete_units(ba.descs[pending_req], pending_layer, 1);
        // only thread 0 completes units: read the slot before it republishes it next iteration
        if (threadIdx.x == 0) pending_req = s_req[b];
        copy_rows(d, unit_src(d, u), u.nrows, tab);
        pending = true;
        pending_layer = u.layer;
    }
    __syncthreads();
    if (threadIdx.x == 0 && pending) complete_units(ba.descs[pending_req], pending_layer, 1);
}

// Offload on the TMA (put_from_paged): the mirror of fetch_bulk_kernel.  A unit is R rows of
// one new chunk's layer slice; its rows are gathered from their paged slots (one bulk load per
// contiguous run, all completing on the stage's mbarrier) into shared memory, then written to the
// slot with one contiguous bulk store.  One warp per CTA, units claimed from the job's counter.
__global__ void __launch_bounds__(32) offload_bulk_kernel(const __grid_constant__ DevDesc d,
                                                          const uint32_t* __restrict__ pos, uint32_t total,
                                                          uint32_t stages, uint32_t stage_bytes) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint32_t s_unit[32];
    constexpr uint32_t kEnd = 0xffffffffu;
    uint64_t* bars = (uint64_t*)smem;
    uint8_t* buf = smem + 128;
    const uint32_t lane = threadIdx.x;
    if (lane == 0) {
        for (uint32_t s = 0; s < stages; s++) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // CTA b's first unit is b (the grid never exceeds the job's units), so its first loads go out
    // without a claim round trip; later units come from the counter (value c -> unit grid + c),
    // claimed one ahead so the atomic's latency overlaps a unit's copy, as in fetch_bulk_kernel.
    uint32_t next_raw = lane == 0 ? atomicAdd(d.next_unit, 1u) : 0u;
    auto claim = [&](uint32_t k) {  // all lanes; returns whether unit k exists
        if (lane == 0) {
            uint32_t g = blockIdx.x;
            if (k != 0) {
                g = gridDim.x + next_raw;
                if (g < total) next_raw = atomicAdd(d.next_unit, 1u);
            }
            s_unit[k % 32] = g < total ? g : kEnd;
        }
        __syncwarp();
        return s_unit[k % 32] != kEnd;
    };
    auto issue_loads = [&](uint32_t k) {  // all lanes
        const UnitGeo u = unit_geo(d, s_unit[k % 32]);
        const uint32_t p = __ldg(&pos[u.j]);
        const uint32_t s = k % stages;
        uint8_t* sb = buf + (size_t)s * stage_bytes;
        if (lane == 0) mbar_expect_tx(&bars[s], (uint32_t)(u.nrows * d.row));
        __syncwarp();
        if (d.nhd) {
            for (uint32_t r = lane; r < u.nrows; r += 32) {
                const uint32_t q = u.q0 + r;
                uint32_t slot;
                const uint64_t src = row_addr(d, u.layer, p, q, &slot);
                if (r == 0 || slot == 0 || q == d.G) {
                    uint32_t len = min(u.nrows - r, d.Bs - slot);
                    if (q < d.G) len = min(len, d.G - q);
                    bulk_load(sb + (size_t)r * d.row, (const void*)src, (uint32_t)(len * d.row), &bars[s]);
                }
            }
        } else {
            const uint32_t hdv = d.div_hdv.d;
            const uint32_t heads = d.vpr / hdv;
            const uint32_t hbytes = hdv * 16;
            for (uint32_t i = lane; i < u.nrows * heads; i += 32) {
                const uint32_t r = i / heads;
                const uint32_t h = i - r * heads;
                const uint64_t src = row_addr(d, u.layer, p, u.q0 + r, nullptr) + (uint64_t)h * d.head_stride;
                bulk_load(sb + (size_t)r * d.row + (size_t)h * hbytes, (const void*)src, hbytes, &bars[s]);
            }
        }
    };
    for (uint32_t k = 0; k + 1 < stages; k++) {
        if (!claim(k)) break;
        issue_loads(k);
    }
    for (uint32_t k = 0;; k++) {
        __syncwarp();
        const uint32_t g = s_unit[k % 32];
        if (g == kEnd) break;
        const UnitGeo u = unit_geo(d, g);
        const uint32_t s = k % stages;
        mbar_wait(&bars[s], (k / stages) & 1u);
        if (lane == 0) {
            bulk_store((uint64_t)unit_src(d, u), buf + (size_t)s * stage_bytes, (uint32_t)(u.nrows * d.row));
            bulk_commit();
            bulk_wait_read<1>();  // unit k-1's stage has been read by its store
        }
        __syncwarp();
        if (claim(k + stages - 1)) issue_loads(k + stages - 1);
    }
    if (lane == 0) bulk_wait<0>();  // the slots are written before the kernel ends
}

__global__ void stamp_kernel(uint64_t* ts) { ts[0] = globaltimer(); }

// CE engine into a flat client buffer: layer l has landed (the copies before this kernel on the
// copy stream are complete) -- stamp it and announce it, as the fetch kernel's observer does.
__global__ void announce_kernel(uint64_t* ts, uint32_t* ready, uint32_t* ready_host, uint32_t value) {
    ts[0] = globaltimer();
    st_release(ready, value);
    mirror_ready(ready_host, value);
}

__global__ void wait_geq_kernel(const uint32_t* addr, uint32_t value) {
    while ((int32_t)(ld_acquire(addr) - value) < 0) __nanosleep(256);
}

// Compute window C_l of the stall measurement: one thread spins on %globaltimer for
// `ns` and stamps its start and end on the same clock as the fetch's layer-ready stamps.
__global__ void emulate_kernel(uint64_t ns, uint64_t* stamps) {
    const uint64_t t0 = globaltimer();
    uint64_t t = t0;
    while (t - t0 < ns) t = globaltimer();
    if (stamps) {
        stamps[0] = t0;
        stamps[1] = t;
    }
}

}  // namespace oc
