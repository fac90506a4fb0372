// Internal definitions shared by the host C++ and the CUDA kernels of libobjcache.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <shared_mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/objcache.h"

namespace oc {

// ---- errors ----------------------------------------------------------------
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define OC_CUDA(call)                                               \
    do {                                                            \
        cudaError_t oc_e_ = (call);                                 \
        if (oc_e_ != cudaSuccess) return ::oc::cuda_fail(oc_e_, #call); \
    } while (0)

// Switch the calling thread's current device for the scope of a call.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) { prev = -1; cudaGetLastError(); }
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// ---- geometry ----------------------------------------------------------------
struct Geometry {
    uint32_t L, n_kv, d, p, G;
    uint64_t row;    // n_kv*d*p
    uint64_t hd;     // d*p
    uint64_t S;      // 2*G*row
    uint64_t chunk;  // L*S
};
int make_geometry(const oc_layout* lay, Geometry* g);
// Byte distance between consecutive slots of a store slab (common.cpp; >= g.chunk).
uint64_t slot_pitch(const Geometry& g, int tier);
bool same_layout(const oc_layout& a, const oc_layout& b);

// ---- keys --------------------------------------------------------------------
void sha256(const void* data, size_t n, uint8_t out[32]);
void chunk_key(const uint8_t prev[32], const uint32_t* tokens, uint32_t G, uint8_t out[32]);

struct KeyHash {
    size_t operator()(const oc_key& k) const {
        uint64_t h;
        std::memcpy(&h, k.b, 8);  // SHA-256 output bits are uniform
        return (size_t)h;
    }
};
struct KeyEq {
    bool operator()(const oc_key& a, const oc_key& b) const { return std::memcmp(a.b, b.b, 32) == 0; }
};

// ---- fast division for 32-bit numerators (Granlund-Montgomery round-up) -----
struct FastDiv {
    uint32_t d, m, s;
};
FastDiv make_fastdiv(uint32_t d);

__host__ __device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
#ifdef __CUDA_ARCH__
    uint64_t t = (uint64_t)__umulhi(n, f.m) + n;
#else
    uint64_t t = (((uint64_t)n * f.m) >> 32) + n;
#endif
    return (uint32_t)(t >> f.s);
}

// ---- store -------------------------------------------------------------------
struct Store {
    oc_layout layout;
    Geometry geo;
    int tier;
    int device;
    uint64_t capacity;
    uint64_t pitch = 0;       // slot i at slab + i * pitch (slot_pitch: >= geo.chunk)
    uint8_t* slab = nullptr;  // device address (HBM, mapped host, or IPC-mapped peer)
    bool owns_slab = true;
    bool ipc_mapped = false;
    bool read_only = false;
    uint64_t count = 0;
    std::unordered_map<oc_key, uint64_t, KeyHash, KeyEq> index;  // key -> slot
    std::vector<Store*> peers;
    mutable std::shared_mutex mu;
    cudaStream_t put_stream = nullptr;
    // Pinned-host stores may mirror the first hot_layers layers of every chunk in HBM (slot i's
    // mirror: hot_slab + i * hot_layers * S, the same layout as the slot's first layers), so a
    // fetch's first layers -- its exposed X0 -- come from HBM.
    uint32_t hot_layers = 0;
    uint8_t* hot_slab = nullptr;
    // put_from_paged inserts its keys before its kernel (on the caller's stream) has written the
    // slots; a later put_chunks of one of those keys compares bytes only after these events.
    std::vector<cudaEvent_t> offload_evs;  // guarded by mu
};
// Resolve a key to a device address (and the tier holding it; and its HBM mirror and mirrored
// layer count, 0 if none): local slots first, then peers.
bool store_resolve(Store* s, const oc_key& k, uint64_t* addr, int* tier = nullptr, uint64_t* hot = nullptr,
                   uint32_t* hot_layers = nullptr);

// Host -> device upload of a descriptor/offload block (descriptor.cpp).  The bytes are staged in
// pooled pinned memory and copied on a private non-blocking stream of the device; `ev` completes
// when they have landed.  Every launch that reads the block is ordered after `ev` (upload_order);
// a plain cudaMemcpy would not do: from pageable memory it may return before the DMA lands, and
// it runs on the legacy stream, which the caller's non-blocking streams do not wait for.
struct Upload {
    cudaEvent_t ev = nullptr;
    void* stage = nullptr;     // pinned staging block (released once ev is observed complete)
    uint64_t stage_cls = 0;
    bool done = false;
};
int upload_order(Upload* u, cudaStream_t s);  // make s wait for the upload (no-op once complete)
cudaStream_t upload_stream(int device);        // the device's private non-blocking upload stream
void upload_release(Upload* u);               // wait for the upload, free the stage and the event

// ---- device descriptor -----------------------------------------------------------
// Everything the copy kernel needs, passed by value as a kernel parameter.
struct DevDesc {
    const uint64_t* src;      // [N] chunk slot device addresses
    const int32_t* bt;        // block table (first entry = block of token 0)
    const uint64_t* k_base;   // [L]
    const uint64_t* v_base;   // [L]
    uint32_t* unit_cnt;       // [L] units completed (monotone across fetches)
    uint32_t* next_unit;      // unit claim counter of this launch's slot (monotone across launches)
    uint32_t* ready;          // (epoch-1)*L + number of layers announced in this fetch (monotone)
    uint32_t* ready_host;     // pinned host copy of `ready`, written after it (wait_layer's fast path)
    uint64_t* ts;             // [L+1] globaltimer: [0] kernel start, [1+l] layer ready
    uint64_t S;               // bytes of one layer of one chunk
    uint64_t row;             // bytes of one token row (n_kv*d*p)
    uint64_t block_stride, token_stride, head_stride;
    uint32_t N, L, G, Bs, first_token;
    uint32_t rows_per_unit;   // R
    uint32_t tiles;           // ceil(2G / R) units per chunk-layer slice (K and V rows)
    uint32_t units_per_layer; // N * tiles
    uint32_t vpr;             // 16-byte vectors per row
    uint32_t nhd;             // 1: a row is contiguous in the destination
    uint32_t epoch;           // fetch sequence number (>= 1)
    uint32_t cnt_target;      // unit_cnt[l] value once this fetch's units of layer l are done
    uint32_t chunk_major;     // 1: only the completion of the whole prefix is announced
    uint64_t pace_ns;         // persistent mode: ns between layer releases (0 = off)
    double pace_ns_per_byte;  // strict pacing: unit released at t0 + (fetch bytes before it) * this
    const uint64_t* src_hot;  // [N] HBM mirror of each chunk's first hot_layers layers
    uint32_t hot_layers;      // layers l < hot_layers are read from src_hot (0: none)
    uint64_t stage_base[2];   // CE engine: layer l's slices were staged at stage_base[l & 1] as [N][S]
    uint32_t staged;          // 0: sources from src[]; 1: CE stage (stage_base[l & 1]); 2: a flat
                              // layer-major payload [L][N][S] at stage_base[0] (oc_scatter_flat)
    FastDiv div_upl;          // units_per_layer
    FastDiv div_tiles;        // tiles per chunk-layer slice
    FastDiv div_vpr;
    FastDiv div_Bs;
    FastDiv div_hdv;          // (d*p)/16
    uint64_t* trace;          // measurement support (OC_TRACE=1): per-CTA ramp stamps, else null
    uint32_t ramp;            // kRampStatic2 | kRampFirstLayer (single-descriptor BULK launches)
    uint32_t wait_prev_layers;  // oc_fetch_layers continuation: the observer first waits for the
                                // earlier layers' announcement (layers announced in order)
};
// First-layer ramp of a single-descriptor BULK launch (fetch_kernels.cuh):
//   kRampStatic2     the first layer's units beyond one per copy CTA are also assigned statically
//                    (CTA b's second unit), so the whole first layer is loaded at once
//   kRampFirstLayer  a CTA retires its first-layer units before it loads a later layer's unit, so
//                    the first layer's completion is not queued behind the next layer's traffic
constexpr uint32_t kRampStatic2 = 1, kRampFirstLayer = 2;
// Units a launch of units [g0, g1) assigns statically as second units (kRampStatic2): the first
// layer's remainder beyond the copy CTAs' first units, at most one per CTA.
inline __host__ __device__ uint32_t ramp_extra(uint32_t g0, uint32_t g1, uint32_t upl, uint32_t copy_ctas) {
    const uint64_t layer_end = ((uint64_t)(g0 / upl) + 1) * upl;
    const uint32_t first_end = layer_end < g1 ? (uint32_t)layer_end : g1;
    const uint32_t base2 = g0 + copy_ctas;
    if (first_end <= base2) return 0u;
    return first_end - base2 < copy_ctas ? first_end - base2 : copy_ctas;
}
constexpr uint32_t kTraceSlots = 8;     // stamps per CTA (fetch_kernels.cuh, bulk engine)
// Claim counters per descriptor: consecutive launches claim from different slots (32 bytes apart),
// so a launch that starts during the previous one's tail (programmatic dependent launch) cannot mix
// its claims with that launch's; a launch waits (once, before its first counter claim) until its
// slot's previous user has made all of its claims.
constexpr uint32_t kClaimSlots = 4;
constexpr uint32_t kClaimSlotStride = 8;  // uint32 words
constexpr uint32_t kTraceCtas = 2048;   // CTAs traced per launch

struct Desc {
    Store* store;
    Geometry geo;
    oc_layout layout;
    int device;
    int delivery;
    uint64_t N;
    uint64_t nb;               // block table entries uploaded
    uint64_t host_chunks = 0;  // chunks whose source lives in pinned host memory (PCIe reads)
    void* dev_mem = nullptr;   // one pooled block: src, k/v base, ts, counters, block table
    uint64_t dev_mem_class = 0;
    Upload up;                 // the block's host -> device upload (launches wait for it)
    DevDesc dd;                // geometry part filled at build; epoch/units/pace at fetch
    uint32_t epoch = 0;
    uint32_t cnt_base = 0;     // unit_cnt[l] before the next fetch (same for every layer)
    uint32_t grab_ctr[kClaimSlots] = {};  // each claim slot's counter value before its next launch
    uint32_t launch_seq = 0;   // launches so far: launch n claims from slot n % kClaimSlots
    uint32_t last_mode = OC_FETCH_PERSISTENT;
    bool fetched = false;
    bool poisoned = false;     // a launch failed after the counters moved to a new epoch
    std::vector<cudaEvent_t> events;  // per-layer (PER_LAYER mode), created lazily
    cudaEvent_t done_ev = nullptr;    // recorded after every fetch launch
    cudaStream_t last_stream = nullptr;
    cudaStream_t sync_stream = nullptr;  // oc_sync_layer in PERSISTENT mode
    cudaEvent_t sync_ev = nullptr;
    // CE engine (pinned-host chunks): runs of chunks in consecutive slots, copied per layer by one
    // strided copy-engine transfer into a double-buffered HBM stage, then scattered by the kernel
    std::vector<uint64_t> run_first, run_len, run_src, run_hot;  // run_hot: the runs' HBM mirrors
    std::vector<uint64_t> run_hot_pitch;  // bytes between consecutive chunks' mirrors in a run
    uint32_t hot_layers = 0;   // leading layers with an HBM mirror for every chunk (0: none)
    uint64_t flat_base = 0;    // FLAT target: the client buffer [L][N][S] (the CE engine writes it directly)
    void* stage_mem = nullptr;
    uint64_t stage_class = 0;
    struct CeKit* ce_kit = nullptr;  // copy stream + per-layer events, pooled per (device, L)
    uint32_t* ready_host = nullptr;  // pinned mirror of dd.ready (ready_mirror_alloc)
    uint32_t range_open = 0;         // oc_fetch_layers: next layer of an incomplete fetch (0: none)
    std::vector<cudaEvent_t> range_evs;  // oc_fetch_layers: completion of each range of the open fetch
    uint32_t n_ranges = 0;               // ranges recorded in range_evs for the open fetch
    // wait_layer relay (PERSISTENT mode): a private stream turns the ready word into per-layer CUDA
    // events, so the consumer stream waits on an event (cheaper in the front end than a value wait)
    std::mutex relay_mu;
    struct RelayKit* relay = nullptr;    // stream + L events, pooled per (device, L) (fetch.cu)
    uint32_t range_unit_bytes = 0;   // unit size of the current fetch (fixed for its continuations)
};

// CE engine resources returned to their pool when a descriptor is freed (fetch.cu).
void ce_release(Desc* d);
// wait_layer relay resources returned to their pool when a descriptor is freed (fetch.cu).
void relay_release(Desc* d);
// PER_LAYER mode's events: taken from / returned to a pool per (device, L) (fetch.cu).
int per_layer_events_get(int device, uint32_t L, std::vector<cudaEvent_t>* out);
void per_layer_events_release(Desc* d);

// Pooled memory (pool.cpp): power-of-two blocks of device memory on `device`, or of pinned host
// memory (device = -1), recycled instead of returned to the driver.
void* dev_pool_alloc(int device, size_t n, uint64_t* cls_out);
void dev_pool_free(int device, void* p, uint64_t cls);
// A pinned, device-mapped word (its own 64-byte line) that mirrors a descriptor's ready word, so
// the host can see which layers are announced without a device round trip; zeroed on allocation.
uint32_t* ready_mirror_alloc();
void ready_mirror_free(uint32_t* w);


// Plan work units of about `unit_bytes` bytes and fill the unit fields of d->dd.
void plan_units(Desc* d, uint32_t unit_bytes);

// WDRR claim order (dispatch.cpp; Alg. A2 lines 6-7): entry = request, first unit, units, release us.
struct WdrrEntry {
    uint32_t req, first, count, rel_us;
};
int wdrr_plan(const uint64_t* n_units, uint32_t n, const uint32_t* tile_bytes, uint32_t tiles, const oc_wdrr_opts& w,
              std::vector<WdrrEntry>* out);

// kernel launchers (fetch.cu)
int launch_fetch(Desc* d, const oc_fetch_opts& o, cudaStream_t s, uint32_t l_end = UINT32_MAX);
int launch_fetch_range(Desc* d, const oc_fetch_opts& o, uint32_t l0, uint32_t l1, cudaStream_t s);
// Offload gather: new chunk j (slot dd.src[j]) <- the paged rows of request chunk pos[j].
// The caller orders `s` after the block's upload first.
int launch_offload(const DevDesc& dd, const uint32_t* pos, int device, cudaStream_t s, bool host_dst);

// driver entry point for cuStreamWaitValue32 (resolved lazily)
int stream_wait_geq(cudaStream_t s, uint32_t* addr, uint32_t value);

int device_sm_count(int device);

}  // namespace oc
