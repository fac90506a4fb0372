// Hash-addressed chunk store: HBM or pinned-host slab + host key index.
//
// prefix KV chunks are immutable, addressed by their rolling
// prefix hash, deduplicated by key; new KV blocks are offloaded for future reuse.
// prefix lookup returns the ordered list of matched chunks.
// The store is append-only (no eviction in scope), so a slot address handed to a descriptor stays
// valid for the store's lifetime.  The key index is single-writer / multi-reader.
#include <algorithm>

#include <cuda.h>

#include "oc_internal.h"

namespace oc {
namespace {

const uint32_t kExportMagic = 0x4f434558;  // "OCEX"

struct ExportHeader {
    uint32_t magic;
    uint32_t version;
    oc_layout layout;
    uint32_t tier;
    uint64_t capacity;
    uint64_t count;
    uint64_t pitch;
    cudaIpcMemHandle_t handle;
};

// Size of the allocation an (IPC-mapped) device pointer lies in, through cuMemGetAddressRange
// resolved via the runtime (no link-time libcuda).  0 when unavailable.
uint64_t mapped_bytes(const void* p) {
    typedef CUresult (*PFN_range)(CUdeviceptr*, size_t*, CUdeviceptr);
    static std::once_flag once;
    static PFN_range fn = nullptr;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &f, 12000, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_range)f;
        cudaGetLastError();
    });
    CUdeviceptr base = 0;
    size_t size = 0;
    if (!fn || fn(&base, &size, (CUdeviceptr)p) != CUDA_SUCCESS) return 0;
    return (uint64_t)size - ((uint64_t)(uintptr_t)p - (uint64_t)base);
}

}  // namespace

bool store_resolve(Store* s, const oc_key& k, uint64_t* addr, int* tier, uint64_t* hot, uint32_t* hot_layers) {
    std::vector<Store*> peers;
    {
        std::shared_lock<std::shared_mutex> lk(s->mu);
        auto it = s->index.find(k);
        if (it != s->index.end()) {
            *addr = (uint64_t)(uintptr_t)s->slab + it->second * s->pitch;
            if (tier) *tier = s->tier;
            if (hot) *hot = s->hot_layers ? (uint64_t)(uintptr_t)s->hot_slab + it->second * s->hot_layers * s->geo.S : 0;
            if (hot_layers) *hot_layers = s->hot_layers;
            return true;
        }
        // copy the peer list under the lock: attach_peer may grow (reallocate) it concurrently
        peers = s->peers;
    }
    for (Store* p : peers)
        if (store_resolve(p, k, addr, tier, hot, hot_layers)) return true;
    return false;
}

namespace {
// Is `target` reachable from `from` along attached peers (including from itself)?
bool reaches(Store* from, const Store* target) {
    if (from == target) return true;
    std::vector<Store*> peers;
    {
        std::shared_lock<std::shared_mutex> lk(from->mu);
        peers = from->peers;
    }
    for (Store* p : peers)
        if (reaches(p, target)) return true;
    return false;
}
}  // namespace

}  // namespace oc

using oc::Store;

extern "C" {

OC_API int oc_store_create(const oc_layout* layout, int tier, int device, uint64_t capacity, oc_store** out) {
    if (!out) return oc::fail(OC_EINVAL, "store_create: null out");
    *out = nullptr;
    oc::Geometry g;
    int rc = oc::make_geometry(layout, &g);
    if (rc) return rc;
    if (tier != OC_TIER_HBM && tier != OC_TIER_PINNED_HOST) return oc::fail(OC_EINVAL, "store_create: bad tier");
    if (capacity == 0) return oc::fail(OC_EINVAL, "store_create: capacity must be >= 1");
    const uint64_t pitch = oc::slot_pitch(g, tier);
    if (capacity > (1ull << 40) / 1 || (unsigned __int128)capacity * pitch >> 62)
        return oc::fail(OC_EINVAL, "store_create: capacity too large");
    if (g.row % 16 || g.hd % 16) return oc::fail(OC_EALIGN, "store_create: n_kv*d*p and d*p must be multiples of 16");
    int ndev = 0;
    OC_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return oc::fail(OC_EINVAL, "store_create: no such device");
    oc::DeviceGuard dg(device);
    auto s = std::make_unique<Store>();
    s->layout = *layout;
    s->geo = g;
    s->tier = tier;
    s->device = device;
    s->capacity = capacity;
    s->pitch = pitch;
    uint64_t bytes = capacity * pitch;
    void* p = nullptr;
    cudaError_t e;
    if (tier == OC_TIER_HBM) e = cudaMalloc(&p, bytes);
    else e = cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return oc::fail(OC_ENOMEM, std::string("store_create: slab allocation of ") + std::to_string(bytes) +
                                       " bytes failed: " + cudaGetErrorString(e));
    }
    if (tier == OC_TIER_PINNED_HOST) {
        void* dp = nullptr;
        e = cudaHostGetDevicePointer(&dp, p, 0);
        if (e != cudaSuccess || dp != p) {
            cudaFreeHost(p);
            return oc::fail(OC_ECUDA, "store_create: pinned slab is not UVA-mapped");
        }
    }
    s->slab = (uint8_t*)p;
    e = cudaStreamCreateWithFlags(&s->put_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        if (tier == OC_TIER_HBM) cudaFree(p); else cudaFreeHost(p);
        return oc::cuda_fail(e, "store_create: stream");
    }
    s->index.reserve(std::min<uint64_t>(capacity, 1u << 20) * 2);
    *out = (oc_store*)s.release();
    return OC_OK;
}

OC_API int oc_store_destroy(oc_store* h) {
    if (!h) return OC_OK;
    Store* s = (Store*)h;
    {
        oc::DeviceGuard dg(s->device);
        for (cudaEvent_t ev : s->offload_evs) {  // offloads write the slab until they finish
            cudaEventSynchronize(ev);
            cudaEventDestroy(ev);
        }
        if (s->put_stream) cudaStreamDestroy(s->put_stream);
        if (s->hot_slab) cudaFree(s->hot_slab);
        if (s->ipc_mapped) cudaIpcCloseMemHandle(s->slab);
        else if (s->owns_slab) {
            if (s->tier == OC_TIER_HBM) cudaFree(s->slab);
            else cudaFreeHost(s->slab);
        }
        cudaGetLastError();
    }
    delete s;
    return OC_OK;
}

OC_API int oc_store_set_hot_layers(oc_store* h, uint32_t hot_layers) {
    if (!h) return oc::fail(OC_EINVAL, "store_set_hot_layers: null store");
    Store* s = (Store*)h;
    if (s->tier != OC_TIER_PINNED_HOST || s->read_only)
        return oc::fail(OC_EINVAL, "store_set_hot_layers: only for an own pinned-host store");
    if (hot_layers > s->geo.L) return oc::fail(OC_ERANGE, "store_set_hot_layers: more layers than the model has");
    std::unique_lock<std::shared_mutex> lk(s->mu);
    if (s->count) return oc::fail(OC_EINVAL, "store_set_hot_layers: the store already holds chunks");
    oc::DeviceGuard dg(s->device);
    if (s->hot_slab) {
        cudaFree(s->hot_slab);
        s->hot_slab = nullptr;
    }
    s->hot_layers = 0;
    if (hot_layers) {
        OC_CUDA(cudaMalloc((void**)&s->hot_slab, s->capacity * hot_layers * s->geo.S));
        s->hot_layers = hot_layers;
    }
    return OC_OK;
}

OC_API int oc_store_count(const oc_store* h, uint64_t* n) {
    if (!h || !n) return oc::fail(OC_EINVAL, "store_count: null pointer");
    const Store* s = (const Store*)h;
    std::shared_lock<std::shared_mutex> lk(s->mu);
    *n = s->count;
    return OC_OK;
}

OC_API int oc_store_slab(const oc_store* h, uint64_t* base, uint64_t* bytes) {
    if (!h) return oc::fail(OC_EINVAL, "store_slab: null store");
    const Store* s = (const Store*)h;
    if (base) *base = (uint64_t)(uintptr_t)s->slab;
    if (bytes) *bytes = s->capacity * s->pitch;
    return OC_OK;
}

OC_API int oc_put_chunks(oc_store* h, const oc_key* keys, const void* payloads, uint64_t n, uint64_t* n_new,
                         uint64_t* bad_index) {
    if (!h) return oc::fail(OC_EINVAL, "put_chunks: null store");
    Store* s = (Store*)h;
    if (n_new) *n_new = 0;
    if (n == 0) return OC_OK;
    if (!keys || !payloads) return oc::fail(OC_EINVAL, "put_chunks: null keys or payloads");
    if (s->read_only) return oc::fail(OC_EINVAL, "put_chunks: store is a read-only imported peer");
    oc::DeviceGuard dg(s->device);
    std::unique_lock<std::shared_mutex> lk(s->mu);
    const uint64_t cb = s->geo.chunk;
    const uint8_t* src = (const uint8_t*)payloads;
    uint64_t fresh = 0;
    // put_stream is non-blocking: order its copies after the legacy stream's work (the usual
    // producer of device payloads), which an event recorded there captures.
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, payloads) == cudaSuccess && pa.type == cudaMemoryTypeDevice) {
        cudaEvent_t ev;
        OC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        cudaError_t e = cudaEventRecord(ev, cudaStreamLegacy);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s->put_stream, ev, 0);
        cudaEventDestroy(ev);
        if (e != cudaSuccess) return oc::cuda_fail(e, "put_chunks: ordering after the producer");
    }
    cudaGetLastError();
    std::vector<uint8_t> a, b;
    for (uint64_t i = 0; i < n; i++) {
        auto it = s->index.find(keys[i]);
        if (it != s->index.end()) {
            // Existing key: identical bytes deduplicate, different bytes violate immutability.
            // The slot may still be in flight from an offload on another stream: wait for those.
            for (cudaEvent_t ev : s->offload_evs) {
                OC_CUDA(cudaEventSynchronize(ev));
                cudaEventDestroy(ev);
            }
            s->offload_evs.clear();
            OC_CUDA(cudaStreamSynchronize(s->put_stream));
            a.resize(cb);
            b.resize(cb);
            OC_CUDA(cudaMemcpy(a.data(), s->slab + it->second * s->pitch, cb, cudaMemcpyDefault));
            OC_CUDA(cudaMemcpy(b.data(), src + i * cb, cb, cudaMemcpyDefault));
            if (std::memcmp(a.data(), b.data(), cb) != 0) {
                if (bad_index) *bad_index = i;
                if (n_new) *n_new = fresh;
                return oc::fail(OC_EIMMUTABLE, "put_chunks: key " + std::to_string(i) +
                                                   " already stored with different bytes");
            }
            continue;
        }
        if (s->count >= s->capacity) {
            cudaStreamSynchronize(s->put_stream);
            if (bad_index) *bad_index = i;
            if (n_new) *n_new = fresh;
            return oc::fail(OC_EFULL, "put_chunks: store capacity exhausted");
        }
        uint64_t slot = s->count;
        OC_CUDA(cudaMemcpyAsync(s->slab + slot * s->pitch, src + i * cb, cb, cudaMemcpyDefault, s->put_stream));
        if (s->hot_layers) {  // the chunk's first layers are its first hot_layers * S bytes
            const uint64_t hb = (uint64_t)s->hot_layers * s->geo.S;
            OC_CUDA(cudaMemcpyAsync(s->hot_slab + slot * hb, src + i * cb, hb, cudaMemcpyDefault, s->put_stream));
        }
        s->index.emplace(keys[i], slot);
        s->count++;
        fresh++;
    }
    OC_CUDA(cudaStreamSynchronize(s->put_stream));
    if (n_new) *n_new = fresh;
    return OC_OK;
}

OC_API int oc_match_prefix(oc_store* h, const uint32_t* tokens, uint64_t n_tokens, const oc_key* parent,
                           oc_key* out, uint64_t cap, uint64_t* n_matched) {
    if (!h || !n_matched || (!tokens && n_tokens)) return oc::fail(OC_EINVAL, "match_prefix: null pointer");
    Store* s = (Store*)h;
    const uint32_t G = s->geo.G;
    uint8_t prev[32] = {0};
    if (parent) std::memcpy(prev, parent->b, 32);
    uint64_t blocks = n_tokens / G, m = 0;
    oc_key k;
    uint64_t addr;
    for (uint64_t i = 0; i < blocks; i++) {
        oc::chunk_key(prev, tokens + i * G, G, k.b);
        if (!oc::store_resolve(s, k, &addr)) break;
        if (m < cap && out) out[m] = k;
        m++;
        std::memcpy(prev, k.b, 32);
    }
    *n_matched = m;
    if (m > cap) return oc::fail(OC_ERANGE, "match_prefix: output capacity smaller than the match");
    return OC_OK;
}

OC_API int oc_store_lookup(oc_store* h, const oc_key* keys, uint64_t n, uint64_t* addrs, uint64_t* bad_index) {
    if (!h || (!keys && n) || (!addrs && n)) return oc::fail(OC_EINVAL, "store_lookup: null pointer");
    Store* s = (Store*)h;
    for (uint64_t i = 0; i < n; i++) {
        if (!oc::store_resolve(s, keys[i], &addrs[i])) {
            if (bad_index) *bad_index = i;
            return oc::fail(OC_ENOTFOUND, "store_lookup: key " + std::to_string(i) + " not found");
        }
    }
    return OC_OK;
}

OC_API int oc_store_attach_peer(oc_store* h, oc_store* peer_h) {
    if (!h || !peer_h || h == peer_h) return oc::fail(OC_EINVAL, "attach_peer: bad store");
    Store* s = (Store*)h;
    Store* p = (Store*)peer_h;
    if (!oc::same_layout(s->layout, p->layout)) return oc::fail(OC_EINVAL, "attach_peer: layouts differ");
    // A cycle (A -> B -> ... -> A) would make every key miss recurse forever.
    if (oc::reaches(p, s)) return oc::fail(OC_EINVAL, "attach_peer: would close a cycle of attached stores");
    if (p->tier == OC_TIER_HBM && p->device != s->device) {
        int ok = 0;
        OC_CUDA(cudaDeviceCanAccessPeer(&ok, s->device, p->device));
        if (!ok) return oc::fail(OC_ENOTSUP, "attach_peer: no peer access between the two GPUs");
        oc::DeviceGuard dg(s->device);
        cudaError_t e = cudaDeviceEnablePeerAccess(p->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return oc::cuda_fail(e, "enable peer access");
        cudaGetLastError();
    }
    std::unique_lock<std::shared_mutex> lk(s->mu);
    s->peers.push_back(p);
    return OC_OK;
}

OC_API int oc_store_export(oc_store* h, void* buf, uint64_t* size) {
    if (!h || !size) return oc::fail(OC_EINVAL, "store_export: null pointer");
    Store* s = (Store*)h;
    if (s->tier != OC_TIER_HBM || s->ipc_mapped) return oc::fail(OC_ENOTSUP, "store_export: only local HBM stores");
    std::shared_lock<std::shared_mutex> lk(s->mu);
    uint64_t need = sizeof(oc::ExportHeader) + s->count * (32 + 8);
    if (!buf) { *size = need; return OC_OK; }
    if (*size < need) { *size = need; return oc::fail(OC_ERANGE, "store_export: buffer too small"); }
    oc::ExportHeader hd{};
    hd.magic = oc::kExportMagic;
    hd.version = OC_ABI_VERSION;
    hd.layout = s->layout;
    hd.tier = s->tier;
    hd.capacity = s->capacity;
    hd.count = s->count;
    hd.pitch = s->pitch;
    {
        oc::DeviceGuard dg(s->device);
        OC_CUDA(cudaIpcGetMemHandle(&hd.handle, s->slab));
    }
    uint8_t* o = (uint8_t*)buf;
    std::memcpy(o, &hd, sizeof hd);
    o += sizeof hd;
    for (auto& kv : s->index) {
        std::memcpy(o, kv.first.b, 32);
        std::memcpy(o + 32, &kv.second, 8);
        o += 40;
    }
    *size = need;
    return OC_OK;
}

OC_API int oc_store_import(const void* buf, uint64_t size, int device, oc_store** out) {
    if (!buf || !out || size < sizeof(oc::ExportHeader)) return oc::fail(OC_EINVAL, "store_import: bad blob");
    *out = nullptr;
    oc::ExportHeader hd;
    std::memcpy(&hd, buf, sizeof hd);
    if (hd.magic != oc::kExportMagic || hd.version != OC_ABI_VERSION)
        return oc::fail(OC_EINVAL, "store_import: not an objcache export blob");
    if (hd.count > (size - sizeof hd) / 40 || hd.count > hd.capacity)
        return oc::fail(OC_EINVAL, "store_import: truncated or corrupt blob");
    if (hd.tier != OC_TIER_HBM) return oc::fail(OC_EINVAL, "store_import: only HBM stores are exported");
    auto s = std::make_unique<Store>();
    int rc = oc::make_geometry(&hd.layout, &s->geo);
    if (rc) return rc;
    if (hd.pitch < s->geo.chunk || hd.pitch % 16) return oc::fail(OC_EINVAL, "store_import: corrupt slot pitch");
    s->pitch = hd.pitch;
    s->layout = hd.layout;
    s->tier = hd.tier;
    s->device = device;
    s->capacity = hd.capacity;
    s->count = hd.count;
    s->owns_slab = false;
    s->read_only = true;
    // Parse and validate the key table before mapping anything.
    const uint8_t* in = (const uint8_t*)buf + sizeof hd;
    s->index.reserve(hd.count * 2);
    for (uint64_t i = 0; i < hd.count; i++, in += 40) {
        oc_key k;
        uint64_t slot;
        std::memcpy(k.b, in, 32);
        std::memcpy(&slot, in + 32, 8);
        if (slot >= hd.capacity) return oc::fail(OC_EINVAL, "store_import: corrupt slot index");
        s->index.emplace(k, slot);
    }
    {
        oc::DeviceGuard dg(device);
        void* p = nullptr;
        OC_CUDA(cudaIpcOpenMemHandle(&p, hd.handle, cudaIpcMemLazyEnablePeerAccess));
        // the blob's capacity x pitch must lie inside the mapped slab (a corrupt or foreign blob
        // would otherwise send fetches past its end)
        const uint64_t have = oc::mapped_bytes(p);
        if (have && (unsigned __int128)hd.capacity * hd.pitch > have) {
            cudaIpcCloseMemHandle(p);
            return oc::fail(OC_EINVAL, "store_import: capacity x slot pitch exceeds the mapped slab");
        }
        s->slab = (uint8_t*)p;
        s->ipc_mapped = true;
    }
    *out = (oc_store*)s.release();
    return OC_OK;
}

}  // extern "C"
