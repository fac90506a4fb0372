// Errors, geometry (Eq. 1), the Eq. 2 mode rule, fast division and driver entry points.
#include <cstdlib>
#include <cuda.h>

#include "oc_internal.h"

namespace oc {

namespace {
thread_local std::string g_last_error;
}

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    cudaGetLastError();  // clear the sticky-free error state
    return OC_ECUDA;
}

// Eq. 1: row = n_kv*d*p, S = 2*G*row, chunk = L*S.
int make_geometry(const oc_layout* lay, Geometry* g) {
    if (!lay) return fail(OC_EINVAL, "null layout");
    if (!lay->num_layers || !lay->kv_heads || !lay->head_dim || !lay->elem_bytes || !lay->chunk_tokens)
        return fail(OC_EINVAL, "layout fields must all be >= 1");
    g->L = lay->num_layers; g->n_kv = lay->kv_heads; g->d = lay->head_dim;
    g->p = lay->elem_bytes; g->G = lay->chunk_tokens;
    unsigned __int128 row = (unsigned __int128)g->n_kv * g->d * g->p;
    unsigned __int128 S = row * 2 * g->G;
    unsigned __int128 chunk = S * g->L;
    if (chunk >> 62) return fail(OC_EINVAL, "layout too large (L*S overflows)");
    g->row = (uint64_t)row;
    g->hd = (uint64_t)g->d * g->p;
    g->S = (uint64_t)S;
    g->chunk = (uint64_t)chunk;
    return OC_OK;
}

bool same_layout(const oc_layout& a, const oc_layout& b) {
    return a.num_layers == b.num_layers && a.kv_heads == b.kv_heads && a.head_dim == b.head_dim &&
           a.elem_bytes == b.elem_bytes && a.chunk_tokens == b.chunk_tokens;
}

FastDiv make_fastdiv(uint32_t d) {
    FastDiv f;
    f.d = d ? d : 1;
    uint32_t s = 0;
    while ((1ull << s) < f.d) s++;
    f.s = s;
    f.m = (uint32_t)((((1ull << 32) * ((1ull << s) - f.d)) / f.d) + 1);
    return f;
}

int device_sm_count(int device) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

namespace {
typedef CUresult (*PFN_wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
std::once_flag g_wait_once;
PFN_wait32 g_wait32 = nullptr;
}  // namespace

// cuStreamWaitValue32(stream, addr, value, GEQ): the consumer stream stalls in the GPU front end
// until (int32_t)(*addr - value) >= 0.  Resolved through the runtime so the library needs no
// link-time libcuda (it must load on a machine without a driver).
int stream_wait_geq(cudaStream_t s, uint32_t* addr, uint32_t value) {
    std::call_once(g_wait_once, [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &fn, 12000, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_wait32 = (PFN_wait32)fn;
        cudaGetLastError();
    });
    if (!g_wait32) return fail(OC_ECUDA, "cuStreamWaitValue32 entry point unavailable");
    CUresult r = g_wait32((CUstream)s, (CUdeviceptr)addr, value, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) return fail(OC_ECUDA, "cuStreamWaitValue32 failed: CUresult " + std::to_string((int)r));
    return OC_OK;
}

}  // namespace oc

namespace oc {
// Slot pitch of a store slab (profiles/r02_stride_probe.txt, r02_pitch_sweep.txt).  A layer of a
// request reads one S-byte slice from each of its chunks' slots, i.e. N slices spaced by the slot
// pitch.  On B200 the HBM read rate of that pattern depends on the spacing: counted in 32 KiB
// granules, multiples of 5 read at 4.9-6.6 TB/s (160 = 5 MiB: 6.23; 180: 4.95; 90: 5.84), multiples
// of 3 at 6.52-6.72, most others at 6.7-6.8 like randomly placed slices; 161 = 7 * 23 read at 6.66
// (98, 112, 196 at 6.79-6.80: a factor 7 is not always slow).  So an HBM slab of chunks of >= 1 MiB
// spaces its slots by the smallest multiple of 32 KiB >= L*S whose granule count has no factor 3, 5
// or 7 (Llama-3-70B: 163 granules, +1.9%; powers of two, e.g. Llama-3-8B's 2 MiB, stay dense).
// Pinned-host slabs are PCIe-bound and keep dense slots (the copy engine reads runs of consecutive
// slots as one strided transfer of pitch L*S).
uint64_t slot_pitch(const Geometry& g, int tier) {
    constexpr uint64_t q = 32768;
    if (tier != OC_TIER_HBM || g.chunk < (1ull << 20)) return g.chunk;
    // OC_SLOT_PITCH_KIB: sweep override (a multiple of 32 >= L*S/1024; ignored otherwise)
    if (const char* e = std::getenv("OC_SLOT_PITCH_KIB")) {
        const uint64_t v = std::strtoull(e, nullptr, 10) << 10;
        if (v >= g.chunk && v % q == 0) return v;
    }
    uint64_t u = (g.chunk + q - 1) / q;
    while (u % 3 == 0 || u % 5 == 0 || u % 7 == 0) u++;
    return u * q;
}
}  // namespace oc

extern "C" {

OC_API const char* oc_last_error(void) { return oc::g_last_error.c_str(); }

OC_API const char* oc_status_str(int st) {
    switch (st) {
        case OC_OK: return "OC_OK";
        case OC_EINVAL: return "OC_EINVAL";
        case OC_ENOMEM: return "OC_ENOMEM";
        case OC_ENOTFOUND: return "OC_ENOTFOUND";
        case OC_EIMMUTABLE: return "OC_EIMMUTABLE";
        case OC_ERANGE: return "OC_ERANGE";
        case OC_EALIGN: return "OC_EALIGN";
        case OC_ECUDA: return "OC_ECUDA";
        case OC_EFULL: return "OC_EFULL";
        case OC_ENOTSUP: return "OC_ENOTSUP";
        default: return "OC_E?";
    }
}

OC_API int oc_abi_version(void) { return OC_ABI_VERSION; }

OC_API int oc_geometry(const oc_layout* layout, uint64_t* row_bytes, uint64_t* layer_chunk_bytes,
                       uint64_t* chunk_bytes) {
    oc::Geometry g;
    int rc = oc::make_geometry(layout, &g);
    if (rc) return rc;
    if (row_bytes) *row_bytes = g.row;
    if (layer_chunk_bytes) *layer_chunk_bytes = g.S;
    if (chunk_bytes) *chunk_bytes = g.chunk;
    return OC_OK;
}

OC_API int oc_slot_pitch(const oc_layout* layout, int tier, uint64_t* pitch) {
    if (!pitch) return oc::fail(OC_EINVAL, "slot_pitch: null out");
    oc::Geometry g;
    int rc = oc::make_geometry(layout, &g);
    if (rc) return rc;
    if (tier != OC_TIER_HBM && tier != OC_TIER_PINNED_HOST) return oc::fail(OC_EINVAL, "slot_pitch: bad tier");
    *pitch = oc::slot_pitch(g, tier);
    return OC_OK;
}

// Eq. 2: chunkwise if W < Theta, else layerwise + aggregation.
OC_API int oc_select_mode(uint64_t payload_W, uint64_t theta) {
    return payload_W < theta ? OC_DELIVER_CHUNK_MAJOR : OC_DELIVER_LAYER_MAJOR;
}

}  // extern "C"
