// Pooled device and pinned-host memory for descriptors and batches.
//
// cudaMalloc/cudaFree per request cost 0.3-8 ms on B200 (cudaFree synchronises the device), and
// cudaHostAlloc is slower still, which would dominate the control plane of a 4K-token fetch.
// Blocks are power-of-two sized (>= 4 KiB), kept per device (device -1 = pinned host memory) and
// recycled; they are never returned to the driver.
#include "oc_internal.h"

namespace oc {
namespace {

struct Pool {
    std::mutex mu;
    std::unordered_map<uint64_t, std::vector<void*>> free_by_class;  // key: ((device + 1) << 48) | class
};
Pool g_pool;

uint64_t size_class(size_t n) {
    uint64_t c = 4096;
    while (c < n) c <<= 1;
    return c;
}

uint64_t key_of(int device, uint64_t cls) { return ((uint64_t)(device + 1) << 48) | cls; }

}  // namespace

void* dev_pool_alloc(int device, size_t n, uint64_t* cls_out) {
    const uint64_t cls = size_class(n);
    *cls_out = cls;
    {
        std::lock_guard<std::mutex> lk(g_pool.mu);
        auto& fl = g_pool.free_by_class[key_of(device, cls)];
        if (!fl.empty()) {
            void* p = fl.back();
            fl.pop_back();
            return p;
        }
    }
    void* p = nullptr;
    cudaError_t e = device < 0 ? cudaHostAlloc(&p, cls, cudaHostAllocPortable) : cudaMalloc(&p, cls);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void dev_pool_free(int device, void* p, uint64_t cls) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pool.mu);
    g_pool.free_by_class[key_of(device, cls)].push_back(p);
}

namespace {
std::mutex g_mirror_mu;
std::vector<uint32_t*> g_mirror_free;
constexpr size_t kMirrorLine = 64, kMirrorSlab = 64 * 1024;
}  // namespace

uint32_t* ready_mirror_alloc() {
    std::lock_guard<std::mutex> lk(g_mirror_mu);
    if (g_mirror_free.empty()) {
        void* p = nullptr;
        if (cudaHostAlloc(&p, kMirrorSlab, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        for (size_t o = kMirrorSlab; o >= kMirrorLine; o -= kMirrorLine)
            g_mirror_free.push_back((uint32_t*)((uint8_t*)p + o - kMirrorLine));
    }
    uint32_t* w = g_mirror_free.back();
    g_mirror_free.pop_back();
    __atomic_store_n(w, 0u, __ATOMIC_RELEASE);
    return w;
}

void ready_mirror_free(uint32_t* w) {
    if (!w) return;
    std::lock_guard<std::mutex> lk(g_mirror_mu);
    g_mirror_free.push_back(w);
}

}  // namespace oc
