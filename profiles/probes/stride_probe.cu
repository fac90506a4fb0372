// Probe: is the slot-size effect (r02_slot_size_sweep.txt: 32 KiB-unit fetches from 2.5 / 5 MiB
// slots at 6.2 TB/s, from 2 / 4 / 8 MiB slots at 6.8) a property of the source addresses alone?
// A minimal TMA copy kernel (3 CTAs per SM, one warp, 2-stage 32 KiB ring, units claimed from a
// counter in layer-major order) gathers "layer" slices of 64 KiB from N = 1792 pieces placed at
// offset off(j) = j * X (or a random 64 KiB-aligned offset) into a contiguous buffer.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a stride_probe.cu -o /tmp/stride_probe
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("ERR %s line %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t sm32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32) gather(const uint8_t* __restrict__ base, const uint64_t* __restrict__ off,
                                             uint8_t* __restrict__ out, uint32_t N, uint32_t layers, uint32_t unit,
                                             uint32_t* ctr) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar[2];
    if (threadIdx.x != 0) return;
    const uint32_t per_layer = N * (65536 / unit), total = per_layer * layers;
    for (int i = 0; i < 2; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm32(&bar[i])) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    uint32_t phase[2] = {0, 0};
    auto src_of = [&](uint32_t u) {
        const uint32_t l = u / per_layer, r = u - l * per_layer, j = r / (65536 / unit), h = r % (65536 / unit);
        return base + off[j] + (uint64_t)l * 65536 + (uint64_t)h * unit;
    };
    auto load = [&](uint32_t u, int s) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm32(&bar[s])), "r"(unit) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sm32(smem + (size_t)s * unit)), "l"(src_of(u)), "r"(unit), "r"(sm32(&bar[s])) : "memory");
    };
    int s = 0;
    uint32_t u = atomicAdd(ctr, 1u);
    if (u < total) load(u, 0);
    while (u < total) {
        const uint32_t un = atomicAdd(ctr, 1u);
        if (un < total) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            load(un, s ^ 1);
        }
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                     ::"r"(sm32(&bar[s])), "r"(phase[s]) : "memory");
        phase[s] ^= 1;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(out + (uint64_t)u * unit), "r"(sm32(smem + (size_t)s * unit)), "r"(unit) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        u = un;
        s ^= 1;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
    const uint32_t N = 1792, layers = 8;
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t MiB = 1 << 20, cap = (size_t)15 << 30;
    uint8_t *base, *out; uint64_t* doff; uint32_t* ctr;
    CK(cudaMalloc(&base, cap));
    CK(cudaMalloc(&out, (size_t)N * layers * 65536));
    CK(cudaMalloc(&doff, N * 8));
    CK(cudaMalloc(&ctr, 4));
    CK(cudaMemset(base, 3, cap));
    CK(cudaFuncSetAttribute(gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 65536));
    cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    struct Pat { const char* name; double x_mib; bool random; };
    std::vector<Pat> pats;
    if (argc > 1) {  // strides given in 64 KiB units on the command line (fractions allowed)
        for (int i = 1; i < argc; i++) pats.push_back({"stride", atof(argv[i]) / 16.0, false});
    } else {
        pats = {{"stride", 2, false}, {"stride", 2.0625, false}, {"stride", 2.125, false}, {"stride", 2.5, false},
                {"stride", 3, false}, {"stride", 4, false}, {"stride", 5, false}, {"stride", 5.0625, false},
                {"stride", 5.125, false}, {"stride", 5.25, false}, {"stride", 5.5, false}, {"stride", 6, false},
                {"stride", 8, false}, {"random_64k_aligned", 0, true}, {"random_2mib_aligned", 0, true}};
    }
    std::mt19937_64 rng(7);
    for (uint32_t unit : argc > 1 ? std::vector<uint32_t>{32768u} : std::vector<uint32_t>{32768u, 16384u, 65536u}) {
        for (size_t pi = 0; pi < pats.size(); pi++) {
            const Pat& p = pats[pi];
            std::vector<uint64_t> off(N);
            if (!p.random) {
                for (uint32_t j = 0; j < N; j++) off[j] = (uint64_t)(j * p.x_mib * MiB);
            } else {
                const uint64_t align = p.name[7] == '2' ? 2 * MiB : 65536;
                std::vector<uint64_t> cand((cap - layers * 65536) / align);
                for (size_t i = 0; i < cand.size(); i++) cand[i] = i * align;
                std::shuffle(cand.begin(), cand.end(), rng);
                for (uint32_t j = 0; j < N; j++) off[j] = cand[j];
            }
            if (off[N - 1] + layers * 65536 > cap) continue;
            CK(cudaMemcpy(doff, off.data(), N * 8, cudaMemcpyHostToDevice));
            const uint32_t smem = 2 * unit;
            float best = 1e9;
            for (int rep = 0; rep < 6; rep++) {
                CK(cudaMemset(ctr, 0, 4));
                CK(cudaEventRecord(a));
                gather<<<3 * sms, 32, smem>>>(base, doff, out, N, layers, unit, ctr);
                CK(cudaEventRecord(b));
                CK(cudaEventSynchronize(b));
                float ms; CK(cudaEventElapsedTime(&ms, a, b));
                if (rep >= 2) best = std::min(best, ms);
            }
            printf("{\"unit_KiB\": %u, \"pattern\": \"%s\", \"X_MiB\": %.4f, \"ms\": %.4f, \"TBps_rw\": %.3f}\n", unit / 1024, p.name, p.x_mib,
                   best, 2.0 * N * layers * 65536 / best / 1e9);
        }
    }
    return 0;
}
