// Probe: one layer of a 64K hit (N = 3584 chunks of L*S = 2 MiB, S = 64 KiB) moved from an HBM
// chunk store into a flat layer-major buffer B_l by ONE strided copy-engine transfer
// (cudaMemcpy2DAsync: width S, height N, source pitch L*S, destination pitch S).  Measures its rate
// alone, whether it progresses while a kernel holds every SM's thread slots (copy engine, not SMs),
// and how much it slows an FMA-bound kernel running at the same time.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a ce_d2d_probe.cu -o /tmp/ce_d2d
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <chrono>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("ERR %s line %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__global__ void spin_kernel(long long ns, float* sink) {
    long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    float a = threadIdx.x;
    for (;;) {
        for (int i = 0; i < 64; i++) a = a * 1.0001f + 0.5f;
        long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > ns) break;
    }
    if (a == 1234.5f) sink[0] = a;
}

__global__ void fma_kernel(int iters, float* out) {
    float a = threadIdx.x, b = blockIdx.x, c = 1.0f, d = 2.0f;
    for (int i = 0; i < iters; i++) { a = a * 0.999f + b; b = b * 0.999f + c; c = c * 0.999f + d; d = d * 0.999f + a; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}

// a memory-heavy kernel: streams a buffer (read) -- how much does a concurrent CE copy slow it
__global__ void stream_kernel(const int4* __restrict__ a, int4* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main(int argc, char** argv) {
    const size_t N = argc > 1 ? atol(argv[1]) : 3584, L = 32, S = 65536, chunk = L * S;
    const int layers = argc > 2 ? atoi(argv[2]) : 8;
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    uint8_t *src, *dst; float* sink;
    CK(cudaMalloc(&src, N * chunk));
    CK(cudaMalloc(&dst, (size_t)layers * N * S));
    CK(cudaMalloc(&sink, 1 << 24));
    CK(cudaMemset(src, 1, N * chunk));
    cudaStream_t s, a; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
    cudaEvent_t e0, e1, e2, el[64];
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1)); CK(cudaEventCreate(&e2));
    for (int l = 0; l < layers; l++) CK(cudaEventCreate(&el[l]));
    const double bytes_layer = 2.0 * N * S;
    auto layer_copy = [&](int l, cudaStream_t st) {
        CK(cudaMemcpy2DAsync(dst + (size_t)l * N * S, S, src + (size_t)l * S, chunk, S, N, cudaMemcpyDeviceToDevice, st));
    };
    for (int rep = 0; rep < 3; rep++) {
        CK(cudaDeviceSynchronize());
        auto h0 = std::chrono::steady_clock::now();
        CK(cudaEventRecord(e0, s));
        for (int l = 0; l < layers; l++) { layer_copy(l, s); CK(cudaEventRecord(el[l], s)); }
        auto h1 = std::chrono::steady_clock::now();
        CK(cudaEventSynchronize(el[layers - 1]));
        float ms, x0; CK(cudaEventElapsedTime(&ms, e0, el[layers - 1])); CK(cudaEventElapsedTime(&x0, e0, el[0]));
        printf("{\"what\": \"ce 2d per layer, alone\", \"N\": %zu, \"layers\": %d, \"ms\": %.3f, \"X0_ms\": %.3f, \"TBps_rw\": %.3f, \"host_us_per_layer\": %.1f}\n",
               N, layers, ms, x0, bytes_layer * layers / ms / 1e9, std::chrono::duration<double, std::micro>(h1 - h0).count() / layers);
    }
    // one contiguous copy of the same bytes (CE, no stride)
    {
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0, s));
        CK(cudaMemcpyAsync(dst, src, (size_t)layers * N * S, cudaMemcpyDeviceToDevice, s));
        CK(cudaEventRecord(e1, s));
        CK(cudaEventSynchronize(e1));
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("{\"what\": \"contiguous cudaMemcpyAsync of the same bytes\", \"ms\": %.3f, \"TBps_rw\": %.3f}\n", ms, bytes_layer * layers / ms / 1e9);
    }
    // co-run: a 20 ms spin kernel holding every SM's 2048 thread slots on stream a
    for (int rep = 0; rep < 2; rep++) {
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0, a));
        spin_kernel<<<sms * 2, 1024, 0, a>>>(20000000LL, sink);
        CK(cudaEventRecord(e2, a));
        CK(cudaStreamWaitEvent(s, e0, 0));
        for (int l = 0; l < layers; l++) { layer_copy(l, s); CK(cudaEventRecord(el[l], s)); }
        CK(cudaDeviceSynchronize());
        float ms_copy, ms_spin, x0; CK(cudaEventElapsedTime(&ms_copy, e0, el[layers - 1])); CK(cudaEventElapsedTime(&ms_spin, e0, e2));
        CK(cudaEventElapsedTime(&x0, e0, el[0]));
        printf("{\"what\": \"ce 2d with a 20 ms spin on every SM\", \"copy_done_ms\": %.3f, \"X0_ms\": %.3f, \"spin_done_ms\": %.3f, \"copy_TBps_rw\": %.3f}\n",
               ms_copy, x0, ms_spin, bytes_layer * layers / ms_copy / 1e9);
    }
    // slowdown of an FMA-bound kernel and of a streaming kernel by the concurrent copies
    {
        const int iters = 400000;
        float t_alone, t_with, t_cp;
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0, a)); fma_kernel<<<sms * 4, 512, 0, a>>>(iters, sink); CK(cudaEventRecord(e2, a));
        CK(cudaDeviceSynchronize()); CK(cudaEventElapsedTime(&t_alone, e0, e2));
        CK(cudaEventRecord(e0, a)); fma_kernel<<<sms * 4, 512, 0, a>>>(iters, sink); CK(cudaEventRecord(e2, a));
        CK(cudaStreamWaitEvent(s, e0, 0));
        int n = 0;
        for (int r = 0; r < 4; r++) for (int l = 0; l < layers; l++) { layer_copy(l, s); n++; }
        CK(cudaEventRecord(e1, s));
        CK(cudaDeviceSynchronize()); CK(cudaEventElapsedTime(&t_with, e0, e2)); CK(cudaEventElapsedTime(&t_cp, e0, e1));
        printf("{\"what\": \"fma kernel alone vs with concurrent ce copies\", \"alone_ms\": %.3f, \"with_ms\": %.3f, \"copies_ms\": %.3f, \"layers_copied\": %d}\n", t_alone, t_with, t_cp, n);
        const size_t nb = (size_t)4 << 30;
        int4 *x, *y; CK(cudaMalloc(&x, nb)); CK(cudaMalloc(&y, nb));
        CK(cudaMemset(x, 0, nb));
        for (int w = 0; w < 2; w++) {
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(e0, a)); for (int r = 0; r < 4; r++) stream_kernel<<<sms * 4, 512, 0, a>>>(x, y, nb / 16); CK(cudaEventRecord(e2, a));
            if (w) {
                CK(cudaStreamWaitEvent(s, e0, 0));
                for (int l = 0; l < layers; l++) layer_copy(l, s);
                CK(cudaEventRecord(e1, s));
            }
            CK(cudaDeviceSynchronize());
            float t; CK(cudaEventElapsedTime(&t, e0, e2));
            float tc = 0; if (w) CK(cudaEventElapsedTime(&tc, e0, e1));
            printf("{\"what\": \"streaming kernel (4 x 4 GiB copy)\", \"with_ce\": %d, \"ms\": %.3f, \"TBps_rw\": %.3f, \"ce_done_ms\": %.3f}\n", w, t, 4 * 2.0 * nb / t / 1e9, tc);
        }
    }
    return 0;
}
