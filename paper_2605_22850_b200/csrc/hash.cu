// Chunk keys on the GPU for a batch of token streams: H_i = SHA-256(H_{i-1} || LE-u32 tokens_i),
// root = 32 zero bytes (Sec. 2.1; reading c1).  The offload path names new
// chunks by these keys ("newly produced KV blocks are offloaded back to object storage");
// SURVEY 8(f)3 lists GPU-side chain hashing as its optional part.
//
// A chain is sequential (H_i needs H_{i-1}), so one thread hashes one request's chain; requests
// are independent, so a batch of R requests runs R chains at once.  One key hashes 32 + 4G bytes
// (2 compression blocks at G = 16).  A single chain is slower than the host's SHA extensions,
// but a batch of hundreds of requests -- an admission step of config 5 -- is not.
#include "oc_internal.h"

namespace oc {
namespace {

__constant__ uint32_t kK[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

__device__ __forceinline__ uint32_t rotr(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

// FIPS 180-4 compression of one 16-word (big-endian) block into h[8].
__device__ void compress(uint32_t h[8], const uint32_t blk[16]) {
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 16; i++) w[i] = blk[i];
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
#pragma unroll
    for (int i = 0; i < 64; i++) {
        uint32_t wi;
        if (i < 16) {
            wi = w[i];
        } else {
            const uint32_t w15 = w[(i - 15) & 15], w2 = w[(i - 2) & 15];
            const uint32_t s0 = rotr(w15, 7) ^ rotr(w15, 18) ^ (w15 >> 3);
            const uint32_t s1 = rotr(w2, 17) ^ rotr(w2, 19) ^ (w2 >> 10);
            wi = w[i & 15] = w[i & 15] + s0 + w[(i - 7) & 15] + s1;
        }
        const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t t1 = hh + S1 + ch + kK[i] + wi;
        const uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        const uint32_t maj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t t2 = S0 + maj;
        hh = g;
        g = f;
        f = e;
        e = d + t1;
        d = c;
        c = b;
        b = a;
        a = t1 + t2;
    }
    h[0] += a;
    h[1] += b;
    h[2] += c;
    h[3] += d;
    h[4] += e;
    h[5] += f;
    h[6] += g;
    h[7] += hh;
}

// Request r: its tokens, its keys, its parent; one thread per chain.
__global__ void chain_keys_kernel(const uint32_t* __restrict__ tokens, const uint64_t* __restrict__ tok_off,
                                  const uint64_t* __restrict__ n_tokens, uint32_t n_req, uint32_t G,
                                  const uint8_t* __restrict__ parents, uint8_t* __restrict__ out,
                                  const uint64_t* __restrict__ key_off) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_req) return;
    const uint32_t* tok = tokens + tok_off[r];
    const uint64_t nkeys = n_tokens[r] / G;
    uint32_t* dst = (uint32_t*)(out + key_off[r] * 32);
    uint32_t prev[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        uint32_t v = 0;
        if (parents) {  // digest bytes -> big-endian words
            const uint8_t* p = parents + (uint64_t)r * 32 + 4 * i;
            v = ((uint32_t)p[0] << 24) | ((uint32_t)p[1] << 16) | ((uint32_t)p[2] << 8) | p[3];
        }
        prev[i] = v;
    }
    if (G == 16) {  // the default chunk size: two blocks per key, next key's tokens loaded ahead
        uint32_t t[16];
#pragma unroll
        for (int i = 0; i < 16; i++) t[i] = nkeys ? __ldg(&tok[i]) : 0u;
        for (uint64_t k = 0; k < nkeys; k++) {
            uint32_t nt[16];
            const bool more = k + 1 < nkeys;
#pragma unroll
            for (int i = 0; i < 16; i++) nt[i] = more ? __ldg(&tok[(k + 1) * 16 + i]) : 0u;
            uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
            uint32_t blk[16];
#pragma unroll
            for (int i = 0; i < 8; i++) {
                blk[i] = prev[i];
                blk[8 + i] = __byte_perm(t[i], 0, 0x0123);
            }
            compress(h, blk);
#pragma unroll
            for (int i = 0; i < 8; i++) blk[i] = __byte_perm(t[8 + i], 0, 0x0123);
            blk[8] = 0x80000000u;
#pragma unroll
            for (int i = 9; i < 15; i++) blk[i] = 0;
            blk[15] = (8 + 16) * 32;  // message bits: 32-byte digest + 16 tokens
            compress(h, blk);
#pragma unroll
            for (int i = 0; i < 8; i++) {
                prev[i] = h[i];
                dst[k * 8 + i] = __byte_perm(h[i], 0, 0x0123);
            }
#pragma unroll
            for (int i = 0; i < 16; i++) t[i] = nt[i];
        }
        return;
    }
    const uint64_t msg_words = 8 + (uint64_t)G;       // prev digest, then G tokens
    const uint64_t bits = msg_words * 32;
    const uint64_t total = ((msg_words + 1 + 2 + 15) / 16) * 16;  // + 0x80 word + 64-bit length
    for (uint64_t k = 0; k < nkeys; k++) {
        uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
        uint32_t blk[16];
        const uint32_t* tk = tok + k * G;
        for (uint64_t w0 = 0; w0 < total; w0 += 16) {
#pragma unroll
            for (int i = 0; i < 16; i++) {
                const uint64_t wi = w0 + i;
                uint32_t v;
                if (wi < 8) v = prev[wi];
                else if (wi < msg_words) v = __byte_perm(__ldg(&tk[wi - 8]), 0, 0x0123);  // LE token -> BE word
                else if (wi == msg_words) v = 0x80000000u;
                else if (wi == total - 2) v = (uint32_t)(bits >> 32);
                else if (wi == total - 1) v = (uint32_t)bits;
                else v = 0;
                blk[i] = v;
            }
            compress(h, blk);
        }
#pragma unroll
        for (int i = 0; i < 8; i++) {
            prev[i] = h[i];
            dst[k * 8 + i] = __byte_perm(h[i], 0, 0x0123);  // big-endian bytes of the digest
        }
    }
}

}  // namespace
}  // namespace oc

extern "C" OC_API int oc_chunk_keys_batch(const uint32_t* tokens, const uint64_t* tok_off, const uint64_t* n_tokens,
                                          uint32_t n_requests, uint32_t chunk_tokens, const oc_key* parents, oc_key* out,
                                          const uint64_t* key_off, void* stream) {
    if (chunk_tokens == 0) return oc::fail(OC_EINVAL, "chunk_keys_batch: chunk_tokens must be >= 1");
    if (n_requests == 0) return OC_OK;
    if (!tokens || !tok_off || !n_tokens || !out || !key_off) return oc::fail(OC_EINVAL, "chunk_keys_batch: null pointer");
    const uint32_t threads = 64;
    oc::chain_keys_kernel<<<(n_requests + threads - 1) / threads, threads, 0, (cudaStream_t)stream>>>(
        tokens, tok_off, n_tokens, n_requests, chunk_tokens, (const uint8_t*)parents, (uint8_t*)out, key_off);
    OC_CUDA(cudaGetLastError());
    return OC_OK;
}
