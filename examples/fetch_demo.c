/*
 * fetch_demo.c -- the serving node's call order (match -> descriptor ->
 * layer-ready waits) through the plain C ABI of libobjcache, with no Python involved.
 *
 *   1. put_chunks: a 4-layer toy model's KV for a 100-token prompt (6 complete 16-token chunks)
 *      goes into an HBM chunk store under its SHA-256 chain keys;
 *   2. match_prefix: a new request that shares the first 80 tokens matches 5 chunks;
 *   3. build_descriptor: those chunks, delivered layer-major into a vLLM-style paged KV cache
 *      (block size 16, a scrambled block table, the prefix starting at token 0);
 *   4. fetch_layerwise on a copy stream, wait_layer(l) on a consumer stream for every layer;
 *   5. the cache is read back and every delivered row is compared with the definition
 *      (row t of matrix kv of layer l of chunk j = bytes [l*S + kv*G*row + t*row, +row) of the
 *      chunk object, KV_L2TD); bytes outside the prefix must keep their sentinel.
 *
 * Build: gcc -O2 -I include examples/fetch_demo.c -L paper_2605_22850_b200 -lobjcache \
 *            -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,... -o fetch_demo
 * Exit status 0 = every byte as defined; 1 = mismatch; 2 = a call failed (message printed).
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "objcache.h"

#define CHECK(call)                                                                     \
    do {                                                                                \
        int rc_ = (call);                                                               \
        if (rc_ != OC_OK) {                                                             \
            fprintf(stderr, "%s failed: %s (%s)\n", #call, oc_status_str(rc_), oc_last_error()); \
            return 2;                                                                   \
        }                                                                               \
    } while (0)

#define CUDA(call)                                                                      \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            fprintf(stderr, "%s failed: %s\n", #call, cudaGetErrorString(e_));          \
            return 2;                                                                   \
        }                                                                               \
    } while (0)

static uint8_t chunk_byte(uint64_t chunk, uint64_t off) {  /* deterministic payload */
    uint64_t x = chunk * 0x9E3779B97F4A7C15ull + off * 0xBF58476D1CE4E5B9ull;
    x ^= x >> 31;
    return (uint8_t)(x * 0x94D049BB133111EBull >> 56);
}

int main(void) {
    const oc_layout lay = {4, 2, 64, 2, 16};  /* L, n_kv, d, p, G */
    uint64_t row, S, chunk;
    CHECK(oc_geometry(&lay, &row, &S, &chunk));
    const uint32_t G = lay.chunk_tokens, L = lay.num_layers;

    /* 1. the prompt's KV, chunk-major, under its chain keys */
    uint32_t prompt[100];
    for (int i = 0; i < 100; i++) prompt[i] = 1000u + 7u * (uint32_t)i;
    oc_key keys[8];
    uint64_t n_keys = 0;
    CHECK(oc_chunk_keys(prompt, 100, G, NULL, keys, 8, &n_keys));
    uint8_t* payload = (uint8_t*)malloc(n_keys * chunk);
    for (uint64_t j = 0; j < n_keys; j++)
        for (uint64_t o = 0; o < chunk; o++) payload[j * chunk + o] = chunk_byte(j, o);
    oc_store* store = NULL;
    CHECK(oc_store_create(&lay, OC_TIER_HBM, 0, 16, &store));
    uint64_t n_new = 0, bad = 0;
    CHECK(oc_put_chunks(store, keys, payload, n_keys, &n_new, &bad));

    /* 2. a request sharing the first 80 tokens */
    uint32_t query[120];
    for (int i = 0; i < 120; i++) query[i] = i < 80 ? prompt[i] : 5u + (uint32_t)i;
    oc_key hit[8];
    uint64_t n_hit = 0;
    CHECK(oc_match_prefix(store, query, 120, NULL, hit, 8, &n_hit));
    if (n_hit != 5) {
        fprintf(stderr, "match_prefix: %llu chunks, expected 5\n", (unsigned long long)n_hit);
        return 1;
    }

    /* 3. a paged cache [L][2][blocks][Bs][row] and a scrambled block table */
    const uint32_t Bs = 16, blocks = 9;
    const int32_t table[5] = {7, 2, 5, 0, 8};
    const uint64_t per_kv = (uint64_t)blocks * Bs * row, bytes = L * 2 * per_kv;
    uint8_t* cache = NULL;
    CUDA(cudaMalloc((void**)&cache, bytes));
    CUDA(cudaMemset(cache, 0xA5, bytes));
    uint64_t kb[4], vb[4];
    for (uint32_t l = 0; l < L; l++) {
        kb[l] = (uint64_t)(uintptr_t)cache + l * 2 * per_kv;
        vb[l] = kb[l] + per_kv;
    }
    oc_target t;
    memset(&t, 0, sizeof t);
    t.kind = OC_TARGET_PAGED;
    t.block_size = Bs;
    t.k_base = kb;
    t.v_base = vb;
    t.block_stride = Bs * row;
    t.token_stride = row;
    t.head_stride = lay.head_dim * lay.elem_bytes;
    t.block_table = table;
    t.num_blocks = 5;
    oc_desc* desc = NULL;
    CHECK(oc_build_descriptor(store, hit, n_hit, &lay, OC_DELIVER_LAYER_MAJOR, &t, &desc, &bad));

    /* 4. fetch on a copy stream; the consumer waits layer by layer (prefill would run here) */
    cudaStream_t copy_s, cons_s;
    CUDA(cudaStreamCreateWithFlags(&copy_s, cudaStreamNonBlocking));
    CUDA(cudaStreamCreateWithFlags(&cons_s, cudaStreamNonBlocking));
    CHECK(oc_fetch_layerwise(desc, NULL, copy_s));
    for (uint32_t l = 0; l < L; l++) CHECK(oc_wait_layer(desc, l, cons_s));
    CUDA(cudaStreamSynchronize(cons_s));

    /* 5. check every byte */
    uint8_t* host = (uint8_t*)malloc(bytes);
    CUDA(cudaMemcpy(host, cache, bytes, cudaMemcpyDeviceToHost));
    uint64_t wrong = 0, touched = 0;
    for (uint32_t l = 0; l < L; l++)
        for (uint32_t kv = 0; kv < 2; kv++)
            for (uint32_t b = 0; b < blocks; b++)
                for (uint32_t slot = 0; slot < Bs; slot++) {
                    const uint8_t* got = host + l * 2 * per_kv + kv * per_kv + ((uint64_t)b * Bs + slot) * row;
                    int pos = -1;  /* which prefix token, if any, lives in (b, slot) */
                    for (int i = 0; i < 5; i++)
                        if ((uint32_t)table[i] == b) pos = i * (int)Bs + (int)slot;
                    for (uint64_t o = 0; o < row; o++) {
                        uint8_t want = 0xA5;
                        if (pos >= 0) {
                            const uint64_t j = (uint64_t)pos / G, tok = (uint64_t)pos % G;
                            want = chunk_byte(j, l * S + kv * G * row + tok * row + o);
                        }
                        wrong += got[o] != want;
                    }
                    touched += pos >= 0;
                }
    printf("fetch_demo: matched %llu chunks, %llu rows delivered over %u layers, %llu wrong bytes\n",
           (unsigned long long)n_hit, (unsigned long long)touched, L, (unsigned long long)wrong);
    CHECK(oc_desc_free(desc));
    CHECK(oc_store_destroy(store));
    cudaFree(cache);
    free(host);
    free(payload);
    return wrong == 0 ? 0 : 1;
}
