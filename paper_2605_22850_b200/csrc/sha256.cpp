// SHA-256 (FIPS 180-4) and the rolling chunk key H_i = SHA-256(H_{i-1} || LE-u32 tokens_i)
// (Sec. 2.1; the paper names only "Hash", reading c1 in DESIGN.md).
#include <cpuid.h>
#include <immintrin.h>

#include "oc_internal.h"

namespace oc {
namespace {

const uint32_t K256[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

inline uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

// x86 SHA extensions (SHA-NI): the same FIPS 180-4 compression, 4 rounds per sha256rnds2 pair.
// The chain keys of a 64K-token prefix are 4096 sequential hashes on the match_prefix critical
// path; SHA-NI makes them ~5x cheaper than the portable rounds.
bool cpu_has_sha_ni() {
    unsigned a, b, c, d;
    if (!__get_cpuid_count(7, 0, &a, &b, &c, &d)) return false;
    return (b >> 29) & 1u;  // CPUID.(EAX=7,ECX=0):EBX.SHA[bit 29]
}
const bool g_sha_ni = cpu_has_sha_ni();

__attribute__((target("sha,sse4.1,ssse3"))) void blocks_sha_ni(uint32_t h[8], const uint8_t* p, size_t nblocks) {
    const __m128i bswap = _mm_set_epi64x(0x0c0d0e0f08090a0bULL, 0x0405060700010203ULL);
    __m128i tmp = _mm_loadu_si128((const __m128i*)&h[0]);
    __m128i st1 = _mm_loadu_si128((const __m128i*)&h[4]);
    tmp = _mm_shuffle_epi32(tmp, 0xB1);      // CDAB
    st1 = _mm_shuffle_epi32(st1, 0x1B);      // EFGH
    __m128i st0 = _mm_alignr_epi8(tmp, st1, 8);  // ABEF
    st1 = _mm_blend_epi16(st1, tmp, 0xF0);       // CDGH
    for (; nblocks; nblocks--, p += 64) {
        const __m128i abef = st0, cdgh = st1;
        __m128i w[16];
        for (int g = 0; g < 16; g++) {
            if (g < 4) {
                w[g] = _mm_shuffle_epi8(_mm_loadu_si128((const __m128i*)(p + 16 * g)), bswap);
            } else {
                __m128i x = _mm_sha256msg1_epu32(w[g - 4], w[g - 3]);
                x = _mm_add_epi32(x, _mm_alignr_epi8(w[g - 1], w[g - 2], 4));
                w[g] = _mm_sha256msg2_epu32(x, w[g - 1]);
            }
            __m128i m = _mm_add_epi32(w[g], _mm_loadu_si128((const __m128i*)&K256[4 * g]));
            st1 = _mm_sha256rnds2_epu32(st1, st0, m);
            m = _mm_shuffle_epi32(m, 0x0E);
            st0 = _mm_sha256rnds2_epu32(st0, st1, m);
        }
        st0 = _mm_add_epi32(st0, abef);
        st1 = _mm_add_epi32(st1, cdgh);
    }
    tmp = _mm_shuffle_epi32(st0, 0x1B);      // FEBA
    st1 = _mm_shuffle_epi32(st1, 0xB1);      // DCHG
    st0 = _mm_blend_epi16(tmp, st1, 0xF0);   // DCBA
    st1 = _mm_alignr_epi8(st1, tmp, 8);      // HGFE
    _mm_storeu_si128((__m128i*)&h[0], st0);
    _mm_storeu_si128((__m128i*)&h[4], st1);
}

struct Sha {
    uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                     0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    uint8_t buf[64];
    size_t fill = 0;
    uint64_t total = 0;

    void block(const uint8_t* p) {
        if (g_sha_ni) {
            blocks_sha_ni(h, p, 1);
            return;
        }
        uint32_t w[64];
        for (int i = 0; i < 16; i++)
            w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 | (uint32_t)p[4 * i + 2] << 8 |
                   (uint32_t)p[4 * i + 3];
        for (int i = 16; i < 64; i++) {
            uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
            uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
            w[i] = w[i - 16] + s0 + w[i - 7] + s1;
        }
        uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
        for (int i = 0; i < 64; i++) {
            uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
            uint32_t ch = (e & f) ^ (~e & g);
            uint32_t t1 = hh + S1 + ch + K256[i] + w[i];
            uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
            uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
            uint32_t t2 = S0 + mj;
            hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
        }
        h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
    }
    void update(const uint8_t* p, size_t n) {
        total += n;
        if (fill) {
            size_t take = std::min(n, 64 - fill);
            std::memcpy(buf + fill, p, take);
            fill += take; p += take; n -= take;
            if (fill == 64) { block(buf); fill = 0; }
        }
        if (n >= 64 && g_sha_ni) {
            blocks_sha_ni(h, p, n / 64);
            p += n & ~size_t(63);
            n &= 63;
        }
        while (n >= 64) { block(p); p += 64; n -= 64; }
        if (n) { std::memcpy(buf, p, n); fill = n; }
    }
    void finish(uint8_t out[32]) {
        // padding: 0x80, zeros up to 56 mod 64, then the 64-bit big-endian bit length
        const uint64_t bits = total * 8;
        uint8_t pad[72] = {0x80};
        const size_t zeros = (fill < 56 ? 56 - fill : 120 - fill) - 1;
        for (int i = 0; i < 8; i++) pad[1 + zeros + i] = (uint8_t)(bits >> (56 - 8 * i));
        update(pad, 1 + zeros + 8);
        for (int i = 0; i < 8; i++) {
            out[4 * i] = (uint8_t)(h[i] >> 24); out[4 * i + 1] = (uint8_t)(h[i] >> 16);
            out[4 * i + 2] = (uint8_t)(h[i] >> 8); out[4 * i + 3] = (uint8_t)h[i];
        }
    }
};

}  // namespace

void sha256(const void* data, size_t n, uint8_t out[32]) {
    Sha s;
    s.update((const uint8_t*)data, n);
    s.finish(out);
}

void chunk_key(const uint8_t prev[32], const uint32_t* tokens, uint32_t G, uint8_t out[32]) {
    Sha s;
    s.update(prev, 32);
    uint8_t le[4 * 64];
    uint32_t done = 0;
    while (done < G) {
        uint32_t take = std::min<uint32_t>(64, G - done);
        for (uint32_t i = 0; i < take; i++) {
            uint32_t t = tokens[done + i];
            le[4 * i] = (uint8_t)t; le[4 * i + 1] = (uint8_t)(t >> 8);
            le[4 * i + 2] = (uint8_t)(t >> 16); le[4 * i + 3] = (uint8_t)(t >> 24);
        }
        s.update(le, 4 * take);
        done += take;
    }
    s.finish(out);
}

}  // namespace oc

extern "C" {

OC_API int oc_sha256(const void* data, uint64_t n, uint8_t out[32]) {
    if ((!data && n) || !out) return oc::fail(OC_EINVAL, "oc_sha256: null pointer");
    oc::sha256(data, n, out);
    return OC_OK;
}

OC_API int oc_chunk_keys(const uint32_t* tokens, uint64_t n_tokens, uint32_t G, const oc_key* parent,
                         oc_key* out, uint64_t cap, uint64_t* n_out) {
    if (G == 0) return oc::fail(OC_EINVAL, "oc_chunk_keys: chunk_tokens must be >= 1");
    if ((!tokens && n_tokens) || !n_out) return oc::fail(OC_EINVAL, "oc_chunk_keys: null pointer");
    uint64_t count = n_tokens / G;
    *n_out = count;
    if (count > cap) return oc::fail(OC_ERANGE, "oc_chunk_keys: output capacity smaller than key count");
    if (count && !out) return oc::fail(OC_EINVAL, "oc_chunk_keys: null output");
    uint8_t prev[32] = {0};
    if (parent) std::memcpy(prev, parent->b, 32);
    for (uint64_t i = 0; i < count; i++) {
        oc::chunk_key(prev, tokens + i * G, G, out[i].b);
        std::memcpy(prev, out[i].b, 32);
    }
    return OC_OK;
}

}  // extern "C"
