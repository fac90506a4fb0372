// The ObjectCache descriptor (Table 1) made GPU-native.
//
// Table 1 names the matched chunk keys [H_0..H_{N-1}], L, G, S, the delivery order and the RDMA
// target.  Here build_descriptor validates the request, resolves every key to its chunk slot
// (the gateway's key validation and the storage server's object resolution), and
// uploads one packed device descriptor: src[N] slot addresses, the K/V base of every layer, the
// block table and the per-layer completion words.  The descriptor is "arithmetic rather than
// manifest-heavy": every layer range is [lS, (l+1)S) of a slot.
#include <algorithm>
#include <unordered_set>

#include "oc_internal.h"

namespace oc {

namespace {
size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

}  // namespace

void plan_units(Desc* d, uint32_t unit_bytes) {
    DevDesc& dd = d->dd;
    if (unit_bytes == 0) unit_bytes = 32768;
    uint64_t R = std::max<uint64_t>(1, unit_bytes / d->geo.row);
    R = std::min<uint64_t>(R, d->geo.G);
    R = std::min<uint64_t>(R, 1024);  // rows per unit are staged in a 1024-entry shared table
    dd.rows_per_unit = (uint32_t)R;
    dd.tiles = (uint32_t)((d->geo.G + R - 1) / R);
    dd.units_per_layer = (uint32_t)(d->N * 2 * dd.tiles);
    dd.div_upl = make_fastdiv(dd.units_per_layer);
    dd.div_units_per_chunk = make_fastdiv(2 * dd.tiles);
    dd.div_tiles = make_fastdiv(dd.tiles);
}

}  // namespace oc

using oc::Desc;

extern "C" {

OC_API int oc_build_descriptor(oc_store* sh, const oc_key* keys, uint64_t n, const oc_layout* layout, int delivery,
                               const oc_target* t, oc_desc** out, uint64_t* bad_index) {
    if (!sh || !layout || !t || !out) return oc::fail(OC_EINVAL, "build_descriptor: null pointer");
    *out = nullptr;
    oc::Store* s = (oc::Store*)sh;
    if (n == 0) return oc::fail(OC_EINVAL, "build_descriptor: a descriptor names N >= 1 chunks");
    if (!keys) return oc::fail(OC_EINVAL, "build_descriptor: null keys");
    if (!oc::same_layout(*layout, s->layout)) return oc::fail(OC_EINVAL, "build_descriptor: layout differs from the store's");
    if (delivery != OC_DELIVER_LAYER_MAJOR && delivery != OC_DELIVER_CHUNK_MAJOR)
        return oc::fail(OC_EINVAL, "build_descriptor: unknown delivery");
    const oc::Geometry& g = s->geo;
    if ((unsigned __int128)n * g.G >= ((unsigned __int128)1 << 31))
        return oc::fail(OC_ERANGE, "build_descriptor: prefix longer than 2^31 tokens");

    // Resolve every key (first missing key reported by index, in prefix order).
    std::vector<uint64_t> src(n);
    uint64_t host_chunks = 0;
    for (uint64_t i = 0; i < n; i++) {
        int tier = OC_TIER_HBM;
        const bool found = oc::store_resolve(s, keys[i], &src[i], &tier);
        host_chunks += tier == OC_TIER_PINNED_HOST;
        if (!found) {
            if (bad_index) *bad_index = i;
            return oc::fail(OC_ENOTFOUND, "build_descriptor: chunk key " + std::to_string(i) + " not found");
        }
    }

    // Normalise the target to the paged form: the flat client buffer is a paged cache with one
    // G-token block per chunk, identity block table, block_stride = S and V after K in each block.
    const uint32_t L = g.L;
    std::vector<uint64_t> kb(L), vb(L);
    std::vector<int32_t> bt;
    uint64_t block_stride, token_stride, head_stride;
    uint32_t Bs, first_token;
    if (t->kind == OC_TARGET_FLAT) {
        uint64_t W = n * L * g.S;
        if (t->flat_capacity < W) return oc::fail(OC_ERANGE, "build_descriptor: flat target smaller than W = N*L*S");
        if (t->flat_base % 16) return oc::fail(OC_EALIGN, "build_descriptor: flat_base not 16-byte aligned");
        for (uint32_t l = 0; l < L; l++) {
            kb[l] = t->flat_base + (uint64_t)l * n * g.S;
            vb[l] = kb[l] + (uint64_t)g.G * g.row;
        }
        bt.resize(n);
        for (uint64_t i = 0; i < n; i++) bt[i] = (int32_t)i;
        block_stride = g.S;
        token_stride = g.row;
        head_stride = g.hd;
        Bs = g.G;
        first_token = 0;
    } else if (t->kind == OC_TARGET_PAGED) {
        if (!t->k_base || !t->v_base || !t->block_table) return oc::fail(OC_EINVAL, "build_descriptor: null paged arrays");
        if (t->block_size == 0) return oc::fail(OC_EINVAL, "build_descriptor: block_size must be >= 1");
        Bs = t->block_size;
        first_token = t->first_token;
        uint64_t last = (uint64_t)first_token + n * g.G - 1;
        if (last >= (1ull << 31)) return oc::fail(OC_ERANGE, "build_descriptor: token index exceeds 2^31");
        uint64_t need = last / Bs + 1;
        if (t->num_blocks < need) return oc::fail(OC_ERANGE, "build_descriptor: block table does not cover the prefix");
        block_stride = t->block_stride;
        token_stride = t->token_stride;
        head_stride = t->head_stride;
        if (block_stride % 16 || token_stride % 16 || head_stride % 16)
            return oc::fail(OC_EALIGN, "build_descriptor: strides must be multiples of 16 bytes");
        for (uint32_t l = 0; l < L; l++) {
            kb[l] = t->k_base[l];
            vb[l] = t->v_base[l];
            if (kb[l] % 16 || vb[l] % 16) return oc::fail(OC_EALIGN, "build_descriptor: K/V base not 16-byte aligned");
        }
        bt.assign(t->block_table, t->block_table + need);
        std::unordered_set<int32_t> seen;
        seen.reserve(need * 2);
        for (uint64_t b = first_token / Bs; b < need; b++) {
            if (bt[b] < 0) return oc::fail(OC_EINVAL, "build_descriptor: negative block id");
            if (!seen.insert(bt[b]).second)
                return oc::fail(OC_EINVAL, "build_descriptor: duplicate block id in the prefix (reading c4)");
        }
    } else {
        return oc::fail(OC_EINVAL, "build_descriptor: unknown target kind");
    }

    auto d = std::make_unique<Desc>();
    d->store = s;
    d->geo = g;
    d->layout = *layout;
    d->device = s->device;
    d->delivery = delivery;
    d->N = n;
    d->nb = bt.size();
    d->host_chunks = host_chunks;

    // One device allocation: src[N] | k_base[L] | v_base[L] | ts[L+1] | unit_cnt[L] | ready, next | bt
    size_t o_src = 0;
    size_t o_kb = oc::align16(o_src + n * 8);
    size_t o_vb = oc::align16(o_kb + L * 8);
    size_t o_ts = oc::align16(o_vb + L * 8);
    size_t o_cnt = oc::align16(o_ts + (L + 1) * 8);
    size_t o_ready = oc::align16(o_cnt + L * 4);
    size_t o_next = o_ready + 4;
    size_t o_bt = oc::align16(o_ready + 16);
    size_t total = oc::align16(o_bt + bt.size() * 4);
    std::vector<uint8_t> stage(total, 0);
    std::memcpy(stage.data() + o_src, src.data(), n * 8);
    std::memcpy(stage.data() + o_kb, kb.data(), L * 8);
    std::memcpy(stage.data() + o_vb, vb.data(), L * 8);
    std::memcpy(stage.data() + o_bt, bt.data(), bt.size() * 4);

    oc::DeviceGuard dg(d->device);
    uint64_t cls = 0;
    void* mem = oc::dev_pool_alloc(d->device, total, &cls);
    if (!mem) return oc::fail(OC_ENOMEM, "build_descriptor: device allocation failed");
    cudaError_t e = cudaMemcpy(mem, stage.data(), total, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        oc::dev_pool_free(d->device, mem, cls);
        return oc::cuda_fail(e, "build_descriptor: upload");
    }
    d->dev_mem = mem;
    d->dev_mem_class = cls;

    uint8_t* m = (uint8_t*)mem;
    oc::DevDesc& dd = d->dd;
    std::memset(&dd, 0, sizeof dd);
    dd.src = (const uint64_t*)(m + o_src);
    dd.k_base = (const uint64_t*)(m + o_kb);
    dd.v_base = (const uint64_t*)(m + o_vb);
    dd.ts = (uint64_t*)(m + o_ts);
    dd.unit_cnt = (uint32_t*)(m + o_cnt);
    dd.ready = (uint32_t*)(m + o_ready);
    dd.next_unit = (uint32_t*)(m + o_next);
    dd.bt = (const int32_t*)(m + o_bt);
    dd.S = g.S;
    dd.row = g.row;
    dd.block_stride = block_stride;
    dd.token_stride = token_stride;
    dd.head_stride = head_stride;
    dd.N = (uint32_t)n;
    dd.L = L;
    dd.G = g.G;
    dd.Bs = Bs;
    dd.first_token = first_token;
    dd.vpr = (uint32_t)(g.row / 16);
    dd.nhd = (token_stride == g.row && head_stride == g.hd) ? 1u : 0u;
    dd.chunk_major = delivery == OC_DELIVER_CHUNK_MAJOR;
    dd.div_vpr = oc::make_fastdiv(dd.vpr);
    dd.div_Bs = oc::make_fastdiv(Bs);
    dd.div_hdv = oc::make_fastdiv((uint32_t)(g.hd / 16));
    oc::plan_units(d.get(), 0);
    *out = (oc_desc*)d.release();
    return OC_OK;
}

OC_API int oc_desc_free(oc_desc* h) {
    if (!h) return OC_OK;
    Desc* d = (Desc*)h;
    {
        oc::DeviceGuard dg(d->device);
        // Defer until the last fetch has finished with the descriptor's device memory.
        if (d->fetched && d->done_ev) cudaEventSynchronize(d->done_ev);
        for (auto ev : d->events) cudaEventDestroy(ev);
        if (d->done_ev) cudaEventDestroy(d->done_ev);
        if (d->sync_ev) cudaEventDestroy(d->sync_ev);
        if (d->sync_stream) cudaStreamDestroy(d->sync_stream);
        oc::dev_pool_free(d->device, d->dev_mem, d->dev_mem_class);
        cudaGetLastError();
    }
    delete d;
    return OC_OK;
}

OC_API int oc_desc_info(const oc_desc* h, uint64_t* n_chunks, uint64_t* payload_W, uint64_t* units_per_layer) {
    if (!h) return oc::fail(OC_EINVAL, "desc_info: null descriptor");
    const Desc* d = (const Desc*)h;
    if (n_chunks) *n_chunks = d->N;
    if (payload_W) *payload_W = d->N * d->geo.L * d->geo.S;
    if (units_per_layer) *units_per_layer = d->dd.units_per_layer;
    return OC_OK;
}

}  // extern "C"
