// The ObjectCache descriptor (Table 1) made GPU-native, and the offload path.
//
// Table 1 names the matched chunk keys [H_0..H_{N-1}], L, G, S, the delivery order and the RDMA
// target.  build_descriptor validates the request, resolves every key to its chunk slot (the
// gateway's key validation and the storage server's object resolution), and uploads
// one packed device descriptor: src[N] slot addresses, the K/V base of every layer, the block
// table and the per-layer completion words.  The descriptor is "arithmetic rather than
// manifest-heavy": every layer range is [lS, (l+1)S) of a slot.
//
// put_from_paged is the inverse direction (newly produced KV blocks are offloaded back for
// future reuse): the same target normalisation, then a gather kernel from the paged cache into
// freshly reserved slots.
#include <algorithm>
#include <mutex>
#include <unordered_map>
#include <unordered_set>

#include "oc_internal.h"

namespace oc {

namespace {
size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// A target in the paged form: the flat client buffer is a paged cache with one G-token block per
// chunk, identity block table, block_stride = S and V after K in each block.
struct PagedView {
    std::vector<uint64_t> kb, vb;
    std::vector<int32_t> bt;
    uint64_t block_stride = 0, token_stride = 0, head_stride = 0;
    uint32_t Bs = 0, first_token = 0;
};

int normalize_target(const Geometry& g, uint64_t n, const oc_target* t, const char* who, PagedView* v) {
    const uint32_t L = g.L;
    v->kb.resize(L);
    v->vb.resize(L);
    if (t->kind == OC_TARGET_FLAT) {
        uint64_t W = n * L * g.S;
        if (t->flat_capacity < W) return fail(OC_ERANGE, std::string(who) + ": flat target smaller than W = N*L*S");
        if (t->flat_base % 16) return fail(OC_EALIGN, std::string(who) + ": flat_base not 16-byte aligned");
        for (uint32_t l = 0; l < L; l++) {
            v->kb[l] = t->flat_base + (uint64_t)l * n * g.S;
            v->vb[l] = v->kb[l] + (uint64_t)g.G * g.row;
        }
        v->bt.resize(n);
        for (uint64_t i = 0; i < n; i++) v->bt[i] = (int32_t)i;
        v->block_stride = g.S;
        v->token_stride = g.row;
        v->head_stride = g.hd;
        v->Bs = g.G;
        v->first_token = 0;
        return OC_OK;
    }
    if (t->kind != OC_TARGET_PAGED) return fail(OC_EINVAL, std::string(who) + ": unknown target kind");
    if (!t->k_base || !t->v_base || !t->block_table)
        return fail(OC_EINVAL, std::string(who) + ": null paged arrays");
    if (t->block_size == 0) return fail(OC_EINVAL, std::string(who) + ": block_size must be >= 1");
    v->Bs = t->block_size;
    v->first_token = t->first_token;
    const uint64_t last = (uint64_t)v->first_token + n * g.G - 1;
    if (last >= (1ull << 31)) return fail(OC_ERANGE, std::string(who) + ": token index exceeds 2^31");
    const uint64_t need = last / v->Bs + 1;
    if (t->num_blocks < need) return fail(OC_ERANGE, std::string(who) + ": block table does not cover the prefix");
    v->block_stride = t->block_stride;
    v->token_stride = t->token_stride;
    v->head_stride = t->head_stride;
    if (v->block_stride % 16 || v->token_stride % 16 || v->head_stride % 16)
        return fail(OC_EALIGN, std::string(who) + ": strides must be multiples of 16 bytes");
    for (uint32_t l = 0; l < L; l++) {
        v->kb[l] = t->k_base[l];
        v->vb[l] = t->v_base[l];
        if (v->kb[l] % 16 || v->vb[l] % 16) return fail(OC_EALIGN, std::string(who) + ": K/V base not 16-byte aligned");
    }
    v->bt.assign(t->block_table, t->block_table + need);
    std::unordered_set<int32_t> seen;
    seen.reserve(need * 2);
    for (uint64_t b = v->first_token / v->Bs; b < need; b++) {
        if (v->bt[b] < 0) return fail(OC_EINVAL, std::string(who) + ": negative block id");
        if (!seen.insert(v->bt[b]).second)
            return fail(OC_EINVAL, std::string(who) + ": duplicate block id in the prefix (reading c4)");
    }
    return OC_OK;
}

// Device block layout shared by descriptors and offload jobs:
//   src[N] | k_base[L] | v_base[L] | ts[L+1] | unit_cnt[L] | ready, next | bt[nb] | pos[N] | hot[N]
struct BlockLayout {
    size_t o_src, o_kb, o_vb, o_ts, o_cnt, o_ready, o_next, o_bt, o_pos, o_hot, total;
};

BlockLayout block_layout(uint64_t n, uint32_t L, size_t nb, bool with_pos, bool with_hot = false) {
    BlockLayout b;
    b.o_src = 0;
    b.o_kb = align16(b.o_src + n * 8);
    b.o_vb = align16(b.o_kb + L * 8);
    b.o_ts = align16(b.o_vb + L * 8);
    b.o_cnt = align16(b.o_ts + (L + 1) * 8);
    b.o_ready = align16(b.o_cnt + L * 4);
    // the claim slots on their own 128-byte line (apart from the polled ready word)
    b.o_next = (b.o_ready + 4 + 127) & ~size_t(127);
    b.o_bt = b.o_next + kClaimSlots * kClaimSlotStride * 4;
    b.o_pos = align16(b.o_bt + nb * 4);
    b.o_hot = align16(b.o_pos + (with_pos ? n * 4 : 0));
    b.total = align16(b.o_hot + (with_hot ? n * 8 : 0));
    return b;
}


// Upload src/bases/bt(/pos) into a pooled device block and fill the static DevDesc fields.  The
// block is staged in pooled pinned memory and copied asynchronously: on `on_stream` itself when
// `ordered` (the caller launches its kernel on that stream next), else on the device's private
// upload stream with up->ev marking completion (see Upload in oc_internal.h).
int upload_block(int device, const Geometry& g, const std::vector<uint64_t>& src, const PagedView& v,
                 const std::vector<uint32_t>* pos, const char* who, void** mem_out, uint64_t* cls_out, DevDesc* dd,
                 const uint32_t** pos_dev, Upload* up, bool ordered, cudaStream_t on_stream,
                 const std::vector<uint64_t>* src_hot = nullptr, uint32_t hot_layers = 0) {
    const uint64_t n = src.size();
    const uint32_t L = g.L;
    const BlockLayout b = block_layout(n, L, v.bt.size(), pos != nullptr, src_hot != nullptr);
    uint64_t scls = 0;
    uint8_t* stage = (uint8_t*)dev_pool_alloc(-1, b.total, &scls);
    if (!stage) return fail(OC_ENOMEM, std::string(who) + ": pinned staging allocation failed");
    std::memset(stage, 0, b.total);
    std::memcpy(stage + b.o_src, src.data(), n * 8);
    std::memcpy(stage + b.o_kb, v.kb.data(), L * 8);
    std::memcpy(stage + b.o_vb, v.vb.data(), L * 8);
    std::memcpy(stage + b.o_bt, v.bt.data(), v.bt.size() * 4);
    if (pos) std::memcpy(stage + b.o_pos, pos->data(), n * 4);
    if (src_hot) std::memcpy(stage + b.o_hot, src_hot->data(), n * 8);
    uint64_t cls = 0;
    void* mem = dev_pool_alloc(device, b.total, &cls);
    if (!mem) {
        dev_pool_free(-1, stage, scls);
        return fail(OC_ENOMEM, std::string(who) + ": device allocation failed");
    }
    cudaStream_t us = ordered ? on_stream : upload_stream(device);
    cudaEvent_t ev = nullptr;
    cudaError_t e = !ordered && !us ? cudaErrorInvalidResourceHandle : cudaSuccess;
    if (e == cudaSuccess && !ordered) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMemcpyAsync(mem, stage, b.total, cudaMemcpyHostToDevice, us);
    if (e == cudaSuccess && ev) e = cudaEventRecord(ev, us);
    if (e != cudaSuccess) {
        if (us) cudaStreamSynchronize(us);
        if (ev) cudaEventDestroy(ev);
        dev_pool_free(device, mem, cls);
        dev_pool_free(-1, stage, scls);
        return cuda_fail(e, who);
    }
    up->ev = ev;
    up->stage = stage;
    up->stage_cls = scls;
    up->done = false;
    *mem_out = mem;
    *cls_out = cls;
    uint8_t* m = (uint8_t*)mem;
    std::memset(dd, 0, sizeof *dd);
    dd->src = (const uint64_t*)(m + b.o_src);
    dd->k_base = (const uint64_t*)(m + b.o_kb);
    dd->v_base = (const uint64_t*)(m + b.o_vb);
    dd->ts = (uint64_t*)(m + b.o_ts);
    dd->unit_cnt = (uint32_t*)(m + b.o_cnt);
    dd->ready = (uint32_t*)(m + b.o_ready);
    dd->next_unit = (uint32_t*)(m + b.o_next);
    dd->bt = (const int32_t*)(m + b.o_bt);
    if (pos_dev) *pos_dev = pos ? (const uint32_t*)(m + b.o_pos) : nullptr;
    if (src_hot) {
        dd->src_hot = (const uint64_t*)(m + b.o_hot);
        dd->hot_layers = hot_layers;
    }
    dd->S = g.S;
    dd->row = g.row;
    dd->block_stride = v.block_stride;
    dd->token_stride = v.token_stride;
    dd->head_stride = v.head_stride;
    dd->N = (uint32_t)n;
    dd->L = L;
    dd->G = g.G;
    dd->Bs = v.Bs;
    dd->first_token = v.first_token;
    dd->vpr = (uint32_t)(g.row / 16);
    dd->nhd = (v.token_stride == g.row && v.head_stride == g.hd) ? 1u : 0u;
    dd->div_vpr = make_fastdiv(dd->vpr);
    dd->div_Bs = make_fastdiv(v.Bs);
    dd->div_hdv = make_fastdiv((uint32_t)(g.hd / 16));
    return OC_OK;
}

void plan_into(DevDesc& dd, const Geometry& g, uint64_t n, uint32_t unit_bytes) {
    if (unit_bytes == 0) unit_bytes = 32768;
    // A unit is R consecutive rows of a chunk's 2G-row layer slice (K rows, then V rows).
    uint64_t R = std::max<uint64_t>(1, unit_bytes / g.row);
    R = std::min<uint64_t>(R, 2ull * g.G);
    R = std::min<uint64_t>(R, 1024);  // rows per unit are staged in a 1024-entry shared table
    dd.rows_per_unit = (uint32_t)R;
    dd.tiles = (uint32_t)((2ull * g.G + R - 1) / R);
    dd.units_per_layer = (uint32_t)(n * dd.tiles);
    dd.div_upl = make_fastdiv(dd.units_per_layer);
    dd.div_tiles = make_fastdiv(dd.tiles);
}

// Blocks of offload jobs still in flight.  They are recycled once the job's event has completed,
// polled at the next put_from_paged -- a host callback in the caller's stream would make that
// stream wait for a host thread's wake-up after every offload.
struct OffloadJob {
    cudaEvent_t done;
    int device;
    void* mem;
    uint64_t cls;
    void* stage;
    uint64_t stage_cls;
};
std::mutex g_jobs_mu;
std::vector<OffloadJob> g_jobs;

void release_job(const OffloadJob& j) {
    dev_pool_free(j.device, j.mem, j.cls);
    dev_pool_free(-1, j.stage, j.stage_cls);
    if (j.done) cudaEventDestroy(j.done);
}

void reap_jobs() {
    std::lock_guard<std::mutex> lk(g_jobs_mu);
    size_t keep = 0;
    for (size_t i = 0; i < g_jobs.size(); i++) {
        cudaError_t q = cudaEventQuery(g_jobs[i].done);
        if (q == cudaErrorNotReady) {
            g_jobs[keep++] = g_jobs[i];
        } else {
            release_job(g_jobs[i]);
        }
    }
    g_jobs.resize(keep);
    cudaGetLastError();
}
}  // namespace

void plan_units(Desc* d, uint32_t unit_bytes) { plan_into(d->dd, d->geo, d->N, unit_bytes); }

cudaStream_t upload_stream(int device) {
    static std::mutex mu;
    static std::unordered_map<int, cudaStream_t> streams;
    std::lock_guard<std::mutex> lk(mu);
    auto it = streams.find(device);
    if (it != streams.end()) return it->second;
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    streams.emplace(device, s);
    return s;
}

int upload_order(Upload* u, cudaStream_t s) {
    if (!u->ev || u->done) return OC_OK;
    cudaError_t q = cudaEventQuery(u->ev);
    if (q == cudaSuccess) {  // landed: later launches need no wait; recycle the stage
        u->done = true;
        dev_pool_free(-1, u->stage, u->stage_cls);
        u->stage = nullptr;
        return OC_OK;
    }
    if (q != cudaErrorNotReady) return cuda_fail(q, "descriptor upload");
    cudaGetLastError();
    OC_CUDA(cudaStreamWaitEvent(s, u->ev, 0));
    return OC_OK;
}

void upload_release(Upload* u) {
    if (u->ev) {
        cudaEventSynchronize(u->ev);
        cudaEventDestroy(u->ev);
        u->ev = nullptr;
    }
    if (u->stage) dev_pool_free(-1, u->stage, u->stage_cls);
    u->stage = nullptr;
    u->done = true;
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
    std::vector<uint64_t> src(n), hot(n);
    std::vector<uint32_t> hot_pitch_layers(n);  // layers per mirror slot of the chunk's own store
    uint64_t host_chunks = 0;
    uint32_t hot_layers = ~0u;  // leading layers mirrored in HBM for EVERY chunk
    for (uint64_t i = 0; i < n; i++) {
        int tier = OC_TIER_HBM;
        uint32_t hl = 0;
        const bool found = oc::store_resolve(s, keys[i], &src[i], &tier, &hot[i], &hl);
        host_chunks += tier == OC_TIER_PINNED_HOST;
        hot_pitch_layers[i] = hl;
        hot_layers = std::min(hot_layers, found ? hl : 0u);
        if (!found) {
            if (bad_index) *bad_index = i;
            return oc::fail(OC_ENOTFOUND, "build_descriptor: chunk key " + std::to_string(i) + " not found");
        }
    }
    oc::PagedView v;
    int rc = oc::normalize_target(g, n, t, "build_descriptor", &v);
    if (rc) return rc;

    auto d = std::make_unique<Desc>();
    d->store = s;
    d->geo = g;
    d->layout = *layout;
    d->device = s->device;
    d->delivery = delivery;
    d->N = n;
    d->nb = v.bt.size();
    d->host_chunks = host_chunks;
    if (t->kind == OC_TARGET_FLAT) d->flat_base = t->flat_base;
    if (hot_layers == ~0u) hot_layers = 0;
    if (host_chunks == n) {  // CE engine: maximal runs of chunks in consecutive slots
        // With mirrors, a run also needs consecutive mirror slots of ONE pitch: stores (own and
        // attached peers) may mirror different numbers of layers, and each lays its mirror out with
        // its own pitch hot_layers*S -- a run crossing stores would read the wrong mirror bytes.
        for (uint64_t i = 0; i < n; i++) {
            const uint64_t pitch = (uint64_t)hot_pitch_layers[i] * g.S;
            const bool cont = i > 0 && src[i] == src[i - 1] + g.chunk &&
                              (!hot_layers || (hot_pitch_layers[i] == hot_pitch_layers[i - 1] &&
                                               hot[i] == hot[i - 1] + pitch));
            if (cont) {
                d->run_len.back()++;
            } else {
                d->run_first.push_back(i);
                d->run_len.push_back(1);
                d->run_src.push_back(src[i]);
                if (hot_layers) {
                    d->run_hot.push_back(hot[i]);
                    d->run_hot_pitch.push_back(pitch);
                }
            }
        }
    }
    oc::DeviceGuard dg(d->device);
    d->hot_layers = hot_layers;
    rc = oc::upload_block(d->device, g, src, v, nullptr, "build_descriptor", &d->dev_mem, &d->dev_mem_class, &d->dd,
                          nullptr, &d->up, false, nullptr, hot_layers ? &hot : nullptr, hot_layers);
    if (rc) return rc;
    // Without a mirror (pinned allocation failed) wait_layer always enqueues its stream wait.
    d->ready_host = oc::ready_mirror_alloc();
    d->dd.ready_host = d->ready_host;
    d->dd.chunk_major = delivery == OC_DELIVER_CHUNK_MAJOR;
    oc::plan_units(d.get(), 0);
    *out = (oc_desc*)d.release();
    return OC_OK;
}

OC_API int oc_put_from_paged(oc_store* sh, const oc_key* keys, uint64_t n, const oc_layout* layout,
                             const oc_target* t, void* stream, uint64_t* n_new, uint64_t* bad_index) {
    if (!sh || !layout || !t) return oc::fail(OC_EINVAL, "put_from_paged: null pointer");
    oc::reap_jobs();  // recycle the blocks of finished offloads
    oc::Store* s = (oc::Store*)sh;
    if (n_new) *n_new = 0;
    if (n == 0) return OC_OK;
    if (!keys) return oc::fail(OC_EINVAL, "put_from_paged: null keys");
    if (s->read_only) return oc::fail(OC_EINVAL, "put_from_paged: store is a read-only imported peer");
    if (s->hot_layers) return oc::fail(OC_ENOTSUP, "put_from_paged: store mirrors hot layers (use put_chunks)");
    if (t->kind != OC_TARGET_PAGED) return oc::fail(OC_EINVAL, "put_from_paged: source must be a paged cache");
    if (!oc::same_layout(*layout, s->layout)) return oc::fail(OC_EINVAL, "put_from_paged: layout differs from the store's");
    const oc::Geometry& g = s->geo;
    if ((unsigned __int128)n * g.G >= ((unsigned __int128)1 << 31))
        return oc::fail(OC_ERANGE, "put_from_paged: prefix longer than 2^31 tokens");
    oc::PagedView v;
    int rc = oc::normalize_target(g, n, t, "put_from_paged", &v);
    if (rc) return rc;

    // Reserve slots for the new keys (dedup by key), in prefix order.
    std::vector<uint64_t> dst;
    std::vector<uint32_t> pos;
    int status = OC_OK;
    {
        std::unique_lock<std::shared_mutex> lk(s->mu);
        for (uint64_t i = 0; i < n; i++) {
            if (s->index.count(keys[i])) continue;
            if (s->count >= s->capacity) {
                if (bad_index) *bad_index = i;
                status = oc::fail(OC_EFULL, "put_from_paged: store capacity exhausted");
                break;
            }
            const uint64_t slot = s->count++;
            s->index.emplace(keys[i], slot);
            dst.push_back((uint64_t)(uintptr_t)s->slab + slot * s->pitch);
            pos.push_back((uint32_t)i);
        }
    }
    if (n_new) *n_new = dst.size();
    if (dst.empty()) return status;
    auto rollback = [&]() {  // the reserved slots never received their bytes: forget the keys
        std::unique_lock<std::shared_mutex> lk(s->mu);
        for (uint32_t p : pos) s->index.erase(keys[p]);
        // give the slots back when nobody reserved after them (they are the slab's last ones)
        const uint64_t first = (dst.front() - (uint64_t)(uintptr_t)s->slab) / s->pitch;
        if (s->count == first + dst.size()) s->count = first;
        if (n_new) *n_new = 0;
    };
    oc::DeviceGuard dg(s->device);
    oc::DevDesc dd;
    void* mem = nullptr;
    uint64_t cls = 0;
    const uint32_t* pos_dev = nullptr;
    cudaStream_t st = (cudaStream_t)stream;
    oc::Upload up;
    // The block goes up on the library's upload stream, not on `st`: a small H2D copy queued
    // between two back-to-back offload kernels would idle the GPU for its DMA latency.  `st` only
    // waits on the copy's event, which has long fired when the previous kernel ends.
    rc = oc::upload_block(s->device, g, dst, v, &pos, "put_from_paged", &mem, &cls, &dd, &pos_dev, &up, false, st);
    if (rc) {
        rollback();
        return rc;
    }
    {
        cudaError_t e = cudaStreamWaitEvent(st, up.ev, 0);
        cudaEventDestroy(up.ev);
        up.ev = nullptr;
        if (e != cudaSuccess) {
            cudaStreamSynchronize(oc::upload_stream(s->device));
            oc::dev_pool_free(s->device, mem, cls);
            oc::dev_pool_free(-1, up.stage, up.stage_cls);
            rollback();
            return oc::cuda_fail(e, "put_from_paged: ordering after the upload");
        }
    }
    oc::plan_into(dd, g, dst.size(), 0);
    rc = oc::launch_offload(dd, pos_dev, s->device, st, s->tier == OC_TIER_PINNED_HOST);
    if (rc) {
        cudaStreamSynchronize(st);
        oc::dev_pool_free(s->device, mem, cls);
        oc::dev_pool_free(-1, up.stage, up.stage_cls);
        rollback();
        return rc;
    }
    oc::OffloadJob job{nullptr, s->device, mem, cls, up.stage, up.stage_cls};
    cudaError_t e = cudaEventCreateWithFlags(&job.done, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(job.done, st);
    if (e != cudaSuccess) {
        cudaStreamSynchronize(st);
        oc::release_job(job);
        return oc::cuda_fail(e, "put_from_paged: completion event");
    }
    {
        std::lock_guard<std::mutex> lk(oc::g_jobs_mu);
        oc::g_jobs.push_back(job);
    }
    {  // the store's record of offloads in flight (put_chunks' byte compare waits on them)
        cudaEvent_t ev = nullptr;
        if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess && cudaEventRecord(ev, st) == cudaSuccess) {
            std::unique_lock<std::shared_mutex> lk(s->mu);
            auto& v = s->offload_evs;
            for (size_t i = 0; i < v.size();) {  // drop the finished ones
                if (cudaEventQuery(v[i]) == cudaSuccess) {
                    cudaEventDestroy(v[i]);
                    v[i] = v.back();
                    v.pop_back();
                } else {
                    i++;
                }
            }
            v.push_back(ev);
        } else {
            if (ev) cudaEventDestroy(ev);
            cudaStreamSynchronize(st);  // no event: make the slots final before returning
        }
        cudaGetLastError();
    }
    return status;
}

OC_API int oc_desc_free(oc_desc* h) {
    if (!h) return OC_OK;
    Desc* d = (Desc*)h;
    {
        oc::DeviceGuard dg(d->device);
        // Defer until the last fetch has finished with the descriptor's device memory.
        if (d->fetched && d->done_ev) cudaEventSynchronize(d->done_ev);
        for (auto ev : d->range_evs) {  // an incomplete ranged fetch: every range's launch
            cudaEventSynchronize(ev);
            cudaEventDestroy(ev);
        }
        oc::upload_release(&d->up);
        oc::per_layer_events_release(d);
        if (d->done_ev) cudaEventDestroy(d->done_ev);
        if (d->sync_ev) cudaEventDestroy(d->sync_ev);
        if (d->sync_stream) cudaStreamDestroy(d->sync_stream);
        oc::relay_release(d);
        oc::ce_release(d);
        oc::dev_pool_free(d->device, d->dev_mem, d->dev_mem_class);
        oc::ready_mirror_free(d->ready_host);
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
