// Weighted deficit round robin dispatch of layer payloads (PAPER.md Alg. A2 lines 6-7,
// P:2595-2596; Sec. 3.6).
//
// The requests of one epoch share a link; Alg. A2 holds each request's rate r_i for the epoch and
// dispatches layer payloads with weighted deficit round robin.  On B200 the dispatcher is the
// claim order of one batched copy kernel: this file turns the requests' unit streams into that
// order, as a table of claim entries (request, first unit, count <= E) that copy CTAs take in
// sequence (fetch_kernels.cuh, fetch_bulk_kernel<kWdrr>).
//
// Deficit round robin (Shreedhar & Varghese): a round visits the backlogged requests in index
// order; a visit adds q_i to D_i and sends units from the request's head while the head unit's
// bytes are <= D_i; a request that runs out resets D_i = 0 and leaves.  A request's units are its
// layer-major unit stream (layer 0 of every chunk first), so its layers still complete in order
// (reading c21).  q_i = floor(Q * w_i / min_j w_j): the lightest request's quantum is Q, which must
// cover the largest unit (the textbook condition that makes every visit send).  With hold_rates
// (reading c22) entry e of request i is released no earlier than t0 + (bytes of request i in
// earlier entries) / r_i -- in whole microseconds, floor(bytes * 1e6 / r_i) -- and never before
// the previous entry, so releases are monotone along the claim order.  Units a request reads from
// HBM (free_units[i] leading units: the layers a pinned-host store mirrors, reading c24) never
// cross the paced link, so they neither wait nor count toward the request's bytes; nor does DRR
// schedule them: they are dispatched first, request by request (reading c25).
//
// Packet granularity: by default a packet is one copy unit (reading c21: a request's layer is many
// units, so its bytes interleave finely with the other requests'); with layer_packets = L a packet
// is a whole layer payload of N_i*S bytes, Alg. A2 line 7 as written, and the quantum must cover the
// largest one.  Both are DRR with the same weights, so their byte shares agree within one round
// of each (tests/test_oracle_dispatch.py pins the bound; test_lib_dispatch.py checks both planners).
#include <cmath>

#include "oc_internal.h"

namespace oc {

int wdrr_plan(const uint64_t* n_units, uint32_t n, const uint32_t* tile_bytes, uint32_t tiles, const oc_wdrr_opts& w,
              std::vector<WdrrEntry>* out) {
    out->clear();
    if (n == 0 || !n_units || !tile_bytes || tiles == 0 || !w.weights)
        return fail(OC_EINVAL, "wdrr: need n >= 1 requests, weights and tile sizes");
    uint64_t max_tile = 0, period = 0;
    std::vector<uint64_t> prefix(tiles + 1, 0);  // bytes of tiles [0, t)
    for (uint32_t t = 0; t < tiles; t++) {
        if (tile_bytes[t] == 0) return fail(OC_EINVAL, "wdrr: empty unit");
        max_tile = std::max<uint64_t>(max_tile, tile_bytes[t]);
        prefix[t + 1] = prefix[t] + tile_bytes[t];
    }
    period = prefix[tiles];
    // bytes of units [0, u) of a request: whole periods of `tiles` units, then a partial period
    auto bytes_upto = [&](uint64_t u) { return (u / tiles) * period + prefix[u % tiles]; };
    // Packets: one unit (reading c21), or with layer_packets = L one request's whole layer payload
    // (Alg. A2 line 7 as written): request i has L packets of upl_i = n_units[i] / L units.
    const uint32_t LP = w.layer_packets;
    std::vector<uint64_t> upl(n, 0), pkt(n, 0);
    uint64_t max_packet = max_tile;
    if (LP) {
        max_packet = 0;
        for (uint32_t i = 0; i < n; i++) {
            if (n_units[i] % LP) return fail(OC_EINVAL, "wdrr: layer packets need n_units a multiple of L");
            upl[i] = n_units[i] / LP;
            pkt[i] = bytes_upto(upl[i]);
            if (w.free_units && upl[i] && (std::min(w.free_units[i], n_units[i]) % upl[i]))
                return fail(OC_EINVAL, "wdrr: layer packets need free_units in whole layers");
            max_packet = std::max(max_packet, pkt[i]);
        }
    }
    const uint64_t Q = w.quantum_bytes ? w.quantum_bytes : std::max<uint64_t>(256 * 1024, max_packet);
    if (Q < max_packet) return fail(OC_EINVAL, LP ? "wdrr: quantum below the largest layer payload"
                                                  : "wdrr: quantum below the largest unit");
    const uint32_t E = w.entry_units ? w.entry_units : 8;
    double wmin = INFINITY;
    for (uint32_t i = 0; i < n; i++) {
        if (!(w.weights[i] > 0) || !std::isfinite(w.weights[i]))
            return fail(OC_EINVAL, "wdrr: weights must be finite and > 0 (index " + std::to_string(i) + ")");
        if (n_units[i] >= (1ull << 32)) return fail(OC_ERANGE, "wdrr: too many units in one request");
        wmin = std::min(wmin, w.weights[i]);
    }
    std::vector<uint64_t> q(n), D(n, 0), head(n, 0);
    for (uint32_t i = 0; i < n; i++) {
        const double qi = std::floor((double)Q * w.weights[i] / wmin);
        if (!(qi < 4.0e18)) return fail(OC_ERANGE, "wdrr: weight ratio too large");
        q[i] = (uint64_t)qi;
    }
    std::vector<uint32_t> active;
    uint64_t total_units = 0, visits = 0;  // reserve: ~one entry per visit plus one per E units
    for (uint32_t i = 0; i < n; i++) {
        if (n_units[i]) active.push_back(i);
        total_units += n_units[i];
        const uint64_t bytes_i = bytes_upto(n_units[i]);
        visits += bytes_i / std::max<uint64_t>(1, q[i]) + 1;
    }
    out->reserve(total_units / E + visits + 16);
    uint64_t prev_rel = 0;
    auto emit = [&](uint32_t i, uint64_t first, uint64_t cnt) -> int {
        for (uint64_t k = 0; k < cnt; k += E) {
            const uint64_t c = std::min<uint64_t>(E, cnt - k);
            uint64_t rel = 0;
            if (w.hold_rates) {
                // request i's link bytes before this entry: its bytes so far minus its free units'
                const uint64_t fu = w.free_units ? w.free_units[i] : 0;
                const uint64_t b = first + k <= fu ? 0 : bytes_upto(first + k) - bytes_upto(fu);
                const double t = std::floor((double)b * 1e6 / w.weights[i]);
                if (!(t < 4294967295.0)) return fail(OC_ERANGE, "wdrr: release time beyond 2^32 us");
                rel = std::max(prev_rel, (uint64_t)t);
                prev_rel = rel;
            }
            out->push_back(WdrrEntry{i, (uint32_t)(first + k), (uint32_t)c, (uint32_t)rel});
        }
        return OC_OK;
    };
    // reading c25: units a request reads from a store's HBM mirror are not link traffic -- they
    // go first, request by request, and DRR schedules the rest
    if (w.free_units) {
        size_t keep = 0;
        for (size_t a = 0; a < active.size(); a++) {
            const uint32_t i = active[a];
            head[i] = std::min(w.free_units[i], n_units[i]);
            if (head[i]) {
                int rc = emit(i, 0, head[i]);
                if (rc) return rc;
            }
            if (head[i] < n_units[i]) active[keep++] = i;
        }
        active.resize(keep);
    }
    uint32_t run_req = 0;
    uint64_t run_first = 0, run_cnt = 0;  // the dispatch run being extended
    while (!active.empty()) {
        size_t keep = 0;
        for (size_t a = 0; a < active.size(); a++) {
            const uint32_t i = active[a];
            D[i] += q[i];
            const uint64_t start = head[i];
            if (LP) {  // whole layer payloads while they fit in the deficit
                const uint64_t left = (n_units[i] - head[i]) / upl[i];
                const uint64_t k = std::min<uint64_t>(left, D[i] / pkt[i]);
                head[i] += k * upl[i];
                D[i] -= k * pkt[i];
            }
            // send units while the head unit fits in the deficit: the partial period first, then
            // whole periods arithmetically, then the rest unit by unit
            while (!LP && head[i] < n_units[i] && head[i] % tiles != 0 && tile_bytes[head[i] % tiles] <= D[i]) {
                D[i] -= tile_bytes[head[i] % tiles];
                head[i]++;
            }
            if (!LP && head[i] % tiles == 0) {
                const uint64_t periods = std::min<uint64_t>((n_units[i] - head[i]) / tiles, D[i] / period);
                head[i] += periods * tiles;
                D[i] -= periods * period;
                while (head[i] < n_units[i] && tile_bytes[head[i] % tiles] <= D[i]) {
                    D[i] -= tile_bytes[head[i] % tiles];
                    head[i]++;
                }
            }
            if (head[i] > start) {  // maximal runs: a visit continuing the previous one extends it
                if (run_cnt && run_req == i && run_first + run_cnt == start) {
                    run_cnt += head[i] - start;
                } else {
                    if (run_cnt) {
                        int rc = emit(run_req, run_first, run_cnt);
                        if (rc) return rc;
                    }
                    run_req = i;
                    run_first = start;
                    run_cnt = head[i] - start;
                }
            }
            if (head[i] == n_units[i]) D[i] = 0;
            else active[keep++] = i;
        }
        active.resize(keep);
    }
    return run_cnt ? emit(run_req, run_first, run_cnt) : OC_OK;
}

}  // namespace oc

extern "C" OC_API int oc_wdrr_plan(const uint64_t* n_units, uint32_t n, const uint32_t* tile_bytes, uint32_t tiles,
                                   const oc_wdrr_opts* w, uint32_t* ent_req, uint32_t* ent_first, uint32_t* ent_count,
                                   uint32_t* ent_release_us, uint64_t cap, uint64_t* n_entries) {
    if (!w || !n_entries) return oc::fail(OC_EINVAL, "wdrr_plan: null pointer");
    std::vector<oc::WdrrEntry> ents;
    int rc = oc::wdrr_plan(n_units, n, tile_bytes, tiles, *w, &ents);
    if (rc) return rc;
    *n_entries = ents.size();
    if (ents.size() > cap) return oc::fail(OC_ERANGE, "wdrr_plan: output capacity too small");
    for (size_t e = 0; e < ents.size(); e++) {
        if (ent_req) ent_req[e] = ents[e].req;
        if (ent_first) ent_first[e] = ents[e].first;
        if (ent_count) ent_count[e] = ents[e].count;
        if (ent_release_us) ent_release_us[e] = ents[e].rel_us;
    }
    return OC_OK;
}
