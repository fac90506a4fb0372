// Stall-target bandwidth scheduling (Sec. 3.6; Alg. A2).
//
// Request i moves s_i bytes per layer and has c_i seconds of compute per layer; its zero-stall
// rate is r_i* = s_i / c_i.  Stall-opt (Eq. 6) minimises sum s_i/r_i
// subject to sum r_i = B and 0 < r_i <= r_i*; Calibrated Stall-opt (Eq. 7) raises the
// caps to r_i* + delta.  Stationarity of the Lagrangian gives r_i = min(cap_i, lambda*sqrt(s_i))
// (reading c8): requests whose cap_i/sqrt(s_i) lies below lambda are held at their cap, the rest
// share what is left in proportion to sqrt(s_i).  Here that is solved in O(n log n) by sorting on
// cap_i/sqrt(s_i) and scanning for the first consistent split.  If the caps fit in B every
// request receives its cap and the remainder is not handed out (reading c10).
// Baselines: Equal, KV-prop (proportional to s_i), BW-prop (proportional to r_i*).
#include <algorithm>
#include <cmath>
#include <numeric>

#include "oc_internal.h"

extern "C" OC_API int oc_schedule_bandwidth(int policy, const oc_profile* prof, uint64_t n, double B,
                                            double delta, double* rates) {
    if (!(B > 0) || !std::isfinite(B)) return oc::fail(OC_EINVAL, "schedule_bandwidth: cap B must be > 0");
    if (!(delta >= 0) || !std::isfinite(delta)) return oc::fail(OC_EINVAL, "schedule_bandwidth: delta must be >= 0");
    if (policy < OC_POL_EQUAL || policy > OC_POL_CAL_STALL_OPT)
        return oc::fail(OC_EINVAL, "schedule_bandwidth: unknown policy");
    if (n == 0) return OC_OK;
    if (!prof || !rates) return oc::fail(OC_EINVAL, "schedule_bandwidth: null pointer");
    for (uint64_t i = 0; i < n; i++) {
        double s = prof[i].bytes_per_layer, c = prof[i].compute_per_layer_s;
        if (!(s > 0) || !(c > 0) || !std::isfinite(s) || !std::isfinite(c))
            return oc::fail(OC_EINVAL, "schedule_bandwidth: s_i and c_i must be finite and > 0 (index " +
                                           std::to_string(i) + ")");
    }
    switch (policy) {
        case OC_POL_EQUAL:
            for (uint64_t i = 0; i < n; i++) rates[i] = B / (double)n;
            return OC_OK;
        case OC_POL_KV_PROP: {
            double tot = 0;
            for (uint64_t i = 0; i < n; i++) tot += prof[i].bytes_per_layer;
            for (uint64_t i = 0; i < n; i++) rates[i] = B * prof[i].bytes_per_layer / tot;
            return OC_OK;
        }
        case OC_POL_BW_PROP: {
            double tot = 0;
            for (uint64_t i = 0; i < n; i++) tot += prof[i].bytes_per_layer / prof[i].compute_per_layer_s;
            for (uint64_t i = 0; i < n; i++)
                rates[i] = B * (prof[i].bytes_per_layer / prof[i].compute_per_layer_s) / tot;
            return OC_OK;
        }
        default: break;
    }
    const double add = policy == OC_POL_CAL_STALL_OPT ? delta : 0.0;
    std::vector<double> cap(n), sq(n);
    double cap_sum = 0;
    for (uint64_t i = 0; i < n; i++) {
        cap[i] = prof[i].bytes_per_layer / prof[i].compute_per_layer_s + add;
        sq[i] = std::sqrt(prof[i].bytes_per_layer);
        cap_sum += cap[i];
    }
    if (cap_sum <= B) {
        for (uint64_t i = 0; i < n; i++) rates[i] = cap[i];
        return OC_OK;
    }
    std::vector<uint64_t> ord(n);
    std::iota(ord.begin(), ord.end(), 0);
    std::sort(ord.begin(), ord.end(), [&](uint64_t a, uint64_t b) { return cap[a] / sq[a] < cap[b] / sq[b]; });
    // suffix sums of sqrt(s) over the sorted order, prefix sums of caps
    std::vector<double> suf(n + 1, 0.0);
    for (uint64_t m = n; m-- > 0;) suf[m] = suf[m + 1] + sq[ord[m]];
    double capped = 0;
    for (uint64_t k = 0; k < n; k++) {
        double lam = (B - capped) / suf[k];
        uint64_t nxt = ord[k];
        if (cap[nxt] / sq[nxt] >= lam) {
            for (uint64_t m = 0; m < n; m++) {
                uint64_t i = ord[m];
                rates[i] = m < k ? cap[i] : lam * sq[i];
            }
            return OC_OK;
        }
        capped += cap[nxt];
    }
    return oc::fail(OC_EINVAL, "schedule_bandwidth: no feasible split (numerical)");
}

// Mirror depth for a pinned-host store (oc_store_set_hot_layers; DESIGN reading c24).  With the
// first K layers in HBM (ready at once) and the rest streamed back to back at X seconds per layer,
// layer l >= K is ready at (l - K + 1) X and the free-running pipeline of Eq. 3 adds no
// TTFT iff (l - K + 1) X <= l C for every l >= K; the binding case is the last layer, so
// K = max(1, ceil(L - (L - 1) C / X)), clamped to L.
extern "C" OC_API int oc_hot_layers_for(double X_s, double C_s, uint32_t L, uint32_t* K) {
    if (!K) return oc::fail(OC_EINVAL, "hot_layers_for: null out");
    if (!(X_s > 0) || !(C_s > 0) || !std::isfinite(X_s) || !std::isfinite(C_s) || L == 0)
        return oc::fail(OC_EINVAL, "hot_layers_for: X, C must be finite and > 0, L >= 1");
    const double k = std::ceil((double)L - (double)(L - 1) * C_s / X_s - 1e-12);
    *K = (uint32_t)std::max(1.0, std::min((double)L, k));
    return OC_OK;
}
