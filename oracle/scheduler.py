"""Bandwidth allocation across concurrent layerwise requests (oracle; test infrastructure only).

Sec. 3.6.  Request i moves s_i bytes per layer and has a
per-layer compute window c_i seconds.
  Eq. 4  tau_i(r_i) = max(0, s_i/r_i - c_i)
  P:530-532          zero-stall rate r_i* = s_i / c_i
  Eq. 6  min sum_i s_i/r_i  s.t. sum_i r_i = B, 0 < r_i <= r_i*
  P:566-567          if sum_i r_i* <= B every request gets r_i*
  Eq. 7  Calibrated Stall-opt: the upper bounds become r_i* + delta
  Alg. A2 lines 2-5: n_i = b_i/t_i + Delta; allocate up to n_i
                     while capacity remains; redistribute to requests with
                     remaining stall.
Baselines: Equal (same share), KV-prop (proportional to the
retrieved KV size), BW-prop (proportional to the zero-stall estimate).

Readings: c8 -- the closed form the paper asserts but does not print is the
KKT solution of Eq. 6, r_i = min(cap_i, lambda*sqrt(s_i)) ("capped
water-filling"); c9 -- delta raises the caps of the same program; c10 -- when
the caps fit in B each request gets its cap and the rest of B is left unused;
c12 -- sum s_i/r_i is strictly convex, so the optimum is unique.
Units are whatever the caller uses consistently (bytes/s in the library).
"""
import math


def zero_stall_rate(s: float, c: float) -> float:
    """r* = s / c."""
    return s / c


def per_layer_stall(s: float, c: float, r: float) -> float:
    """Eq. 4: tau(r) = max(0, s/r - c)."""
    return max(0.0, s / r - c)


def _check(s, c, B):
    if B <= 0:
        raise ValueError("bandwidth cap B must be > 0")
    if len(s) != len(c):
        raise ValueError("s and c differ in length")
    for si, ci in zip(s, c):
        if not (si > 0 and ci > 0):
            raise ValueError("s_i and c_i must be > 0 (requests with no matched bytes "
                             "never enter the layerwise pool, P:405-410)")


def equal(s, c, B):
    _check(s, c, B)
    n = len(s)
    return [B / n for _ in range(n)]


def kv_prop(s, c, B):
    _check(s, c, B)
    tot = sum(s)
    return [B * si / tot for si in s]


def bw_prop(s, c, B):
    _check(s, c, B)
    rs = [zero_stall_rate(si, ci) for si, ci in zip(s, c)]
    tot = sum(rs)
    return [B * r / tot for r in rs]


def water_fill(s, caps, B):
    """argmin sum s_i/r_i  s.t.  sum r_i = B, 0 < r_i <= cap_i   (or r = caps if they fit).

    Iteration: with the capped set F fixed at its caps, the free requests share
    what is left in proportion to sqrt(s_i) (stationarity of Eq. 6's
    Lagrangian, -s_i/r_i^2 + lambda = 0); every free request whose share
    exceeds its cap joins F.  Terminates in at most n rounds.
    """
    n = len(s)
    if sum(caps) <= B:
        return list(caps)                       # P:566-567 and reading c10
    fixed = [False] * n
    r = [0.0] * n
    while True:
        left = B - sum(caps[i] for i in range(n) if fixed[i])
        weight = sum(math.sqrt(s[i]) for i in range(n) if not fixed[i])
        lam = left / weight
        newly = False
        for i in range(n):
            if not fixed[i]:
                r[i] = lam * math.sqrt(s[i])
                if r[i] > caps[i]:
                    fixed[i] = True
                    newly = True
        if not newly:
            break
    for i in range(n):
        if fixed[i]:
            r[i] = caps[i]
    return r


def water_fill_sorted(s, caps, B):
    """Second formulation: sort by cap_i/sqrt(s_i); the first k requests are capped.

    For the optimum, request i is capped iff cap_i/sqrt(s_i) < lambda.  Scan k
    = 0..n and take the first k whose lambda_k = (B - sum_{first k} cap) /
    sum_{rest} sqrt(s) satisfies cap_k/sqrt(s_k) >= lambda_k for the (k+1)-th.
    """
    n = len(s)
    if sum(caps) <= B:
        return list(caps)
    order = sorted(range(n), key=lambda i: caps[i] / math.sqrt(s[i]))
    for k in range(n):
        left = B - sum(caps[order[m]] for m in range(k))
        weight = sum(math.sqrt(s[order[m]]) for m in range(k, n))
        lam = left / weight
        nxt = order[k]
        if caps[nxt] / math.sqrt(s[nxt]) >= lam:
            r = [0.0] * n
            for m in range(n):
                i = order[m]
                r[i] = caps[i] if m < k else lam * math.sqrt(s[i])
            return r
    raise AssertionError("unreachable: sum(caps) > B means some request stays free")


def stall_opt(s, c, B):
    """Eq. 6 with caps r_i* (Stall-opt)."""
    _check(s, c, B)
    return water_fill(s, [zero_stall_rate(si, ci) for si, ci in zip(s, c)], B)


def calibrated_stall_opt(s, c, B, delta):
    """Eq. 7 + Alg. A2 lines 2-5: caps r_i* + delta (Calibrated Stall-opt)."""
    _check(s, c, B)
    if delta < 0:
        raise ValueError("delta must be >= 0")
    return water_fill(s, [zero_stall_rate(si, ci) + delta for si, ci in zip(s, c)], B)


POLICIES = {
    "equal": lambda s, c, B, delta=0.0: equal(s, c, B),
    "kv_prop": lambda s, c, B, delta=0.0: kv_prop(s, c, B),
    "bw_prop": lambda s, c, B, delta=0.0: bw_prop(s, c, B),
    "stall_opt": lambda s, c, B, delta=0.0: stall_opt(s, c, B),
    "cal_stall_opt": lambda s, c, B, delta=0.0: calibrated_stall_opt(s, c, B, delta),
}


def schedule(policy: str, s, c, B, delta=0.0):
    if len(s) == 0:
        if B <= 0:
            raise ValueError("bandwidth cap B must be > 0")
        return []
    return POLICIES[policy](s, c, B, delta)


def epoch_admission(policy: str, running_rates, s, c, B, delta=0.0):
    """One scheduling epoch (Sec. 3.6; Alg. A2 lines 1-6): the waiting requests
    (s_i, c_i) are admitted under the budget the still-running requests leave, B - sum(running),
    with the policy's allocation; rates then stay fixed for the whole load, and bandwidth of a
    request that finishes returns only at the next epoch.  Returns None when nothing is admitted
    (no waiting request, or no budget left)."""
    budget = B - sum(running_rates)
    if len(s) == 0 or budget <= 0:
        return None
    return schedule(policy, s, c, budget, delta)
