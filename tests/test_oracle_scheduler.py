"""Pins for oracle.scheduler: every cell of Table A6, a numeric minimiser, KKT and invariants."""
import math
import random

import numpy as np
import pytest
from scipy.optimize import minimize

from oracle import scheduler as sch
from conftest import read_golden

GBPS = 1e9 / 8          # bytes/s per Gbps (decimal, reading c6)
A5 = {(int(r["context"]), float(r["hit"])): r for r in read_golden("table_a5.csv")}


def profile(context, hit):
    r = A5[(context, hit)]
    s = int(r["cached"]) * 4096                     # bytes per layer (Table A5 caption)
    c = float(r["t_total_ms"]) / 32 / 1e3            # seconds per layer, unrounded (reading c11)
    return s, c


def workloads():
    rows = read_golden("table_a6.csv")
    out = {}
    for r in rows:
        out.setdefault(r["workload"], []).append(r)
    return out


@pytest.mark.parametrize("wl", ["A", "B", "C"])
@pytest.mark.parametrize("policy,tol", [("equal", 0.006), ("kv_prop", 0.006), ("bw_prop", 0.1),
                                        ("stall_opt", 0.006), ("cal_stall_opt", 0.006)])
def test_table_a6(wl, policy, tol):
    rows = workloads()[wl]
    s, c = zip(*[profile(int(r["context"]), float(r["hit"])) for r in rows])
    B = float(rows[0]["cap_gbps"]) * GBPS
    got = sch.schedule(policy, list(s), list(c), B, 5 * GBPS)
    for r, x in zip(rows, got):
        assert abs(x / GBPS - float(r[policy])) <= tol, (wl, policy, r, x / GBPS)


def test_zero_stall_rates_of_table_a6_requests():
    # r* in Gbps: the Stall-opt column equals r* wherever the request is not cut (Workload A rows 1, 3, 4).
    want = {(16384, 0.5): 8.99, (16384, 0.875): 53.35, (65536, 0.5): 3.96,
            (65536, 0.875): 24.81, (32768, 0.5): 6.64, (32768, 0.875): 39.39}
    for k, v in want.items():
        s, c = profile(*k)
        assert abs(sch.zero_stall_rate(s, c) / GBPS - v) <= 0.006
    # "91 Gbps in aggregate, or 111 Gbps after adding the 5 Gbps calibration margin";
    # Workload C: "137 Gbps, or 167 Gbps after calibration".
    ab = sum(sch.zero_stall_rate(*profile(*k)) for k in [(16384, .5), (16384, .875), (65536, .5), (65536, .875)]) / GBPS
    assert round(ab) == 91 and round(ab + 4 * 5) == 111
    cc = sum(sch.zero_stall_rate(*profile(*k)) for k in want) / GBPS
    assert round(cc) == 137 and round(cc + 6 * 5) == 167


def _numeric_opt(s, caps, B):
    """Brute-force reference: SLSQP on Eq. 6 (library minimiser), several starts."""
    n = len(s)
    best = None
    for start in range(4):
        rng = np.random.default_rng(start)
        x0 = np.minimum(np.array(caps) * 0.999, B / n * (0.5 + rng.random(n)))
        x0 = x0 * (B / x0.sum()) if x0.sum() > B else x0
        res = minimize(lambda r: float(np.sum(np.array(s) / r)), x0,
                       jac=lambda r: -np.array(s) / r**2,
                       bounds=[(1e-9 * B, cp) for cp in caps],
                       constraints=[{"type": "eq", "fun": lambda r: float(np.sum(r) - B),
                                     "jac": lambda r: np.ones(n)}],
                       method="SLSQP", options={"ftol": 1e-15, "maxiter": 1000})
        if res.success and (best is None or res.fun < best.fun):
            best = res
    return best


@pytest.mark.parametrize("seed", range(12))
def test_water_fill_matches_numeric_minimiser(seed):
    rng = random.Random(seed)
    n = rng.randint(1, 5)
    s = [rng.uniform(1, 100) for _ in range(n)]
    c = [rng.uniform(0.1, 5) for _ in range(n)]
    caps = [si / ci for si, ci in zip(s, c)]
    B = rng.uniform(0.2, 0.95) * sum(caps)
    r = sch.stall_opt(s, c, B)
    ref = _numeric_opt(s, caps, B)
    assert ref is not None
    obj = sum(si / ri for si, ri in zip(s, r))
    assert obj <= ref.fun * (1 + 1e-7)
    assert np.allclose(r, ref.x, rtol=2e-3, atol=1e-6 * B)


@pytest.mark.parametrize("seed", range(40))
def test_invariants_and_two_formulations(seed):
    rng = random.Random(1000 + seed)
    n = rng.randint(1, 12)
    s = [rng.uniform(1e6, 5e8) for _ in range(n)]
    c = [rng.uniform(1e-4, 0.3) for _ in range(n)]
    B = rng.uniform(0.1, 2.0) * sum(si / ci for si, ci in zip(s, c))
    delta = rng.choice([0.0, rng.uniform(0, 1e9)])
    for policy in ("stall_opt", "cal_stall_opt"):
        r = sch.schedule(policy, s, c, B, delta)
        caps = [si / ci + (delta if policy == "cal_stall_opt" else 0.0) for si, ci in zip(s, c)]
        assert all(0 < ri <= cp * (1 + 1e-12) for ri, cp in zip(r, caps))
        assert math.isclose(sum(r), min(B, sum(caps)), rel_tol=1e-12)
        r2 = sch.water_fill_sorted(s, caps, B)
        assert np.allclose(r, r2, rtol=1e-12)
        # KKT: uncapped requests share one lambda = r_i / sqrt(s_i), at most any capped one's cap ratio... reversed
        free = [i for i in range(n) if r[i] < caps[i] * (1 - 1e-12)]
        if free:
            lam = [r[i] / math.sqrt(s[i]) for i in free]
            assert max(lam) - min(lam) <= 1e-9 * max(lam)
            for i in range(n):
                if i not in free:
                    assert caps[i] / math.sqrt(s[i]) <= max(lam) * (1 + 1e-9)
    for policy in ("equal", "kv_prop", "bw_prop"):
        r = sch.schedule(policy, s, c, B)
        assert math.isclose(sum(r), B, rel_tol=1e-12)


def test_monotone_in_B_and_no_excess():
    rng = random.Random(7)
    s = [rng.uniform(1, 10) for _ in range(6)]
    c = [rng.uniform(0.1, 1) for _ in range(6)]
    caps = [si / ci for si, ci in zip(s, c)]
    prev = None
    for B in np.linspace(0.05, 1.5, 40) * sum(caps):
        r = sch.stall_opt(s, c, B)
        if prev is not None:
            assert all(a >= b - 1e-12 for a, b in zip(r, prev))
        prev = r
        # no request beyond its stall target (reading c10); enough bandwidth -> zero added stall
        assert all(ri <= cp * (1 + 1e-12) for ri, cp in zip(r, caps))
        if B >= sum(caps):
            assert all(sch.per_layer_stall(si, ci, ri) <= 1e-12 for si, ci, ri in zip(s, c, r))


def test_stall_opt_never_worse_than_equal():
    # Eq. 6 objective: Stall-opt minimises sum s_i/r_i over the feasible set that contains Equal when B/n <= r*.
    rng = random.Random(3)
    for _ in range(50):
        n = rng.randint(2, 8)
        s = [rng.uniform(1, 10) for _ in range(n)]
        c = [rng.uniform(0.1, 1) for _ in range(n)]
        B = rng.uniform(0.1, 0.9) * sum(si / ci for si, ci in zip(s, c))
        r = sch.stall_opt(s, c, B)
        tot_opt = sum(sch.per_layer_stall(si, ci, ri) for si, ci, ri in zip(s, c, r))
        tot_eq = sum(sch.per_layer_stall(si, ci, B / n) for si, ci in zip(s, c))
        assert tot_opt <= tot_eq + 1e-12


def test_errors_and_empty():
    with pytest.raises(ValueError):
        sch.schedule("equal", [1.0], [1.0], 0.0)
    with pytest.raises(ValueError):
        sch.schedule("stall_opt", [0.0], [1.0], 1.0)
    with pytest.raises(ValueError):
        sch.schedule("stall_opt", [1.0], [-1.0], 1.0)
    assert sch.schedule("cal_stall_opt", [], [], 5.0, 1.0) == []
    assert sch.stall_opt([4.0], [2.0], 100.0) == [2.0]           # caps fit: r = r*, leftover unused
    assert sch.calibrated_stall_opt([4.0], [2.0], 100.0, 1.0) == [3.0]
    assert sch.stall_opt([4.0, 9.0], [1.0, 1.0], 5.0) == pytest.approx([2.0, 3.0])   # sqrt-proportional


def test_epoch_admission():
    s = [4e9, 9e9]
    c = [1.0, 1.0]
    # nothing running: one epoch is plain scheduling
    assert sch.epoch_admission("stall_opt", [], s, c, 5e9) == pytest.approx(sch.stall_opt(s, c, 5e9))
    # running requests hold their rates: the new ones share what is left, never more than B in total
    r = sch.epoch_admission("equal", [1e9, 1.5e9], s, c, 5e9)
    assert r == pytest.approx([1.25e9, 1.25e9]) and sum(r) + 2.5e9 == pytest.approx(5e9)
    r = sch.epoch_admission("cal_stall_opt", [3e9], s, c, 5e9, 0.5e9)
    assert sum(r) <= 2e9 * (1 + 1e-12)
    assert sch.epoch_admission("equal", [5e9], s, c, 5e9) is None        # budget exhausted: wait
    assert sch.epoch_admission("equal", [1e9], [], [], 5e9) is None       # nobody waiting
