"""Pins for oracle.stall: Eq. 3 closed forms, equivalence with a discrete-event simulation, and the
free-running pipeline (equal to Eq. 3 for uniform layers, never above it)."""
import random

import pytest

from oracle import stall


def test_eq3_closed_forms():
    assert stall.eq3_ttft([3.0], [4.0]) == 7.0                       # L = 1 -> X + C
    L, X, C = 32, 1.0, 2.5
    assert stall.eq3_ttft([X] * L, [C] * L) == pytest.approx(X + L * C)       # X <= C: only X_0 exposed
    X, C = 3.0, 2.0
    assert stall.eq3_ttft([X] * L, [C] * L) == pytest.approx(L * X + C)       # X > C: transfer bound
    with pytest.raises(ValueError):
        stall.eq3_ttft([], [])


@pytest.mark.parametrize("seed", range(30))
def test_eq3_is_one_layer_prefetch_des(seed):
    rng = random.Random(seed)
    L = rng.randint(1, 40)
    X = [rng.uniform(0, 3) for _ in range(L)]
    C = [rng.uniform(0, 3) for _ in range(L)]
    assert stall.eq3_ttft(X, C) == pytest.approx(stall.simulate(X, C, 1))
    assert stall.free_running_ttft(X, C) == pytest.approx(stall.simulate(X, C, None))
    assert stall.free_running_ttft(X, C) <= stall.eq3_ttft(X, C) + 1e-9
    if L > 1:                                    # deeper prefetch never hurts
        assert stall.simulate(X, C, 2) <= stall.simulate(X, C, 1) + 1e-9


@pytest.mark.parametrize("seed", range(20))
def test_uniform_layers_models_coincide(seed):
    rng = random.Random(100 + seed)
    L = rng.randint(1, 80)
    X, C = rng.uniform(0, 5), rng.uniform(0, 5)
    assert stall.free_running_ttft([X] * L, [C] * L) == pytest.approx(stall.eq3_ttft([X] * L, [C] * L))


def test_free_running_stall_accounting():
    ready = [1.0, 1.5, 2.0, 6.0]
    C = [1.0, 1.0, 1.0, 1.0]
    ttft, start, end, st = stall.free_running(ready, C)
    assert start == [1.0, 2.0, 3.0, 6.0] and end == [2.0, 3.0, 4.0, 7.0]
    assert st == [1.0, 0.0, 0.0, 2.0]
    assert ttft == 7.0 and stall.added_ttft(ttft, C) == 3.0 == sum(st)


def test_hot_layers_for_closed_form_and_invariants():
    """The brute-force mirror depth equals the closed form K = max(1, ceil(L - (L-1) C / X)) that
    follows from requiring (l - K + 1) X <= l C for the last layer; K - 1 layers leave a stall."""
    import math
    import random
    rng = random.Random(3)
    for _ in range(300):
        L = rng.randint(1, 80)
        X = rng.uniform(0.01, 5.0)
        C = rng.uniform(0.01, 5.0)
        K = stall.hot_layers_for(X, C, L)
        closed = max(1, min(L, math.ceil(L - (L - 1) * C / X - 1e-12)))
        assert K == closed, (L, X, C, K, closed)
        if K > 1:
            ttft = stall.free_running(stall.mirrored_ready(K - 1, X, L), [C] * L)[0]
            assert stall.added_ttft(ttft, [C] * L) > 0
    assert stall.hot_layers_for(1.0, 2.0, 32) == 1          # compute outpaces the link: mirror layer 0 only
    assert stall.hot_layers_for(2.0, 1.0, 33) == 17         # X = 2C: half the layers (33 - 32/2 = 17)
