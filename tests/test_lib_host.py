"""libobjcache on the host (no GPU): the library loads, exports every symbol the header declares, and
its host-side steps -- SHA-256 chain keys, Eq. 1 geometry, the Eq. 2 rule and the bandwidth
scheduler -- equal the oracle.  Data-path calls without a GPU must fail loudly (OC_ECUDA/OC_EINVAL)."""
import os
import random
import re
import subprocess

import numpy as np
import pytest

import paper_2605_22850_b200 as oc
import synth
from oracle import keys as okeys
from oracle import scheduler as osch
from oracle import geometry as ogeo
from conftest import ROOT, read_golden

HEADER = os.path.join(ROOT, "include", "objcache.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"OC_API\s+[\w\s\*]+?\b(oc_\w+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    syms = declared_symbols()
    assert len(syms) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", oc.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (oc_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    # nothing else leaks out of the library's C ABI
    assert not [s for s in exported if s not in syms]
    assert set(syms) == set(oc.EXPORTED)


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", oc.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


@pytest.mark.parametrize("row", read_golden("sha256_fips180.csv"))
def test_sha256_fips_vectors(row):
    msg = b"a" * 1000000 if row["message"] == "@million_a" else row["message"].encode()
    assert oc.sha256(msg).hex() == row["digest"]


@pytest.mark.parametrize("seed", range(8))
def test_chunk_keys_equal_oracle(seed):
    rng = random.Random(seed)
    G = rng.choice([1, 3, 16, 64, 100])
    t = synth.tokens(seed, rng.randint(0, 20 * G + G - 1))
    parent = bytes(rng.getrandbits(8) for _ in range(32)) if seed % 2 else None
    mine = oc.chunk_keys(t, G, parent)
    ref = okeys.chunk_keys(t, G, parent if parent else okeys.ROOT)
    assert [bytes(k) for k in mine] == ref


def test_chunk_keys_edge_cases():
    assert oc.chunk_keys(np.zeros(0, np.uint32), 16).shape == (0, 32)
    assert oc.chunk_keys(np.arange(15, dtype=np.uint32), 16).shape == (0, 32)
    with pytest.raises(oc.ObjcacheError) as e:
        oc.chunk_keys(np.arange(4, dtype=np.uint32), 0)
    assert e.value.code == oc.OC_EINVAL
    big = np.array([2**32 - 1] * 16, dtype=np.uint32)
    assert bytes(oc.chunk_keys(big, 16)[0]) == okeys.chunk_keys(big.tolist(), 16)[0]


@pytest.mark.parametrize("lay", [synth.TINY, synth.LLAMA3_8B, synth.LLAMA3_70B, synth.with_chunk_tokens(synth.LLAMA3_8B, 256)])
def test_geometry_equals_oracle(lay):
    L = ogeo.Layout(*lay.as_tuple())
    assert oc.geometry(lay) == (ogeo.row_bytes(L), ogeo.chunk_layer_bytes(L), ogeo.chunk_bytes(L))


def test_geometry_rejects_zero_fields():
    with pytest.raises(oc.ObjcacheError):
        oc.geometry((0, 8, 128, 2, 16))


def test_select_mode_equals_eq2():
    theta = 512 * 2**20
    for W in (0, 1, theta - 1, theta, theta + 1, 2**40):
        want = oc.DELIVER_CHUNK_MAJOR if ogeo.delivery_mode(W, theta) == "chunkwise" else oc.DELIVER_LAYER_MAJOR
        assert oc.select_mode(W, theta) == want


def _a6_workloads():
    a5 = {(int(r["context"]), float(r["hit"])): r for r in read_golden("table_a5.csv")}
    out = {}
    for r in read_golden("table_a6.csv"):
        a = a5[(int(r["context"]), float(r["hit"]))]
        out.setdefault(r["workload"], ([], [], float(r["cap_gbps"]) * 1e9 / 8))
        out[r["workload"]][0].append(int(a["cached"]) * 4096)
        out[r["workload"]][1].append(float(a["t_total_ms"]) / 32 / 1e3)
    return out


@pytest.mark.parametrize("policy", list(oc.POLICIES))
def test_scheduler_equals_oracle_on_table_a6(policy):
    for wl, (s, c, B) in _a6_workloads().items():
        mine = oc.schedule_bandwidth(policy, s, c, B, 5e9 / 8)
        ref = osch.schedule(policy, s, c, B, 5e9 / 8)
        assert np.allclose(mine, ref, rtol=1e-12, atol=0), (wl, policy)


@pytest.mark.parametrize("seed", range(30))
def test_scheduler_equals_oracle_random(seed):
    rng = random.Random(seed)
    n = rng.randint(1, 64)
    s = [rng.uniform(1e3, 1e9) for _ in range(n)]
    c = [rng.uniform(1e-5, 1.0) for _ in range(n)]
    B = rng.uniform(0.05, 1.5) * sum(si / ci for si, ci in zip(s, c))
    delta = rng.uniform(0, 1e9)
    for policy in oc.POLICIES:
        assert np.allclose(oc.schedule_bandwidth(policy, s, c, B, delta),
                           osch.schedule(policy, s, c, B, delta), rtol=1e-11, atol=0)


def test_scheduler_errors():
    with pytest.raises(oc.ObjcacheError):
        oc.schedule_bandwidth("equal", [1.0], [1.0], 0.0)
    with pytest.raises(oc.ObjcacheError):
        oc.schedule_bandwidth("stall_opt", [1.0], [0.0], 1.0)
    with pytest.raises(oc.ObjcacheError):
        oc.schedule_bandwidth("cal_stall_opt", [1.0], [1.0], 1.0, -1.0)
    with pytest.raises(oc.ObjcacheError):
        oc.schedule_bandwidth(9, [1.0], [1.0], 1.0)
    assert oc.schedule_bandwidth("stall_opt", [], [], 1.0).shape == (0,)


def test_data_path_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(oc.ObjcacheError) as e:
        oc.Store(synth.TINY, 4)
    assert e.value.code in (oc.OC_ECUDA, oc.OC_EINVAL)


def test_abi_version():
    assert oc.abi_version() == 1


def test_sha256_padding_boundaries_vs_hashlib():
    import hashlib
    data = bytes(range(256)) * 8
    for n in (0, 1, 55, 56, 57, 63, 64, 65, 96, 119, 120, 127, 128, 129, 1000, 2048):
        assert oc.sha256(data[:n]) == hashlib.sha256(data[:n]).digest(), n


def test_hot_layers_for_equals_oracle():
    import random
    from oracle import stall as ostall
    rng = random.Random(24)
    for _ in range(500):
        L = rng.randint(1, 80)
        X, C = rng.uniform(0.01, 5.0), rng.uniform(0.01, 5.0)
        assert oc.hot_layers_for(X, C, L) == ostall.hot_layers_for(X, C, L), (X, C, L)
    for bad in ((0.0, 1.0, 4), (1.0, -1.0, 4), (1.0, 1.0, 0), (float("inf"), 1.0, 4)):
        with pytest.raises(oc.ObjcacheError) as e:
            oc.hot_layers_for(*bad)
        assert e.value.code == oc.OC_EINVAL


def test_slot_pitch_rule():
    """oc_slot_pitch (include/objcache.h): dense slots for pinned-host slabs and chunks < 1 MiB; an
    HBM slab spaces slots by the smallest multiple of 32 KiB >= L*S whose granule count has no
    factor 3, 5 or 7 (the measured B200 rule, profiles/r02_pitch_sweep.txt)."""
    q = 32768
    for lay, pitch in (((32, 8, 128, 2, 16), 2 << 20),            # Llama-3-8B: 64 granules, unchanged
                       ((80, 8, 128, 2, 16), 163 * q),            # Llama-3-70B: 160 -> 163
                       ((40, 8, 128, 2, 16), 82 * q),             # 80 -> 81 (3^4) -> 82
                       ((48, 8, 128, 2, 16), 97 * q),             # 96 -> 97
                       ((4, 2, 16, 2, 4), 4 * 2 * 4 * 2 * 16 * 2)):  # tiny: dense
        assert oc.slot_pitch(lay, oc.TIER_HBM) == pitch, lay
        assert oc.slot_pitch(lay, oc.TIER_PINNED_HOST) == oc.geometry(lay)[2]
    for L in range(1, 257):
        for n_kv, d in ((8, 128), (4, 64), (16, 128), (1, 80)):
            lay = (L, n_kv, d, 2, 16)
            ch = oc.geometry(lay)[2]
            p = oc.slot_pitch(lay, oc.TIER_HBM)
            if ch < 1 << 20:
                assert p == ch
                continue
            assert p >= ch and p % q == 0 and p - ch < 6 * q
            u = p // q
            assert u % 3 and u % 5 and u % 7
            assert all(v % 3 == 0 or v % 5 == 0 or v % 7 == 0 for v in range(-(-ch // q), u))   # the smallest
    with pytest.raises(oc.ObjcacheError):
        oc.slot_pitch((32, 8, 128, 2, 16), 7)
