"""The bench's in-run verification (benchlib/verify.py) on CPU: the GPU-side digest formula (torch
int64 wrap-around, run here on CPU tensors) equals the oracle side's u64 digest for a request
placed into a paged cache by the oracle's own scatter, and a single corrupted or swapped row
changes it; the sampled full check compares against the oracle's Alg. A1 gather."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import synth  # noqa: E402
from benchlib import verify  # noqa: E402
from oracle import keys as okeys  # noqa: E402
from oracle.assemble import gather_layer, scatter_paged_advanced_index  # noqa: E402
from oracle.descriptor import PagedTarget, build_descriptor  # noqa: E402
from oracle.geometry import Layout, chunk_bytes, chunk_layer_bytes, row_bytes  # noqa: E402
from oracle.store import ChunkStore  # noqa: E402


def _placed(lay, seed, N, Bs=16, pool_factor=1.5):
    (tok,), (ids,) = synth.family_streams(seed, lay.chunk_tokens, 0, [N])
    keys = okeys.chunk_keys(tok, lay.chunk_tokens)
    st = ChunkStore(lay)
    st.put(keys, synth.payloads(seed, ids, chunk_bytes(lay)))
    L, G, row = lay.num_layers, lay.chunk_tokens, row_bytes(lay)
    need = -(-N * G // Bs)
    pool = int(need * pool_factor)
    bt = synth.block_table(seed + 1, need, pool).tolist()
    per_kv = pool * Bs * row
    kb = [l * 2 * per_kv for l in range(L)]
    desc = build_descriptor(st, keys, lay, PagedTarget(kb, [x + per_kv for x in kb], Bs * row, row,
                                                       lay.head_dim * lay.elem_bytes, Bs, bt, 0))
    mem = synth.sentinel(L * 2 * per_kv)
    for l in range(L):
        scatter_paged_advanced_index(gather_layer(st, desc, l), l, desc, mem)
    cache = torch.from_numpy(mem).view(L, 2, pool, Bs, row)
    return keys, ids, bt, cache, st, desc


def test_digest_sides_agree_and_detect_changes():
    lay = Layout(3, 2, 32, 2, 16)
    N, seed = 9, 3
    keys, ids, bt, cache, st, desc = _placed(lay, seed, N)
    S = chunk_layer_bytes(lay)
    T = verify.digest_table(S)
    idx = verify.slot_index(torch, "cpu", bt, N * lay.chunk_tokens, 16)
    got = verify.gpu_digests(torch, cache, idx, N, lay.chunk_tokens, torch.from_numpy(T.view(np.int64)))
    fam = verify.FamilyDigests(seed, ids, N, lay.num_layers, S, T, threads=2)
    assert np.array_equal(got, fam.request(N))
    # a prefix of the family: the first 5 chunks
    idx5 = verify.slot_index(torch, "cpu", bt, 5 * lay.chunk_tokens, 16)
    assert np.array_equal(verify.gpu_digests(torch, cache, idx5, 5, 16, torch.from_numpy(T.view(np.int64))),
                          fam.request(5))
    # one flipped byte in layer 1, then two swapped token rows in layer 2
    bad = cache.clone()
    r = bad[1, 0].reshape(-1, row_bytes(lay))
    r[int(idx[7])][3] ^= 1
    d = verify.gpu_digests(torch, bad, idx, N, 16, torch.from_numpy(T.view(np.int64)))
    assert d[0] == got[0] and d[1] != got[1] and d[2] == got[2]
    bad = cache.clone()
    r = bad[2, 1].reshape(-1, row_bytes(lay))
    a, b = int(idx[4]), int(idx[40])
    tmp = r[a].clone()
    r[a] = r[b]
    r[b] = tmp
    d = verify.gpu_digests(torch, bad, idx, N, 16, torch.from_numpy(T.view(np.int64)))
    assert d[2] != got[2] and d[0] == got[0]


def test_full_check_against_oracle_gather():
    lay = Layout(2, 2, 32, 2, 16)
    keys, ids, bt, cache, st, desc = _placed(lay, 8, 6)
    idx = verify.slot_index(torch, "cpu", bt, 6 * 16, 16)
    ok, nbytes, _, _ = verify.full_check(torch, lay, 8, keys, ids, cache, idx, [0, 1])
    assert ok and nbytes == 2 * 6 * chunk_layer_bytes(lay)
    cache[1, 1, bt[0], 0, 0] ^= 0xFF
    ok, _, _, _ = verify.full_check(torch, lay, 8, keys, ids, cache, idx, [1])
    assert not ok


def test_fill_store_scattered_interleaves_and_puts_synth_bytes():
    """fill_store_scattered: every (key, payload) pair of every request is put exactly once, with
    the synth payload fill_store would put, in an order that interleaves the requests (so a
    request's chunks land at scattered slots of an append-only slab)."""
    lay = Layout(2, 2, 16, 2, 16)
    cb = chunk_bytes(lay)

    class Rec:
        def __init__(self):
            self.keys, self.rows = [], []

        def put_chunks(self, keys, pl):
            self.keys += [bytes(k) for k in np.asarray(keys)]
            self.rows += [r.copy() for r in pl]

    reqs = []
    for r in range(3):
        (tok,), (ids,) = synth.family_streams(300 + r, 16, 0, [20])
        reqs.append((np.frombuffer(b"".join(okeys.chunk_keys(tok, 16)), np.uint8).reshape(-1, 32), 300 + r, ids))
    rec = Rec()
    verify.fill_store_scattered(rec, reqs, cb, order_seed=5, batch=7, threads=2)
    want = {bytes(k): synth.chunk_payload(seed, pid, cb) for keys, seed, ids in reqs for k, pid in zip(keys, ids)}
    assert len(rec.keys) == len(want) == 60 and set(rec.keys) == set(want)
    for k, row in zip(rec.keys, rec.rows):
        assert np.array_equal(row, want[k])
    owner = {bytes(k): r for r, (keys, _, _) in enumerate(reqs) for k in keys}
    slots_of_0 = [i for i, k in enumerate(rec.keys) if owner[k] == 0]
    assert slots_of_0 != list(range(slots_of_0[0], slots_of_0[0] + 20))   # not one contiguous run
