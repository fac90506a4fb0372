"""Pins for oracle.assemble / oracle.descriptor: Alg. A1 by transposition, two scatter formulations,
read-back through the block table, sentinel bytes, and the descriptor's error conventions."""
import numpy as np
import pytest

import synth
from oracle import keys
from oracle.assemble import (fetch_layerwise, gather_layer, scatter_paged,
                             scatter_paged_advanced_index)
from oracle.descriptor import (FlatTarget, NotFoundError, PagedTarget, RangeError,
                               build_descriptor)
from oracle.geometry import Layout, chunk_bytes, chunk_layer_bytes, row_bytes, head_bytes
from oracle.store import ChunkStore


def make_store(lay, n_chunks, seed=0):
    G = lay.chunk_tokens
    (t,), (ids,) = synth.family_streams(seed, G, 0, [n_chunks])
    ks = keys.chunk_keys(t, G)
    pl = synth.payloads(seed, ids, chunk_bytes(lay))
    st = ChunkStore(lay)
    st.put(ks, pl)
    return st, ks, pl


def paged_nhd(lay, N, Bs, first_token, pool, seed=0, base=0):
    """FlashAttention-style [L][2][pool][Bs][n_kv][d] cache inside one byte array."""
    row = row_bytes(lay)
    per_kv = pool * Bs * row
    n_tok = first_token + N * lay.chunk_tokens
    bt = synth.block_table(seed, -(-n_tok // Bs), pool).tolist()
    k_base = [base + l * 2 * per_kv for l in range(lay.num_layers)]
    v_base = [kb + per_kv for kb in k_base]
    tgt = PagedTarget(k_base, v_base, Bs * row, row, head_bytes(lay), Bs, bt, first_token)
    return tgt, base + lay.num_layers * 2 * per_kv


def paged_hnd(lay, N, Bs, first_token, pool, seed=0):
    """FlashInfer-HND-style [L][pool][2][n_kv][Bs][d] cache."""
    hd = head_bytes(lay)
    blk = 2 * lay.kv_heads * Bs * hd
    n_tok = first_token + N * lay.chunk_tokens
    bt = synth.block_table(seed + 1, -(-n_tok // Bs), pool).tolist()
    k_base = [l * pool * blk for l in range(lay.num_layers)]
    v_base = [kb + lay.kv_heads * Bs * hd for kb in k_base]
    tgt = PagedTarget(k_base, v_base, blk, hd, Bs * hd, Bs, bt, first_token)
    return tgt, lay.num_layers * pool * blk


@pytest.mark.parametrize("lay", [Layout(2, 2, 16, 2, 16), Layout(3, 1, 8, 2, 4), Layout(4, 3, 8, 4, 8)])
def test_gather_equals_transpose_of_chunk_stack(lay):
    st, ks, pl = make_store(lay, 7)
    desc = build_descriptor(st, ks, lay, FlatTarget(0, 10**9))
    S = chunk_layer_bytes(lay)
    stack = pl.reshape(7, lay.num_layers, S)               # [N][L][S] chunk-major objects (KV_L2TD)
    layer_major = stack.transpose(1, 0, 2)                   # [L][N][S]
    for l in range(lay.num_layers):
        assert gather_layer(st, desc, l) == layer_major[l].tobytes()
    # invertibility: reshaping the layer-major payloads back recovers every chunk
    B = np.stack([np.frombuffer(gather_layer(st, desc, l), np.uint8).reshape(7, S)
                  for l in range(lay.num_layers)])
    assert np.array_equal(B.transpose(1, 0, 2).reshape(7, -1), pl)


def test_flat_delivery_layout_and_events():
    lay = Layout(2, 2, 16, 2, 16)
    st, ks, pl = make_store(lay, 10)
    W = 10 * 2 * chunk_layer_bytes(lay)
    dst = synth.sentinel(W + 64)
    desc = build_descriptor(st, ks, lay, FlatTarget(32, W))
    events = fetch_layerwise(st, desc, dst)
    assert events == [0, 1]                                   # NotifyLayerReady in increasing l
    assert np.all(dst[:32] == 0xA5) and np.all(dst[32 + W:] == 0xA5)
    S = chunk_layer_bytes(lay)
    want = pl.reshape(10, 2, S).transpose(1, 0, 2).reshape(-1)
    assert np.array_equal(dst[32:32 + W], want)


@pytest.mark.parametrize("Bs", [1, 8, 16, 32])
@pytest.mark.parametrize("first_token", [0, 5, 16])
def test_paged_two_formulations_and_readback(Bs, first_token):
    lay = Layout(2, 2, 16, 2, 16)
    N = 10
    st, ks, pl = make_store(lay, N)
    pool = 200 // Bs + 8
    tgt, size = paged_nhd(lay, N, Bs, first_token, pool)
    desc = build_descriptor(st, ks, lay, tgt)
    a = synth.sentinel(size)
    b = synth.sentinel(size)
    for l in range(lay.num_layers):
        B = gather_layer(st, desc, l)
        scatter_paged(B, l, desc, a)
        scatter_paged_advanced_index(B, l, desc, b)
    assert np.array_equal(a, b)
    # read back each token row through the block table -> the layer-major payload
    row, G, S = row_bytes(lay), lay.chunk_tokens, chunk_layer_bytes(lay)
    touched = np.zeros(size, bool)
    for l in range(lay.num_layers):
        B = np.frombuffer(gather_layer(st, desc, l), np.uint8).reshape(N, 2, G, row)
        for kv in (0, 1):
            base = (tgt.k_base, tgt.v_base)[kv][l]
            for u in range(first_token, first_token + N * G):
                off = base + tgt.block_table[u // Bs] * tgt.block_stride + (u % Bs) * row
                j, t = divmod(u - first_token, G)
                assert np.array_equal(a[off:off + row], B[j, kv, t])
                touched[off:off + row] = True
    assert touched.sum() == 2 * N * S                           # exactly W bytes written
    assert np.all(a[~touched] == 0xA5)                          # the rest keeps its sentinel (c5)


def test_hnd_layout_by_numpy_view():
    lay = Layout(2, 3, 8, 2, 16)
    N, Bs, pool, ft = 6, 8, 40, 3
    st, ks, pl = make_store(lay, N, seed=4)
    tgt, size = paged_hnd(lay, N, Bs, ft, pool)
    desc = build_descriptor(st, ks, lay, tgt)
    dst = synth.sentinel(size)
    fetch_layerwise(st, desc, dst)
    hd, G, nkv = head_bytes(lay), lay.chunk_tokens, lay.kv_heads
    cache = dst.reshape(lay.num_layers, pool, 2, nkv, Bs, hd)
    for l in range(lay.num_layers):
        B = np.frombuffer(gather_layer(st, desc, l), np.uint8).reshape(N, 2, G, nkv, hd)
        for u in range(ft, ft + N * G):
            j, t = divmod(u - ft, G)
            blk = tgt.block_table[u // Bs]
            for kv in (0, 1):
                assert np.array_equal(cache[l, blk, kv, :, u % Bs], B[j, kv, t])


def test_flat_is_paged_with_identity_table():
    # The flat client buffer equals a paged target with Bs = G, block_stride = S, identity block table.
    lay = Layout(3, 2, 16, 2, 8)
    N = 5
    st, ks, _ = make_store(lay, N, seed=9)
    S, row, G = chunk_layer_bytes(lay), row_bytes(lay), lay.chunk_tokens
    W = N * lay.num_layers * S
    flat = synth.sentinel(W)
    fetch_layerwise(st, build_descriptor(st, ks, lay, FlatTarget(0, W)), flat)
    k_base = [l * N * S for l in range(lay.num_layers)]
    tgt = PagedTarget(k_base, [k + G * row for k in k_base], S, row, head_bytes(lay), G, list(range(N)), 0)
    paged = synth.sentinel(W)
    fetch_layerwise(st, build_descriptor(st, ks, lay, tgt), paged)
    assert np.array_equal(flat, paged)


def test_descriptor_errors():
    lay = Layout(2, 2, 16, 2, 16)
    st, ks, _ = make_store(lay, 4)
    with pytest.raises(ValueError):
        build_descriptor(st, [], lay, FlatTarget(0, 10**6))
    missing = keys.chunk_key(bytes(32), [1, 2, 3])
    with pytest.raises(NotFoundError) as e:
        build_descriptor(st, ks[:2] + [missing] + ks[2:], lay, FlatTarget(0, 10**6))
    assert e.value.index == 2
    with pytest.raises(RangeError):
        build_descriptor(st, ks, lay, FlatTarget(0, 4 * 2 * chunk_layer_bytes(lay) - 1))
    tgt, _ = paged_nhd(lay, 4, 16, 0, 8)
    tgt.block_table = tgt.block_table[:3]
    with pytest.raises(RangeError):
        build_descriptor(st, ks, lay, tgt)
    tgt, _ = paged_nhd(lay, 4, 16, 0, 8)
    tgt.block_table[1] = tgt.block_table[0]
    with pytest.raises(ValueError):
        build_descriptor(st, ks, lay, tgt)


@pytest.mark.parametrize("maker,Bs,first", [(paged_nhd, 16, 0), (paged_nhd, 8, 5), (paged_hnd, 8, 3)])
def test_offload_is_inverse_of_scatter(maker, Bs, first):
    """offload(scatter(chunks)) == chunks, and scatter(offload(cache)) reproduces the cache rows."""
    from oracle.assemble import offload_paged
    lay = Layout(2, 2, 16, 2, 16)
    N = 6
    st, ks, pl = make_store(lay, N, seed=21)
    tgt, size = maker(lay, N, Bs, first, 200 // Bs + 8)
    cache = synth.sentinel(size)
    fetch_layerwise(st, build_descriptor(st, ks, lay, tgt), cache)
    fresh = ChunkStore(lay)
    assert offload_paged(fresh, ks, lay, tgt, cache) == N
    for k, p in zip(ks, pl):
        assert fresh.get(k) == p.tobytes()
    assert offload_paged(fresh, ks, lay, tgt, cache) == 0            # dedup by key
    # random cache -> offload -> scatter into a sentinel copy reproduces exactly the touched rows
    rng = np.random.default_rng(5)
    rand = rng.integers(0, 256, size, dtype=np.uint8)
    st2 = ChunkStore(lay)
    offload_paged(st2, ks, lay, tgt, rand)
    back = synth.sentinel(size)
    fetch_layerwise(st2, build_descriptor(st2, ks, lay, tgt), back)
    touched = back != 0xA5
    assert np.array_equal(back[touched], rand[touched])
    S = chunk_layer_bytes(lay)
    assert np.count_nonzero(touched) >= 2 * N * S - np.count_nonzero(rand[~touched] == 0xA5) - 2 * N * S // 64
