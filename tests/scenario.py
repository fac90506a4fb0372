"""Test scenarios: the same seeded request run through the CUDA library and through the oracle.

Both sides get identical inputs from ``synth`` (tokens, payload bytes, block tables); each side
computes its own keys, descriptor and result.  Destination memory is one byte buffer: a CUDA
uint8 tensor for the library, a numpy array for the oracle, with every target address expressed
as base + offset so the two layouts coincide byte for byte.
"""
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

import synth
from oracle import keys as okeys
from oracle.assemble import fetch_layerwise as oracle_fetch, gather_layer, scatter_paged_advanced_index
from oracle.descriptor import FlatTarget as OFlat, PagedTarget as OPaged, build_descriptor as obuild
from oracle.geometry import Layout as OLayout, chunk_bytes, chunk_layer_bytes, row_bytes, head_bytes
from oracle.store import ChunkStore


@dataclass
class Request:
    tokens: np.ndarray
    payload_ids: list
    n_chunks: int


@dataclass
class Dest:
    """Offsets (bytes, relative to the destination buffer) of a paged or flat target."""
    kind: str                      # "nhd", "hnd" or "flat"
    size: int
    k_off: List[int] = field(default_factory=list)
    v_off: List[int] = field(default_factory=list)
    block_stride: int = 0
    token_stride: int = 0
    head_stride: int = 0
    block_size: int = 0
    block_table: List[int] = field(default_factory=list)
    first_token: int = 0
    flat_off: int = 0
    flat_cap: int = 0


def make_dest(lay: OLayout, n_chunks: int, kind: str, Bs: int = 16, first_token: int = 0,
              pool_factor: float = 1.5, seed: int = 0, pad: int = 256) -> Dest:
    L, G = lay.num_layers, lay.chunk_tokens
    row, hd, S = row_bytes(lay), head_bytes(lay), chunk_layer_bytes(lay)
    if kind == "flat":
        W = n_chunks * L * S
        return Dest("flat", pad + W + pad, flat_off=pad, flat_cap=W)
    n_tok = first_token + n_chunks * G
    need = -(-n_tok // Bs)
    pool = max(need, int(need * pool_factor))
    bt = synth.block_table(seed, need, pool).tolist()
    if kind == "nhd":       # vLLM FlashAttention: [L][2][pool][Bs][n_kv][d]
        per_kv = pool * Bs * row
        k = [pad + l * 2 * per_kv for l in range(L)]
        v = [x + per_kv for x in k]
        return Dest("nhd", pad + L * 2 * per_kv + pad, k, v, Bs * row, row, hd, Bs, bt, first_token)
    if kind == "hnd":       # FlashInfer HND: [L][pool][2][n_kv][Bs][d]
        blk = 2 * lay.kv_heads * Bs * hd
        k = [pad + l * pool * blk for l in range(L)]
        v = [x + lay.kv_heads * Bs * hd for x in k]
        return Dest("hnd", pad + L * pool * blk + pad, k, v, blk, hd, Bs * hd, Bs, bt, first_token)
    raise ValueError(kind)


def requests_family(lay: OLayout, seed: int, shared: int, own: Sequence[int] = (), tails=None):
    streams, ids = synth.family_streams(seed, lay.chunk_tokens, shared, list(own), tails)
    return [Request(t, i, len(i)) for t, i in zip(streams, ids)]


def payload_stack(lay: OLayout, seed: int, ids) -> np.ndarray:
    return synth.payloads(seed, ids, chunk_bytes(lay))


# ---- oracle side ---------------------------------------------------------------------------------
def oracle_result(lay: OLayout, seed: int, req: Request, dest: Dest, layers=None) -> np.ndarray:
    """Expected destination bytes (sentinel 0xA5 elsewhere) for fetching req's whole chain."""
    st = ChunkStore(lay)
    ks = okeys.chunk_keys(req.tokens, lay.chunk_tokens)[:req.n_chunks]
    st.put(ks, payload_stack(lay, seed, req.payload_ids[:req.n_chunks]))
    dst = synth.sentinel(dest.size)
    desc = obuild(st, ks, lay, oracle_target(dest))
    if layers is None:
        oracle_fetch(st, desc, dst)
    else:
        for l in layers:
            B = gather_layer(st, desc, l)
            scatter_paged_advanced_index(B, l, desc, dst)
    return dst


def oracle_target(dest: Dest):
    if dest.kind == "flat":
        return OFlat(dest.flat_off, dest.flat_cap)
    return OPaged(dest.k_off, dest.v_off, dest.block_stride, dest.token_stride, dest.head_stride,
                  dest.block_size, dest.block_table, dest.first_token)


# ---- library side --------------------------------------------------------------------------------
def sentinel_buffer(size: int, device="cuda"):
    """A destination buffer of 0xA5 bytes, filled before any later work on ANY stream: the fill runs
    on torch's current stream, the fetches on the tests' own non-blocking streams, which are not
    ordered after it."""
    import torch
    buf = torch.full((int(size),), 0xA5, dtype=torch.uint8, device=device)
    torch.cuda.current_stream(buf.device).synchronize()
    return buf


def lib_target(oc, dest: Dest, base: int):
    if dest.kind == "flat":
        return oc.FlatTarget(base + dest.flat_off, dest.flat_cap)
    return oc.PagedTarget([base + x for x in dest.k_off], [base + x for x in dest.v_off], dest.block_stride,
                          dest.token_stride, dest.head_stride, dest.block_size, dest.block_table, dest.first_token)


class SynthStore:
    """Oracle-side chunk store whose objects are regenerated from ``synth`` on demand: RangeGet(H, o,
    S) (Alg. A1 line 5) returns bytes [o, o+S) of the chunk's seeded payload.  For at-size checks
    (8-9 GiB corpora) that a dict of payloads would not hold; what it returns equals what
    ``oracle.store.ChunkStore`` would return after put()s of the same payloads."""

    def __init__(self, seed, keys, payload_ids):
        self.seed = seed
        self.ids = {bytes(k): pid for k, pid in zip(keys, payload_ids)}

    def __contains__(self, key):
        return bytes(key) in self.ids

    def range_get(self, key, offset, length):
        return synth.chunk_payload_range(self.seed, self.ids[bytes(key)], offset, length).tobytes()


def put_in_batches(store, lay: OLayout, seed, keys, payload_ids, batch=256):
    """Library-side puts of a large corpus, `batch` chunks of synth payload at a time."""
    n_new = 0
    for i in range(0, len(payload_ids), batch):
        n_new += store.put_chunks(keys[i:i + batch], payload_stack(lay, seed, payload_ids[i:i + batch]))
    return n_new


def oracle_layer(lay: OLayout, ostore, okeys_list, dest: Dest, layer: int):
    """Expected bytes of layer `layer`'s region of a paged NHD destination (its K and V caches,
    [2][pool][Bs][row], sentinel 0xA5 where no token lands) and the region's offset: Alg. A1's
    gather (oracle.assemble.gather_layer) of the layer, then the paged scatter into a buffer holding
    just that region (the target's bases rebased to it)."""
    assert dest.kind == "nhd"
    lo = dest.k_off[layer]
    hi = dest.v_off[layer] + (dest.v_off[layer] - dest.k_off[layer])
    rebased = OPaged([x - lo for x in dest.k_off], [x - lo for x in dest.v_off], dest.block_stride,
                     dest.token_stride, dest.head_stride, dest.block_size, dest.block_table, dest.first_token)
    desc = obuild(ostore, okeys_list, lay, rebased)
    region = synth.sentinel(hi - lo)
    scatter_paged_advanced_index(gather_layer(ostore, desc, layer), layer, desc, region)
    return lo, region
