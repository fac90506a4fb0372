"""Layer-major assembly and paged delivery (oracle; test infrastructure only).

Alg. A1 ("ObjectCache layerwise GET"):
    1 for l = 0..L-1
    2   B_l <- empty
    3   for each key H_j in chunk_keys
    4     o <- l * S
    5     append RangeGet(H_j, o, S) to B_l
    6   RDMAWrite(client_buffer[l], B_l)
    7   NotifyLayerReady(l)
Sec. 3.3: slices are appended "in prefix order" (reading c3: B_l
is [N][S], chunk j at bytes [jS, (j+1)S)).

Paged delivery (reading c4/c5): inside B_l, chunk j's slice is
[2][G][n_kv][d] (reading c2), so the byte at (j, kv, t, h, e) of B_l is
    j*S + kv*G*row + t*row + h*(d*p) + e,          row = n_kv*d*p.
It belongs to request token u = first_token + j*G + t and is written to
    kv_base[kv][l] + block_table[u // Bs]*block_stride + (u % Bs)*token_stride
    + h*head_stride + e.
Bytes of the destination that no token maps to are left untouched (c5).
``dst`` is a numpy uint8 array standing for the destination memory; target
bases and strides are byte offsets into it.
"""
import numpy as np

from .geometry import chunk_layer_bytes, row_bytes, head_bytes
from .descriptor import FlatTarget, PagedTarget


def gather_layer(store, desc, layer: int) -> bytes:
    """Alg. A1 lines 2-5: B_l = concat_j RangeGet(H_j, l*S, S)."""
    S = desc.per_layer_chunk_bytes
    if not 0 <= layer < desc.num_layers:
        raise IndexError("layer out of range")
    parts = []
    for key in desc.chunk_keys:
        o = layer * S
        parts.append(store.range_get(key, o, S))
    return b"".join(parts)


def write_flat(B: bytes, layer: int, desc, dst: np.ndarray):
    """Alg. A1 line 6 with the paper's client_buffer[l] at base + l*N*S."""
    t = desc.target
    n = len(B)
    off = t.base + layer * n
    dst[off:off + n] = np.frombuffer(B, dtype=np.uint8)


def scatter_paged(B: bytes, layer: int, desc, dst: np.ndarray):
    """Write payload B_l into the paged cache, one (token, head) run of d*p bytes at a time."""
    lay = desc.layout
    t = desc.target
    S = chunk_layer_bytes(lay)
    G = lay.chunk_tokens
    row = row_bytes(lay)
    hd = head_bytes(lay)
    N = len(desc.chunk_keys)
    src = np.frombuffer(B, dtype=np.uint8)
    for j in range(N):
        for kv in (0, 1):
            base = (t.k_base if kv == 0 else t.v_base)[layer]
            for tok in range(G):
                u = t.first_token + j * G + tok
                blk = t.block_table[u // t.block_size]
                slot = u % t.block_size
                for h in range(lay.kv_heads):
                    s_off = j * S + kv * G * row + tok * row + h * hd
                    d_off = base + blk * t.block_stride + slot * t.token_stride + h * t.head_stride
                    dst[d_off:d_off + hd] = src[s_off:s_off + hd]


def fetch_layerwise(store, desc, dst: np.ndarray):
    """Alg. A1 end to end: for each layer gather, deliver, then notify.

    Returns the list of NotifyLayerReady events, i.e. the layer indices in the
    order they were announced (0, 1, ..., L-1).
    """
    events = []
    for layer in range(desc.num_layers):
        B = gather_layer(store, desc, layer)
        if isinstance(desc.target, FlatTarget):
            write_flat(B, layer, desc, dst)
        elif isinstance(desc.target, PagedTarget):
            scatter_paged(B, layer, desc, dst)
        else:
            raise TypeError("unknown target")
        events.append(layer)
    return events


def scatter_paged_advanced_index(B: bytes, layer: int, desc, dst: np.ndarray):
    """Second, independent formulation for the contiguous NHD cache (vLLM FlashAttention).

    When token_stride = row, head_stride = d*p and block_stride = Bs*row, the
    layer-l K (or V) cache from kv_base is a [num_blocks*Bs][row] array and the
    scatter is the library routine ``cache[slot_mapping] = rows`` with
    slot_mapping[u] = block_table[u // Bs]*Bs + u % Bs.
    """
    lay = desc.layout
    t = desc.target
    G = lay.chunk_tokens
    row = row_bytes(lay)
    N = len(desc.chunk_keys)
    if not (t.token_stride == row and t.head_stride == head_bytes(lay)
            and t.block_stride == t.block_size * row):
        raise ValueError("advanced-index form needs the contiguous NHD layout")
    payload = np.frombuffer(B, dtype=np.uint8).reshape(N, 2, G, row)
    u = t.first_token + np.arange(N * G)
    bt = np.asarray(t.block_table, dtype=np.int64)
    slots = bt[u // t.block_size] * t.block_size + u % t.block_size
    for kv in (0, 1):
        base = (t.k_base if kv == 0 else t.v_base)[layer]
        n_rows = (int(slots.max()) + 1)
        cache = dst[base:base + n_rows * row].reshape(n_rows, row)
        cache[slots] = payload[:, kv].reshape(N * G, row)


def offload_paged(store, keys, layout, target, mem: np.ndarray) -> int:
    """The offload path (Sec. 3: "newly produced KV blocks are offloaded back to object
    storage for future reuse"): chunk j of the request -- tokens first_token + j*G .. +G-1 --
    is read out of the paged cache ``mem`` in KV_L2TD order (layer, then K/V, then token, then
    head; reading c2) and put under key j.  Keys already stored are left as they are (identity is
    the chain key, reading c18).  Returns the number of new keys."""
    G = layout.chunk_tokens
    hd = head_bytes(layout)
    parts_new = 0
    for j, key in enumerate(keys):
        if bytes(key) in store:
            continue
        parts = []
        for layer in range(layout.num_layers):
            for kv in (0, 1):
                base = (target.k_base if kv == 0 else target.v_base)[layer]
                for tok in range(G):
                    u = target.first_token + j * G + tok
                    blk = target.block_table[u // target.block_size]
                    slot = u % target.block_size
                    for h in range(layout.kv_heads):
                        a = base + blk * target.block_stride + slot * target.token_stride + h * target.head_stride
                        parts.append(mem[a:a + hd].tobytes())
        store.put([key], [b"".join(parts)])
        parts_new += 1
    return parts_new
