"""The ObjectCache request descriptor (oracle; test infrastructure only).

P:264-284 (Sec. 3, Table 1): chunk_keys [H_0..H_{N-1}], num_layers L,
chunk_tokens G, per_layer_chunk_bytes S, delivery (layer-major order),
rdma_target (client buffer address, key, length).
P:321-333 (Sec. 3.2): the descriptor is "intentionally arithmetic rather than
manifest-heavy": every layer range follows from (L, S).

On B200 the rdma_target becomes a GPU destination (reading c4): either the
paper's flat client buffer of L layer-major payloads (``FlatTarget``), or a
serving engine's paged KV cache (``PagedTarget``).  Offsets are byte offsets
into one destination byte array (the oracle has no device addresses).
"""
from dataclasses import dataclass, field
from typing import List

from .geometry import Layout, chunk_layer_bytes, row_bytes, head_bytes


class NotFoundError(Exception):
    def __init__(self, index):
        super().__init__(f"chunk key {index} not in store")
        self.index = index


class RangeError(Exception):
    pass


@dataclass
class FlatTarget:
    """The paper's client_buffer[l] (Alg. A1 line 6): L payloads of N*S bytes, layer l at base + l*N*S."""

    base: int
    capacity: int


@dataclass
class PagedTarget:
    """A paged KV cache (reading c4).

    Token u of the request, matrix kv (0 = K, 1 = V), head h, at layer l lives at
    ``kv_base[kv][l] + block_table[u // Bs] * block_stride + (u % Bs) * token_stride
    + h * head_stride`` and is d*p bytes long.  vLLM/FlashAttention NHD is
    token_stride = n_kv*d*p, head_stride = d*p; HND is token_stride = d*p,
    head_stride = Bs*d*p.
    """

    k_base: List[int]
    v_base: List[int]
    block_stride: int
    token_stride: int
    head_stride: int
    block_size: int
    block_table: List[int]
    first_token: int = 0


@dataclass
class Descriptor:
    chunk_keys: List[bytes]
    num_layers: int
    chunk_tokens: int
    per_layer_chunk_bytes: int
    delivery: str
    target: object
    layout: Layout = field(default=None)


def build_descriptor(store, keys, layout: Layout, target, delivery="layer_major") -> Descriptor:
    """Validate and assemble a Table 1 descriptor.

    Errors: N = 0 -> ValueError; first key absent from ``store`` -> NotFoundError(index)
    (in prefix order); target too small -> RangeError.
    """
    keys = [bytes(k) for k in keys]
    if len(keys) == 0:
        raise ValueError("descriptor needs N >= 1 chunk keys")
    if delivery not in ("layer_major", "chunk_major"):
        raise ValueError("delivery must be layer_major or chunk_major")
    for i, k in enumerate(keys):
        if k not in store:
            raise NotFoundError(i)
    N = len(keys)
    S = chunk_layer_bytes(layout)
    G = layout.chunk_tokens
    if isinstance(target, FlatTarget):
        if target.capacity < N * layout.num_layers * S:
            raise RangeError("flat target smaller than W = N*L*S")
    elif isinstance(target, PagedTarget):
        if len(target.k_base) != layout.num_layers or len(target.v_base) != layout.num_layers:
            raise ValueError("need one K and one V base per layer")
        last_token = target.first_token + N * G - 1
        if last_token // target.block_size >= len(target.block_table):
            raise RangeError("block table does not cover the prefix")
        used = target.block_table[target.first_token // target.block_size:
                                  last_token // target.block_size + 1]
        if len(set(used)) != len(used):
            raise ValueError("duplicate block ids: result would depend on write order (c4)")
        if any(b < 0 for b in used):
            raise ValueError("negative block id")
        if row_bytes(layout) % head_bytes(layout) != 0:
            raise ValueError("bad layout")
    else:
        raise TypeError("unknown target")
    return Descriptor(keys, layout.num_layers, G, S, delivery, target, layout)
