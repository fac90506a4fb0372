"""Eq. 1 KV geometry and layer-range arithmetic (oracle; test infrastructure only).

P:110-120 (Sec. 2.1, Eq. 1):  KV_token = 2 L n_kv d p,   S_layer,chunk = 2 G n_kv d p.
P:327-331 (Sec. 3.2): "the byte range for layer l in a chunk is [lS, (l+1)S)".
P:347-354 (Sec. 3.3): KV_L2TD -- layer-major, then the 2 matrices (K, V),
    then token position, then hidden dimension.  Reading c2: the hidden
    dimension is flattened as [n_kv][d], so one token of one matrix is a row of
    n_kv*d*p bytes and a layer slice is [2][G][n_kv][d].
P:378-385 (Sec. 3.4, Eq. 2): W = N L S; chunkwise if W < Theta else layerwise.
"""
from dataclasses import dataclass


@dataclass(frozen=True)
class Layout:
    """The Eq. 1 symbols: L, n_kv, d, p (bytes per element) and G (tokens per chunk)."""

    num_layers: int
    kv_heads: int
    head_dim: int
    elem_bytes: int
    chunk_tokens: int

    def __post_init__(self):
        for name in ("num_layers", "kv_heads", "head_dim", "elem_bytes", "chunk_tokens"):
            if int(getattr(self, name)) < 1:
                raise ValueError(f"{name} must be >= 1")


def kv_token_bytes(lay: Layout) -> int:
    """Eq. 1 left: KV_token = 2 * L * n_kv * d * p (all layers, K and V)."""
    return 2 * lay.num_layers * lay.kv_heads * lay.head_dim * lay.elem_bytes


def per_token_layer_bytes(lay: Layout) -> int:
    """Bytes of one token at one layer, K and V: 2 * n_kv * d * p (P:2693-2694 prints 4096 for Llama 3.1 8B)."""
    return 2 * lay.kv_heads * lay.head_dim * lay.elem_bytes


def row_bytes(lay: Layout) -> int:
    """One token of one matrix (K or V) at one layer: n_kv * d * p (reading c2)."""
    return lay.kv_heads * lay.head_dim * lay.elem_bytes


def head_bytes(lay: Layout) -> int:
    """One head of one token of one matrix: d * p."""
    return lay.head_dim * lay.elem_bytes


def chunk_layer_bytes(lay: Layout) -> int:
    """Eq. 1 right: S = 2 * G * n_kv * d * p."""
    return 2 * lay.chunk_tokens * lay.kv_heads * lay.head_dim * lay.elem_bytes


def chunk_bytes(lay: Layout) -> int:
    """A KV_L2TD chunk object holds all L layers back to back: L * S bytes."""
    return lay.num_layers * chunk_layer_bytes(lay)


def layer_range(lay: Layout, layer: int):
    """layer l of a chunk occupies [l S, (l+1) S).  Returns (offset, length)."""
    if not 0 <= layer < lay.num_layers:
        raise IndexError(f"layer {layer} out of range [0, {lay.num_layers})")
    s = chunk_layer_bytes(lay)
    return layer * s, s


def matched_payload_bytes(lay: Layout, n_chunks: int) -> int:
    """Sec. 3.4: W = N * L * S."""
    if n_chunks < 0:
        raise ValueError("N must be >= 0")
    return n_chunks * lay.num_layers * chunk_layer_bytes(lay)


def layer_payload_bytes(lay: Layout, n_chunks: int) -> int:
    """Size of one layer-major payload B_l of Alg. A1: N * S bytes."""
    return n_chunks * chunk_layer_bytes(lay)


def matched_bytes_per_layer(lay: Layout, context_tokens: int, hit_rate: float) -> float:
    """Sec. 5.3: D^(l) = 2 n_kv d p (P r)."""
    return 2 * lay.kv_heads * lay.head_dim * lay.elem_bytes * (context_tokens * hit_rate)


def delivery_mode(payload_W: int, theta: int) -> str:
    """Eq. 2: chunkwise if W < Theta, layerwise (+ aggregation) if W >= Theta."""
    return "chunkwise" if payload_W < theta else "layerwise"
