"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method: no hashing, no layer ranges,
no scatter addresses, no scheduling.  It only produces raw inputs --
token streams with a chosen sharing structure, chunk payload bytes, free
block lists, and the named layouts of BASELINE.json -- so that the oracle and
the CUDA library can each compute on identical inputs.

Recipe (also in DESIGN.md "Input recipe"):
* tokens: uint32 uniform in [0, 128256) (the Llama-3 vocabulary), PCG64.
* prefix families: streams of one family share their first ``shared_blocks``
  G-token blocks exactly; the rest of each stream is drawn independently.
* chunk payload bytes: the chunk with payload id (family, block) is the
  PCG64([seed, family, block]) byte stream, so chunks shared between streams
  carry identical bytes (content-consistent with the prefix-chain key) and any
  single chunk can be regenerated on its own for sampled checks.
* paged destinations: block tables are a seeded random permutation of a free
  block pool (fragmented, no duplicates).
"""
from dataclasses import dataclass

import numpy as np

LLAMA3_VOCAB = 128256


@dataclass(frozen=True)
class NamedLayout:
    name: str
    num_layers: int
    kv_heads: int
    head_dim: int
    elem_bytes: int
    chunk_tokens: int

    def as_tuple(self):
        return (self.num_layers, self.kv_heads, self.head_dim, self.elem_bytes, self.chunk_tokens)


# BASELINE.json configs[0], [1]-[2]/[4], [3]
TINY = NamedLayout("tiny", 2, 2, 16, 2, 16)
LLAMA3_8B = NamedLayout("llama3-8b", 32, 8, 128, 2, 16)
LLAMA3_70B = NamedLayout("llama3-70b", 80, 8, 128, 2, 16)


def with_chunk_tokens(lay: NamedLayout, G: int) -> NamedLayout:
    return NamedLayout(lay.name + f"-G{G}", lay.num_layers, lay.kv_heads, lay.head_dim,
                       lay.elem_bytes, G)


def tokens(seed: int, n: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64([seed, 0x70C]))
    return rng.integers(0, LLAMA3_VOCAB, size=n, dtype=np.uint32)


def family_streams(seed: int, G: int, shared_blocks: int, own_blocks, tail_tokens=None):
    """Token streams sharing their first ``shared_blocks`` blocks.

    own_blocks[i] more blocks follow for stream i, then tail_tokens[i] extra
    tokens (a partial block).  Returns (streams, payload_ids) where
    payload_ids[i][b] = (owner, b) names the payload of block b of stream i:
    owner 0 for shared blocks, i+1 for the stream's own blocks.
    """
    tail_tokens = tail_tokens or [0] * len(own_blocks)
    shared = tokens(seed, shared_blocks * G)
    streams, ids = [], []
    for i, (own, tail) in enumerate(zip(own_blocks, tail_tokens)):
        mine = tokens(seed * 1000003 + i + 1, own * G + tail)
        streams.append(np.concatenate([shared, mine]).astype(np.uint32))
        ids.append([(0, b) for b in range(shared_blocks)] +
                   [(i + 1, b) for b in range(shared_blocks, shared_blocks + own)])
    return streams, ids


def chunk_payload(seed: int, payload_id, nbytes: int) -> np.ndarray:
    """nbytes of PCG64 output for one chunk (uint8)."""
    owner, block = payload_id
    bg = np.random.PCG64([seed, 0xC4C4, int(owner), int(block)])
    words = bg.random_raw(-(-nbytes // 8)).astype(np.uint64, copy=False)
    return words.view(np.uint8)[:nbytes]


def chunk_payload_range(seed: int, payload_id, offset: int, nbytes: int) -> np.ndarray:
    """Bytes [offset, offset + nbytes) of chunk_payload(seed, payload_id, ...), regenerated on their
    own (offset a multiple of 8): the PCG64 stream advanced by offset/8 words.  Lets at-size checks
    draw one layer slice of one chunk without the whole corpus in memory."""
    if offset % 8:
        raise ValueError("offset must be a multiple of 8")
    owner, block = payload_id
    bg = np.random.PCG64([seed, 0xC4C4, int(owner), int(block)])
    bg.advance(offset // 8)
    words = bg.random_raw(-(-nbytes // 8)).astype(np.uint64, copy=False)
    return words.view(np.uint8)[:nbytes]


def payloads(seed: int, payload_ids, nbytes: int) -> np.ndarray:
    """Stack of chunk payloads, shape [len(payload_ids), nbytes]."""
    out = np.empty((len(payload_ids), nbytes), dtype=np.uint8)
    for i, pid in enumerate(payload_ids):
        out[i] = chunk_payload(seed, pid, nbytes)
    return out


def block_table(seed: int, n_needed: int, pool_blocks: int) -> np.ndarray:
    """n_needed distinct block ids drawn from [0, pool_blocks) in random order."""
    if n_needed > pool_blocks:
        raise ValueError("pool too small")
    rng = np.random.Generator(np.random.PCG64([seed, 0xB7]))
    return rng.permutation(pool_blocks)[:n_needed].astype(np.int32)


def sentinel(nbytes: int, value: int = 0xA5) -> np.ndarray:
    return np.full(nbytes, value, dtype=np.uint8)


def serving_requests(seed: int, n_requests: int, n_fam_short: int, n_fam_long: int, zipf_s: float = 1.1,
                     hits=(0.5, 0.875), home_of=None, rank: int = 0, p_aff: float = 0.875):
    """Config 5's request mix: each request picks a length class (short / long,
    50/50), a prefix family of that class by a Zipf(s) rank law, and a hit rate from ``hits``.
    With ``home_of(long, family) -> rank`` (multi-GPU), a request served by ``rank`` picks a family
    homed on it with probability ``p_aff`` and a family homed elsewhere otherwise (Zipf law
    restricted to that set; unrestricted if the set is empty).
    Returns a list of (long: bool, family index within the class, hit rate)."""
    rng = np.random.Generator(np.random.PCG64([seed, 0x5E7]))
    out = []
    for _ in range(n_requests):
        long = bool(rng.integers(0, 2))
        n = n_fam_long if long else n_fam_short
        w = 1.0 / np.arange(1, n + 1) ** zipf_s
        local = rng.random() < p_aff
        if home_of is not None:
            keep = np.array([(home_of(long, f) == rank) == local for f in range(n)])
            if keep.any():
                w = np.where(keep, w, 0.0)
        fam = int(rng.choice(n, p=w / w.sum()))
        out.append((long, fam, float(hits[int(rng.integers(0, len(hits)))])))
    return out
