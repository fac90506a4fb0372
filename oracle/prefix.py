"""Longest-prefix match (oracle; test infrastructure only).

P:121-123 (Sec. 2.1): "a radix tree or similar prefix index to find the
longest cached match for a new request".  P:202-205 (Sec. 2.2): "prefix
lookup returns an ordered list of matched KV chunks".

Three independent formulations, used to check one another:

* ``brute_force_match``  compares the query's complete G-blocks with every
  inserted token stream and takes the longest common block prefix.
* ``RadixTree``          edges labelled by raw G-token blocks.
* ``probe_match``        walks the query's key chain and stops at the first
  key absent from a store (reading c17: equal to the two above when the store
  holds whole chains from the root, as every put in scope does).
"""
from . import keys as _keys


def _blocks(tokens, G):
    n = len(tokens) // G
    return [tuple(int(t) for t in tokens[i * G:(i + 1) * G]) for i in range(n)]


def brute_force_match(inserted_streams, query, G: int) -> int:
    """Number of leading complete blocks of ``query`` shared with some inserted stream."""
    qb = _blocks(query, G)
    best = 0
    for s in inserted_streams:
        sb = _blocks(s, G)
        k = 0
        while k < len(qb) and k < len(sb) and qb[k] == sb[k]:
            k += 1
        best = max(best, k)
    return best


class RadixTree:
    """Radix tree over G-token blocks; each node stores the key of the chunk ending there."""

    def __init__(self, G: int):
        self.G = G
        self.root = {}          # block -> (key, children)
        self.n_nodes = 0

    def insert(self, tokens):
        """Insert all complete blocks; returns the key chain.  Idempotent."""
        chain = _keys.chunk_keys(tokens, self.G)
        node = self.root
        for blk, key in zip(_blocks(tokens, self.G), chain):
            if blk not in node:
                node[blk] = (key, {})
                self.n_nodes += 1
            node = node[blk][1]
        return chain

    def longest_match(self, tokens):
        """Ordered keys of the longest inserted block prefix of ``tokens``."""
        out = []
        node = self.root
        for blk in _blocks(tokens, self.G):
            if blk not in node:
                break
            key, node = node[blk]
            out.append(key)
        return out


def probe_match(store_contains, tokens, G: int, parent: bytes = _keys.ROOT):
    """Walk H_0, H_1, ... of ``tokens`` and stop at the first key the store lacks."""
    out = []
    prev = parent
    for i in range(len(tokens) // G):
        prev = _keys.chunk_key(prev, tokens[i * G:(i + 1) * G])
        if not store_contains(prev):
            break
        out.append(prev)
    return out
