"""Content-addressed, immutable chunk store (oracle; test infrastructure only).

P:36-40 (Sec. 1) and P:124-128 (Sec. 2.1): prefix KV blocks are "immutable
after prefill, naturally addressable by content-derived prefix hashes";
using H_i as the key gives "immutable writes, content-addressed
deduplication".  P:224 (Sec. 3): newly produced blocks are offloaded back
for future reuse.

A put of an existing key with identical bytes is a no-op (dedup); with
different bytes it is an immutability violation.  Reading c18: identity is
the chain key, so equal bytes under different keys are stored twice.
"""
from .geometry import Layout, chunk_bytes


class ImmutableError(Exception):
    pass


class ChunkStore:
    def __init__(self, layout: Layout):
        self.layout = layout
        self.objects = {}

    def __contains__(self, key):
        return bytes(key) in self.objects

    def __len__(self):
        return len(self.objects)

    def put(self, keys, payloads) -> int:
        """Store each (key, payload); returns how many keys were new."""
        want = chunk_bytes(self.layout)
        n_new = 0
        for k, p in zip(keys, payloads):
            k = bytes(k)
            p = bytes(p)
            if len(k) != 32:
                raise ValueError("keys are 32 bytes")
            if len(p) != want:
                raise ValueError(f"payload must be L*S = {want} bytes, got {len(p)}")
            old = self.objects.get(k)
            if old is None:
                self.objects[k] = p
                n_new += 1
            elif old != p:
                raise ImmutableError(k.hex())
        return n_new

    def get(self, key) -> bytes:
        return self.objects[bytes(key)]

    def range_get(self, key, offset: int, length: int) -> bytes:
        """RangeGet(H_j, o, S) of Alg. A1 line 5."""
        obj = self.objects[bytes(key)]
        if offset < 0 or offset + length > len(obj):
            raise IndexError("range outside object")
        return obj[offset:offset + length]
