"""Rolling chunk hash (oracle; test infrastructure only).

P:124-128 (Sec. 2.1): "Each chunk can be identified by a rolling hash,
H_i = Hash(H_{i-1} || tokens_i), that gives it a deterministic object key."

Reading c1 (the paper names only "Hash"): SHA-256 over the 32-byte previous
digest followed by the chunk's G token ids as little-endian uint32; the root
H_{-1} is 32 zero bytes.  Only complete G-token blocks get keys; a trailing
partial block is ignored.  hashlib is the library primitive for the hash step.
"""
import hashlib
import struct

ROOT = bytes(32)


def chunk_key(prev: bytes, block_tokens) -> bytes:
    """One step of the chain: SHA-256(prev || LE-u32 tokens)."""
    if len(prev) != 32:
        raise ValueError("previous key must be 32 bytes")
    h = hashlib.sha256()
    h.update(prev)
    for t in block_tokens:
        t = int(t)
        if not 0 <= t < 2**32:
            raise ValueError("token ids are unsigned 32-bit")
        h.update(struct.pack("<I", t))
    return h.digest()


def chunk_keys(tokens, G: int, parent: bytes = ROOT):
    """Keys H_0..H_{n-1} of the n = floor(len/G) complete blocks, chained from ``parent``."""
    if G < 1:
        raise ValueError("G must be >= 1")
    keys = []
    prev = parent
    n_blocks = len(tokens) // G
    for i in range(n_blocks):
        prev = chunk_key(prev, tokens[i * G:(i + 1) * G])
        keys.append(prev)
    return keys
