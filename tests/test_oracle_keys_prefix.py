"""Pins for oracle.keys / oracle.prefix / oracle.store: hash standard, chain invariants, brute force."""
import hashlib
import random

import numpy as np
import pytest

import synth
from oracle import keys, prefix
from oracle.geometry import Layout, chunk_bytes
from oracle.store import ChunkStore, ImmutableError
from conftest import read_golden


def _msg(m):
    return b"a" * 1000000 if m == "@million_a" else m.encode()


@pytest.mark.parametrize("row", read_golden("sha256_fips180.csv"))
def test_hash_primitive_is_fips_sha256(row):
    assert hashlib.sha256(_msg(row["message"])).hexdigest() == row["digest"]


def test_chain_definition_by_hand():
    # H_0 = SHA-256(32 zero bytes || LE u32 tokens), H_1 = SHA-256(H_0 || ...), built byte by byte here.
    toks = list(range(32))
    b0 = bytes(32) + b"".join(t.to_bytes(4, "little") for t in toks[:16])
    h0 = hashlib.sha256(b0).digest()
    h1 = hashlib.sha256(h0 + b"".join(t.to_bytes(4, "little") for t in toks[16:])).digest()
    assert keys.chunk_keys(toks, 16) == [h0, h1]
    # convention vectors recorded in SURVEY.md 8(c) for tokens 0..31 at G=16
    assert h0.hex() == "aa330374288acbdcb5008f2959fd6df7d265c735fbb9b4b4c42ec2036accd6d3"
    assert h1.hex() == "8f3d3a653ef4f75ccd8845b6a76dd246da5b5e735809babef53877d21125357c"


def test_chain_invariants():
    t = synth.tokens(1, 16 * 6 + 5)
    k = keys.chunk_keys(t, 16)
    assert len(k) == 6                                # trailing partial block ignored
    assert k == keys.chunk_keys(t, 16)                # deterministic
    assert keys.chunk_keys(t[:16 * 3], 16) == k[:3]   # prefix stable
    t2 = t.copy()
    t2[16 * 2 + 7] ^= 1                               # change one token of block 2
    k2 = keys.chunk_keys(t2, 16)
    assert k2[:2] == k[:2] and all(a != b for a, b in zip(k2[2:], k[2:]))
    # token order matters
    t3 = t.copy()
    t3[[0, 1]] = t3[[1, 0]]
    if t3[0] != t3[1]:
        assert keys.chunk_keys(t3, 16)[0] != k[0]
    # a chain continued from a parent equals the suffix of the full chain
    assert keys.chunk_keys(t[16 * 2:], 16, parent=k[1]) == k[2:]
    with pytest.raises(ValueError):
        keys.chunk_key(bytes(31), [1])
    with pytest.raises(ValueError):
        keys.chunk_key(bytes(32), [2**32])


def test_spec_4096_tokens_give_256_keys():
    assert len(keys.chunk_keys(synth.tokens(0, 4096), 16)) == 256


@pytest.mark.parametrize("seed", range(25))
def test_three_match_formulations_agree(seed):
    rng = random.Random(seed)
    G = rng.choice([1, 2, 4, 16])
    vocab = rng.choice([2, 3, 50])
    streams = []
    for _ in range(rng.randint(1, 5)):
        if streams and rng.random() < 0.6:            # share a prefix with an earlier stream
            base = rng.choice(streams)
            cut = rng.randint(0, len(base))
            s = list(base[:cut]) + [rng.randrange(vocab) for _ in range(rng.randint(0, 4 * G))]
        else:
            s = [rng.randrange(vocab) for _ in range(rng.randint(0, 6 * G))]
        streams.append(s)
    tree = prefix.RadixTree(G)
    store = set()
    for s in streams:
        for k in tree.insert(s):
            store.add(k)
    queries = streams + [list(s[:len(s) // 2]) + [rng.randrange(vocab) for _ in range(2 * G)] for s in streams]
    for q in queries:
        n_bf = prefix.brute_force_match(streams, q, G)
        via_tree = tree.longest_match(q)
        via_probe = prefix.probe_match(lambda k: k in store, q, G)
        assert len(via_tree) == n_bf == len(via_probe)
        assert via_tree == via_probe == keys.chunk_keys(q, G)[:n_bf]


def test_insert_then_match_self_and_idempotence():
    G = 16
    tree = prefix.RadixTree(G)
    t = synth.tokens(5, 16 * 9 + 3)
    tree.insert(t)
    n = tree.n_nodes
    assert len(tree.longest_match(t)) == len(t) // G   # longest_match(insert(x), x) = floor(len/G) blocks
    tree.insert(t)
    assert tree.n_nodes == n


def test_tiny_config_matches():
    # A = 8 shared + 2 own blocks + 5-token tail; B = 8 shared + 3 own.
    G = 16
    (a, b), _ = synth.family_streams(0, G, 8, [2, 3], [5, 0])
    tree = prefix.RadixTree(G)
    tree.insert(a)
    assert len(tree.longest_match(b)) == 8
    tree.insert(b)
    assert len(tree.longest_match(a)) == 10 and len(tree.longest_match(b)) == 11
    q = a.copy()
    q[8 * G + 3] ^= 1                                 # diverge mid block 9
    assert len(tree.longest_match(q)) == 8


def test_store_dedup_and_immutability():
    lay = Layout(2, 2, 16, 2, 16)
    st = ChunkStore(lay)
    n = chunk_bytes(lay)
    (a, b), (ia, ib) = synth.family_streams(0, 16, 8, [2, 3])
    ka, kb = keys.chunk_keys(a, 16), keys.chunk_keys(b, 16)
    pa, pb = synth.payloads(0, ia, n), synth.payloads(0, ib, n)
    assert st.put(ka, pa) == 10
    assert st.put(kb, pb) == 3                        # 8 shared chunks deduplicated
    assert st.put(ka, pa) == 0
    bad = pa[0].copy()
    bad[0] ^= 0xFF
    with pytest.raises(ImmutableError):
        st.put(ka[:1], [bad])
    with pytest.raises(ValueError):
        st.put(ka[:1], [pa[0][:-1]])
    assert st.range_get(ka[3], 5, 7) == bytes(pa[3][5:12])
    with pytest.raises(IndexError):
        st.range_get(ka[3], n - 1, 2)
