"""Chunk keys on the GPU (oc_chunk_keys_batch, the offload path's optional device hashing) equal
the oracle's hashlib chain and the host library's keys, for ragged batches, odd G and parents."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2605_22850_b200 as oc  # noqa: E402
import synth  # noqa: E402
from oracle import keys as okeys  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G", [16, 3, 64, 256])
def test_batch_chain_keys_equal_oracle(G):
    rng = np.random.default_rng(G)
    lens = [int(x) for x in rng.integers(0, 40 * G, size=37)] + [0, G - 1, G, 5 * G + 1]
    streams = [synth.tokens(1000 + i, n) for i, n in enumerate(lens)]
    parents = rng.integers(0, 256, size=(len(streams), 32), dtype=np.uint8)
    for use_parents in (False, True):
        got = oc.chunk_keys_batch(streams, G, parents=parents if use_parents else None)
        for i, t in enumerate(streams):
            par = bytes(parents[i]) if use_parents else okeys.ROOT
            want = np.frombuffer(b"".join(okeys.chunk_keys(t, G, par)), dtype=np.uint8).reshape(-1, 32)
            assert got[i].shape == (len(t) // G, 32)
            assert np.array_equal(got[i], want), (G, i, use_parents)
            host = oc.chunk_keys(t, G, parent=par if use_parents else None)
            assert np.array_equal(got[i], host[:len(t) // G])


def test_batch_chain_keys_convention_golden():
    """SURVEY 8(c) golden vectors of reading c1: tokens 0..31 at G = 16."""
    got = oc.chunk_keys_batch([np.arange(32, dtype=np.uint32)], 16)[0]
    assert got[0].tobytes().hex() == "aa330374288acbdcb5008f2959fd6df7d265c735fbb9b4b4c42ec2036accd6d3"
    assert got[1].tobytes().hex() == "8f3d3a653ef4f75ccd8845b6a76dd246da5b5e735809babef53877d21125357c"


def test_batch_chain_keys_errors():
    with pytest.raises(oc.ObjcacheError) as e:
        oc.chunk_keys_batch([np.arange(8, dtype=np.uint32)], 0)
    assert e.value.code == oc.OC_EINVAL
