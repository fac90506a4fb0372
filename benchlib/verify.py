"""In-run verification of the large bench legs against the oracle ("for configs 4/5
the oracle verifies sampled requests fully plus per-layer digests for all, and its time per
verified byte is reported").  Test infrastructure on the bench's side, like the cpu_baseline leg:
it runs oracle/ code on the host, never on the product path, and only after the timed regions.

Payloads: the legs fill their stores with synth chunk payloads (PCG64 per (seed, owner, block)),
generated on host threads; the oracle regenerates any chunk on its own (scenario-style SynthStore
RangeGet), so no expected value ever comes from the GPU.

Per-layer digest of one request (a verification checksum, not a step of the method): with B_l the
request's layer-l payload in prefix order (Alg. A1 lines 3-5: chunk j's slice at [jS, (j+1)S)),
read as little-endian u64 words x[j][k], and T[k] a fixed table of S/8 pseudo-random u64 words,

    D_l = sum_j (2j + 1) * sum_k T[k] * x[j][k]      (mod 2^64)

Both sides evaluate it independently: the GPU side on the bytes the fetch delivered, read back
from the paged cache through the request's block table (torch gathers, int64 wrap-around
arithmetic); the oracle side on the chunk slices its RangeGet returns (numpy u64 wrap-around).
A corrupted word, a reordered row or a swapped chunk changes D_l except with probability ~2^-64
per term.  The chunk at position j of a family prefix is the same for every request of that
family, so the oracle computes each chunk's per-layer inner sums once and forms every request's
D_l from prefix sums.
"""
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

import synth

TABLE_SEED = 0xD16E57


def host_threads():
    try:
        return max(1, min(16, len(os.sched_getaffinity(0))))
    except Exception:
        return max(1, min(16, os.cpu_count() or 1))


def digest_table(S):
    """T: S/8 pseudo-random u64 words (seeded; an input of both sides)."""
    return np.random.PCG64([TABLE_SEED, S]).random_raw(S // 8).astype(np.uint64)


# ---- library side: fill stores with synth payloads ------------------------------------------------
def fill_store(stores, keys, seed, payload_ids, chunk_bytes, batch=128, threads=None):
    """Put synth payloads of `payload_ids` under `keys` into every store of `stores`, generating
    batches on host threads while the previous batch is put.  Returns seconds spent."""
    t0 = time.perf_counter()
    threads = threads or host_threads()
    n = len(payload_ids)
    starts = list(range(0, n, batch))

    def gen(b0):
        return synth.payloads(seed, payload_ids[b0:b0 + batch], chunk_bytes)

    with ThreadPoolExecutor(threads) as ex:
        futs = [ex.submit(gen, b0) for b0 in starts[:threads]]
        nxt = len(futs)
        for i, b0 in enumerate(starts):
            pl = futs[i].result()
            futs[i] = None
            if nxt < len(starts):
                futs.append(ex.submit(gen, starts[nxt]))
                nxt += 1
            for st in stores:
                st.put_chunks(keys[b0:b0 + pl.shape[0]], pl)
    return time.perf_counter() - t0


def fill_store_scattered(store, requests, chunk_bytes, order_seed, batch=128, threads=None):
    """Put the chunks of several requests -- `requests` = [(keys, seed, payload_ids), ...] -- in one
    seeded random interleaving, so each request's chunks land at random slots of the append-only
    slab ("store slots at random (hash-addressed) slab positions").  Payloads
    are the same synth bytes fill_store puts.  Returns seconds spent."""
    t0 = time.perf_counter()
    threads = threads or host_threads()
    pairs = [(r, i) for r, (_, _, ids) in enumerate(requests) for i in range(len(ids))]
    order = np.random.Generator(np.random.PCG64([order_seed, 0x51])).permutation(len(pairs))
    starts = list(range(0, len(order), batch))

    def gen(b0):
        sel = [pairs[k] for k in order[b0:b0 + batch]]
        keys = np.stack([np.asarray(requests[r][0][i]) for r, i in sel])
        pl = np.empty((len(sel), chunk_bytes), dtype=np.uint8)
        for row, (r, i) in enumerate(sel):
            pl[row] = synth.chunk_payload(requests[r][1], requests[r][2][i], chunk_bytes)
        return keys, pl

    with ThreadPoolExecutor(threads) as ex:   # at most `threads` batches generated ahead
        futs = [ex.submit(gen, b0) for b0 in starts[:threads]]
        for i in range(len(starts)):
            keys, pl = futs[i].result()
            futs[i] = None
            if i + threads < len(starts):
                futs.append(ex.submit(gen, starts[i + threads]))
            store.put_chunks(keys, pl)
    return time.perf_counter() - t0


# ---- GPU side: read back what a fetch delivered -----------------------------------------------------
def slot_index(torch, dev, block_table, n_tokens, Bs, first_token=0):
    """Row index (block * Bs + slot) of each of the prefix's n_tokens in a [pool*Bs, row] view."""
    u = np.arange(first_token, first_token + n_tokens, dtype=np.int64)
    bt = np.asarray(block_table, dtype=np.int64)
    return torch.from_numpy(bt[u // Bs] * Bs + u % Bs).to(dev)


def delivered_layer(torch, cache, layer, idx, N, G):
    """B_l as delivered: [N][S] bytes (K rows then V rows of each chunk) from an NHD paged cache
    tensor [L][2][pool][Bs][row] (uint8), gathered through the request's row index."""
    row = cache.shape[-1]
    k = cache[layer, 0].reshape(-1, row).index_select(0, idx).view(N, G, row)
    v = cache[layer, 1].reshape(-1, row).index_select(0, idx).view(N, G, row)
    return torch.cat([k, v], dim=1).reshape(N, 2 * G * row)


def gpu_digests(torch, cache, idx, N, G, T_dev):
    """D_l for every layer of one request, from the delivered bytes (int64 wrap-around arithmetic
    is arithmetic mod 2^64, bit for bit the u64 of the oracle side)."""
    L = cache.shape[0]
    w = (2 * torch.arange(N, dtype=torch.int64, device=cache.device) + 1)
    out = torch.empty(L, dtype=torch.int64, device=cache.device)
    for l in range(L):
        words = delivered_layer(torch, cache, l, idx, N, G).view(torch.int64)      # [N, S/8]
        out[l] = ((words * T_dev).sum(dim=1) * w).sum()
    return out.cpu().numpy().view(np.uint64)


# ---- oracle side ----------------------------------------------------------------------------------
class FamilyDigests:
    """Per-layer digest prefix sums of one prefix family (payload seed, payload ids in prefix
    order) from the oracle: RangeGet of every chunk (regenerated by synth), the chunk's per-layer
    inner sums c[j][l] = sum_k T[k] * x[j][l][k], then P[n][l] = sum_{j<n} (2j+1) c[j][l]."""

    def __init__(self, seed, payload_ids, n_max, L, S, T, threads=None):
        from oracle.store import ChunkStore  # noqa: F401  (the store whose RangeGet we regenerate)
        self.L, self.S = L, S
        n_max = min(n_max, len(payload_ids))
        c = np.zeros((n_max, L), dtype=np.uint64)

        def one(j):
            obj = synth.chunk_payload(seed, payload_ids[j], L * S)          # RangeGet(H_j, 0, L*S)
            x = obj.view(np.uint64).reshape(L, S // 8)                       # layer l = [lS, (l+1)S)
            with np.errstate(over="ignore"):
                c[j] = (x * T).sum(axis=1, dtype=np.uint64)

        with ThreadPoolExecutor(threads or host_threads()) as ex:
            list(ex.map(one, range(n_max)))
        w = (2 * np.arange(n_max, dtype=np.uint64) + 1)[:, None]
        with np.errstate(over="ignore"):
            self.P = np.concatenate([np.zeros((1, L), np.uint64), np.cumsum(c * w, axis=0, dtype=np.uint64)])
        self.bytes = n_max * L * S

    def request(self, n):
        """Expected D_l (l = 0..L-1) of a request holding the family's first n chunks."""
        return self.P[n]


def oracle_layer_payload(lay, seed, keys, payload_ids, layer):
    """B_l of a request by the oracle's Alg. A1 gather (oracle.assemble.gather_layer) over a store
    that regenerates chunks from synth (RangeGet)."""
    from oracle.assemble import gather_layer
    from oracle.descriptor import FlatTarget, build_descriptor
    from oracle.geometry import chunk_layer_bytes

    class _Regen:
        def __init__(self):
            self.ids = {bytes(k): p for k, p in zip(keys, payload_ids)}

        def __contains__(self, k):
            return bytes(k) in self.ids

        def range_get(self, k, off, n):
            return synth.chunk_payload_range(seed, self.ids[bytes(k)], off, n).tobytes()

    st = _Regen()
    N = len(keys)
    desc = build_descriptor(st, [bytes(k) for k in keys], lay, FlatTarget(0, N * lay.num_layers * chunk_layer_bytes(lay)))
    return np.frombuffer(gather_layer(st, desc, layer), dtype=np.uint8)


def full_check(torch, lay, seed, keys, payload_ids, cache, idx, layers):
    """Sampled request in full: the delivered [N][S] of each layer in `layers` against the oracle's
    B_l byte for byte.  Returns (ok, bytes compared, oracle seconds)."""
    N, G = len(keys), lay.chunk_tokens
    t0 = time.perf_counter()
    ok, nbytes, t_or = True, 0, 0.0
    for l in layers:
        t = time.perf_counter()
        want = oracle_layer_payload(lay, seed, keys, payload_ids, l)
        t_or += time.perf_counter() - t
        got = delivered_layer(torch, cache, l, idx, N, G).reshape(-1).cpu().numpy()
        ok &= bool(np.array_equal(got, want))
        nbytes += want.size
    return ok, nbytes, t_or, time.perf_counter() - t0
