"""Slot-size effect, continued (r02_slot_size_sweep.txt): is it the fetch kernel or the memory system?
(A) a library strided copy -- torch copy_ of src.view(N, L, S)[:, l, :] into a contiguous (N, S)
    buffer, every layer -- at slot sizes L*S of 2, 2.5, 4, 5 MiB; (B) the fetch kernel at the same
    slot sizes with 16/32/64 KiB copy units."""
import json, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2605_22850_b200 as oc
import synth
dev = torch.device("cuda", 0)
S, N = 65536, 1792


def timeit(fn, reps=6):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for L in (32, 40, 64, 80):
    src = torch.randint(0, 256, (N, L, S), dtype=torch.uint8, device=dev)
    dst = torch.empty((N, S), dtype=torch.uint8, device=dev)
    W = 2 * N * S * L

    def lib_copy():
        for l in range(L):
            dst.copy_(src[:, l, :])
    # 8-byte elements: the same bytes with wider accesses
    src64, dst64 = src.view(torch.int64), dst.view(torch.int64)

    def lib_copy64():
        for l in range(L):
            dst64.copy_(src64[:, l, :])
    r = {"L": L, "slot_MiB": L * S / 2**20,
         "torch_strided_copy_u8_TBps": round(W / timeit(lib_copy) / 1e9, 3),
         "torch_strided_copy_i64_TBps": round(W / timeit(lib_copy64) / 1e9, 3)}
    del src, dst, src64, dst64
    torch.cuda.empty_cache()
    lay_t = (L, 8, 128, 2, 16)
    G, Bs = 16, 16
    row, S_, chunk = oc.geometry(lay_t)
    store = oc.Store(lay_t, capacity=N, device=0)
    (tok,), _ = synth.family_streams(900, G, 0, [N])
    keys = oc.chunk_keys(tok, G)
    for b0 in range(0, N, 256):
        store.put_chunks(keys[b0:b0 + 256], torch.randint(0, 256, (min(N, b0 + 256) - b0, chunk), dtype=torch.uint8, device=dev))
    flat = torch.empty(N * L * S, dtype=torch.uint8, device=dev)
    df = oc.build_descriptor(store, keys, lay_t, oc.FlatTarget(flat.data_ptr(), N * L * S))
    s = torch.cuda.current_stream()
    for ub in (16384, 32768, 65536):
        r[f"fetch_flat_u{ub // 1024}k_TBps"] = round(W / timeit(lambda: df.fetch_layerwise(s, engine=oc.COPY_BULK, unit_bytes=ub)) / 1e9, 3)
    print(json.dumps(r), flush=True)
    df.close()
    store.close()
    del flat
    torch.cuda.empty_cache()
