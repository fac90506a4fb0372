"""Probe: a 4K-token hit (Llama-3-8B layout, N = 256) from a pinned-host store into a FLAT target
(the paper's client buffer), engine AUTO (-> CE: direct strided copy-engine transfers, no SMs) vs
BULK (SM zero-copy reads), with the chain in 1, 4 and 8 slot runs (AUTO picks CE up to 4); device time per fetch (events around
the fetch and a wait on its last layer), best of 10 after 3 warm-ups."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import paper_2605_22850_b200 as oc  # noqa: E402
import synth  # noqa: E402

lay = synth.LLAMA3_8B.as_tuple()
L, G = lay[0], lay[4]
row, S, chunk = oc.geometry(lay)
N = 256
for runs in (1, 4, 8):
    st = oc.Store(lay, capacity=N + runs * 4, tier=oc.TIER_PINNED_HOST)
    (tok,), _ = synth.family_streams(7, G, 0, [N])
    keys = oc.chunk_keys(tok, G)
    per = N // runs
    for r in range(runs):                       # interleave filler chunks to break the slot runs
        st.put_chunks(keys[r * per:(r + 1) * per], torch.randint(0, 256, (per, chunk), dtype=torch.uint8))
        if r + 1 < runs:
            (ft,), _ = synth.family_streams(100 + r, G, 0, [2])
            st.put_chunks(oc.chunk_keys(ft, G), torch.zeros((2, chunk), dtype=torch.uint8))
    flat = torch.empty(L * N * S, dtype=torch.uint8, device="cuda")
    d = oc.build_descriptor(st, keys, lay, oc.FlatTarget(flat.data_ptr(), flat.numel()))
    s = torch.cuda.Stream()
    for name, eng in (("auto", oc.COPY_AUTO), ("bulk", oc.COPY_BULK)):
        best = 1e9
        for i in range(13):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            d.fetch_layerwise(s, engine=eng)
            d.wait_layer(L - 1, s)
            e1.record(s)
            s.synchronize()
            if i >= 3:
                best = min(best, e0.elapsed_time(e1))
        print(json.dumps({"probe": "flat_pinned_host", "slot_runs": runs, "engine": name,
                          "ms": round(best, 3), "pcie_read_GBps": round(N * S * L / best / 1e6, 1)}), flush=True)
    d.close()
    st.close()
