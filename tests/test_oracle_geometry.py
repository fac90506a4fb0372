"""Pins for oracle.geometry / oracle.counts: values the paper prints (tests/golden) and closed forms."""
import pytest

from oracle import geometry as g
from oracle import counts
from conftest import read_golden

LLAMA8B = g.Layout(32, 8, 128, 2, 16)


@pytest.mark.parametrize("row", read_golden("eq1_anchors.csv"), ids=lambda r: r["quantity"])
def test_eq1_paper_anchors(row):
    q = row["quantity"]
    lay = g.Layout(int(row["L"]), int(row["n_kv"]), int(row["d"]), int(row["p"]), int(row["G"]))
    want = int(row["value_bytes"])
    if q == "per_token_layer":
        assert g.per_token_layer_bytes(lay) == want
    elif q == "chunk_layer":
        assert g.chunk_layer_bytes(lay) == want
    elif q == "payload_W":
        assert g.matched_payload_bytes(lay, int(row["N"])) == want
    else:
        raise AssertionError(q)


def test_binary_units_of_printed_sizes():
    # "448 MB" and "7 GB" are binary: 448 MiB and 7 GiB exactly.
    G64 = g.Layout(32, 8, 128, 2, 64)
    assert g.matched_payload_bytes(G64, 56) == 448 * 2**20
    assert g.matched_payload_bytes(G64, 896) == 7 * 2**30


def test_layer_ranges_tile_the_chunk():
    for lay in (LLAMA8B, g.Layout(2, 2, 16, 2, 16), g.Layout(3, 1, 1, 1, 1)):
        S = g.chunk_layer_bytes(lay)
        end = 0
        for l in range(lay.num_layers):
            off, n = g.layer_range(lay, l)
            assert off == end and n == S
            end = off + n
        assert end == g.chunk_bytes(lay)
        with pytest.raises(IndexError):
            g.layer_range(lay, lay.num_layers)
        with pytest.raises(IndexError):
            g.layer_range(lay, -1)


def test_spec_examples_layer_range():
    assert g.layer_range(LLAMA8B, 31) == (2031616, 65536)
    assert g.layer_range(g.Layout(32, 8, 128, 2, 64), 1) == (262144, 262144)


def test_kv_token_bytes_is_L_times_per_layer():
    for lay in (LLAMA8B, g.Layout(80, 8, 128, 2, 16), g.Layout(1, 1, 1, 1, 1)):
        assert g.kv_token_bytes(lay) == lay.num_layers * g.per_token_layer_bytes(lay)
    assert g.per_token_layer_bytes(g.Layout(1, 1, 1, 1, 1)) == 2
    assert g.chunk_layer_bytes(g.Layout(1, 1, 1, 1, 1)) == 2


def test_payload_W_sums_layers():
    lay = g.Layout(5, 3, 8, 2, 4)
    for N in (0, 1, 7):
        assert g.matched_payload_bytes(lay, N) == sum(N * g.layer_range(lay, l)[1] for l in range(5))


def test_table_a5_required_bandwidth_closed_form():
    # Table A5: Req. BW = per-layer KV bytes / per-layer compute, decimal GB/s, from T_total/L.
    for r in read_golden("table_a5.csv"):
        D = g.matched_bytes_per_layer(LLAMA8B, int(r["context"]), float(r["hit"]))
        assert D == int(r["cached"]) * 4096
        t_layer = float(r["t_total_ms"]) / 32 / 1e3
        assert abs(t_layer * 1e3 - float(r["t_layer_ms"])) <= 0.005 + 1e-9
        # the paper divides by the rounded per-layer time it prints
        req = D / (float(r["t_layer_ms"]) / 1e3) / 1e9
        assert abs(req - float(r["req_gbs"])) <= 0.006, (r, req)


def test_eq2_mode_rule():
    theta = 512 * 2**20
    assert g.delivery_mode(theta - 1, theta) == "chunkwise"
    assert g.delivery_mode(theta, theta) == "layerwise"
    # 4K configurations fall on the chunkwise side, 16K/64K on the layerwise side (G=64, 87.5% hit).
    G64 = g.Layout(32, 8, 128, 2, 64)
    assert g.delivery_mode(g.matched_payload_bytes(G64, counts.matched_chunks(4096, 0.875, 64)), theta) == "chunkwise"
    assert g.delivery_mode(g.matched_payload_bytes(G64, counts.matched_chunks(16384, 0.875, 64)), theta) == "layerwise"
    assert g.delivery_mode(g.matched_payload_bytes(G64, counts.matched_chunks(65536, 0.5, 64)), theta) == "layerwise"


@pytest.mark.parametrize("row", read_golden("table_a4.csv"))
def test_table_a4_counts(row):
    C, G = int(row["context"]), int(row["chunk_tokens"])
    lay = g.Layout(32, 8, 128, 2, G)
    S = g.chunk_layer_bytes(lay)
    N = counts.matched_chunks(C, 0.875, G)
    assert N == int(row["number"])
    assert counts.original_elements(N, 32) == int(row["original_elements"])
    assert counts.elements_per_aggregate(int(row["agg_bytes"]), S) == int(row["elements_per_agg"])
    after = counts.elements_after_aggregation(N, 32, int(row["agg_bytes"]), S)
    assert after == int(row["elements_after_agg"])
    assert counts.original_elements(N, 32) // after == int(row["reduction"])


def test_recompute_delta_496():
    # P:1374-1377 / Table A3 note: each boundary recomputes up to 496 tokens going from G=16 to G=512.
    worst = max(counts.recompute_delta(P) for P in range(1, 70000))
    assert worst == 496
    for M in (4096, 16384, 65536):
        assert counts.recompute_delta(M - 1) == 496
        assert counts.recompute_delta(M) == 0
