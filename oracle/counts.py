"""Element counts and recompute-token deltas (oracle; test infrastructure only).

Table A4 ("client-visible element count for S3RDMA Agg bounded
layerwise aggregation"): a prefix of N matched chunks issues N*L range reads
("original elements"); bounded aggregation packs floor(agg/S) of them per
aggregate, giving ceil(N*L / floor(agg/S)) elements.  N is the number of
matched G-token chunks at hit rate r of a C-token context: floor(C*r/G).

P:1374-1377 and Table A3: a cache hit boundary at P tokens
reuses floor(P/G)*G tokens, so going from G=16 to G=512 recomputes
floor(P/16)*16 - floor(P/512)*512 extra tokens ("up to 496").
"""


def matched_chunks(context_tokens: int, hit_rate: float, G: int) -> int:
    return int(context_tokens * hit_rate) // G


def original_elements(n_chunks: int, L: int) -> int:
    return n_chunks * L


def elements_per_aggregate(agg_bytes: int, S: int) -> int:
    return agg_bytes // S


def elements_after_aggregation(n_chunks: int, L: int, agg_bytes: int, S: int) -> int:
    per = elements_per_aggregate(agg_bytes, S)
    return -(-(n_chunks * L) // per)


def reused_tokens(P: int, G: int) -> int:
    return (P // G) * G


def recompute_delta(P: int, G_fine: int = 16, G_coarse: int = 512) -> int:
    return reused_tokens(P, G_fine) - reused_tokens(P, G_coarse)
