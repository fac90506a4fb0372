"""CPU oracle for the ObjectCache hot path (arxiv 2605.22850).

TEST INFRASTRUCTURE ONLY.  Nothing on the product path may import, call or
link this package: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` use it.  It shares
no code with ``paper_2605_22850_b200`` (the CUDA library) and neither side
imports the other; the only common module is ``synth`` (seeded inputs, no
method arithmetic).

Every function is a plain, slow restatement of a passage of PAPER.md, cited as
``P:<lines> <section/equation/algorithm>``.  Readings of silent or ambiguous
passages are numbered c1..c22 after SURVEY.md section 8(c) and listed in
DESIGN.md.  All parts are pinned by ``tests/test_oracle_*.py`` (paper-printed
values, closed forms, brute force, invariants); no part is "parity unpinned".

Modules
-------
geometry    Eq. 1 KV geometry, layer ranges, W = N*L*S, Eq. 2 mode rule
keys        rolling chunk hash H_i = Hash(H_{i-1} || tokens_i)           (c1)
prefix      longest prefix match: brute force, radix tree, key probe     (c17)
store       content-addressed immutable chunk store                      (c18)
descriptor  Table 1 descriptor + validation
assemble    Alg. A1 layer-major gather; paged scatter                    (c2-c5)
scheduler   Eqs. 4-7, Equal / KV-prop / BW-prop / Stall-opt / Calibrated (c8-c12)
stall       Eq. 3 TTFT model, free-running pipeline, discrete-event sim  (c14)
counts      Table A4 element counts, recompute-token delta
dispatch    Alg. A2 lines 6-7: weighted deficit round robin, held rates   (c21-c22)
"""
