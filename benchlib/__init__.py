"""The legs of bench.py, one module per family (bench.py keeps the contract line and the orchestration).

common     metric, peaks, clock sampler, in-harness copy, compute-window models
headline   the N=1 workload (BASELINE configs[1]): the 4K-hit fetch, its roofline
e2e        public-API end to end: HBM tier (pipelined control plane) and pinned-host tier (PCIe)
stall      added TTFT over spin windows and over real prefill (GEMMs + attention)
configs    config 3 (64K hit, verified) and config 4 (70B under a shared cap, verified)
config5    mixed concurrent requests over 1..8 GPUs (strong scaling, NVLink peer reads, verified)
verify     oracle-side verification (sampled full checks, per-layer digests) -- test infrastructure
reference  the oracle arm (--impl reference, cpu_baseline)
extra      optional legs
"""
