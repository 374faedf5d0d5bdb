"""The five BASELINE.json configurations as concrete synthetic inputs
(SURVEY §8d).  Traces are generated on the host with the product's
generate_bursty (workload.cpp:244-298), identical for CPU and GPU runs.

  C1  single-node FairBatching, 931-request Poisson trace
  C2  Sarathi vs FairBatching A/B over 2048 seeds -> 4096 instances (bench)
  C3  request-rate x SLO x policy grid, 65,536 instances
  C4  decode-heavy, 120,000 live requests per instance
  C5  64-node cluster (load-estimation dispatch) -- see cluster.py

Every builder takes an optional `gen(profile, horizon_us) -> Rows` (default:
the product's fbgpu.generate_bursty) and `scale(rows, factor) -> Rows`
(default: Rows.scaled), so the reference arm of bench.py and the golden
fixtures build the identical batches with the reference's own generator
(tests/backends.py RefLib) without loading libfbgpu.so.
"""
from __future__ import annotations

import numpy as np

from . import fbgpu
from .batch import Batch, CostModel, Rows, engine_config, ms_to_us

MODEL_7B = CostModel(5.0, 0.05, 0.0001)  # single_node.json:21, acceptance.cpp:59
HORIZON_RUN_US = ms_to_us(3.6e6)  # acceptance.cpp:98


def qwen_profile(seed: int, ttft_ms: float = 500.0, tpot_ms: float = 50.0):
    """acceptance.cpp:73-85."""
    return fbgpu.burst_profile(1.0, 10.0, 1500.0, 3500.0, 892.0, 1776.0, 377.0, 742.0, seed,
                               ttft_ms, tpot_ms)


def _gen(gen):
    return fbgpu.generate_bursty if gen is None else gen


def _scale(scale):
    return (lambda rows, f: rows.scaled(f)) if scale is None else scale


def c1_rows(gen=None) -> Rows:
    """C1: pure Poisson 4 rps, seed 33, 250 s -> 931 requests."""
    p = fbgpu.burst_profile(4.0, 4.0, 1500.0, 3500.0, 892.0, 1776.0, 377.0, 742.0, 33)
    return _gen(gen)(p, ms_to_us(250_000.0))


def c1_batch(policies=("fairbatch",), gen=None) -> Batch:
    b = Batch()
    rows = c1_rows(gen)
    off = b.add_rows(rows)
    budgets = {"fairbatch": 2048, "fairbatch_pab": 2048, "sarathi": 512, "prefill_first": 8192}
    for pol in policies:
        b.add_instance(engine_config(pol, budgets[pol], MODEL_7B, 500, 50), off, len(rows),
                       HORIZON_RUN_US, rows.offered_rps())
    return b


def c2_batch(n_seeds: int = 2048, seed0: int = 0, gen=None, scale=None, stride: int = 1) -> Batch:
    """C2: qwen_profile(seed) x1.5 over 40 s, seeds x {sarathi 512, fairbatch 2048}.
    Both policies of a seed share the same trace rows.  `stride` > 1 takes
    every stride-th seed of the range (bounded CPU samples of the same sweep)."""
    b = Batch()
    gen, scale = _gen(gen), _scale(scale)
    for s in range(seed0, seed0 + n_seeds, stride):
        rows = scale(gen(qwen_profile(s), ms_to_us(40_000.0)), 1.5)
        off = b.add_rows(rows)
        rps = rows.offered_rps()
        b.add_instance(engine_config("sarathi", 512, MODEL_7B, 500, 50), off, len(rows),
                       HORIZON_RUN_US, rps)
        b.add_instance(engine_config("fairbatch", 2048, MODEL_7B, 500, 50), off, len(rows),
                       HORIZON_RUN_US, rps)
    return b


C3_SCALES = tuple(float(x) for x in np.geomspace(0.5, 4.0, 16))
C3_TTFT = (500.0, 1000.0, 1500.0, 2000.0)
C3_TPOT = (50.0, 100.0, 150.0, 200.0)
C3_POLICIES = (("prefill_first", 8192), ("sarathi", 512), ("fairbatch", 2048),
               ("fairbatch_pab", 2048))


def c3_batch(n_seeds: int = 64, scales=C3_SCALES, ttfts=C3_TTFT, tpots=C3_TPOT,
             policies=C3_POLICIES, horizon_ms: float = 40_000.0, shard: int = 0,
             n_shards: int = 1, seed0: int = 0, gen=None, scale=None) -> Batch:
    """C3: the "balanced" shape (acceptance.cpp:347) over a 40 s horizon,
    16 scales x 4 TTFT x 4 TPOT x 4 policies x 64 seeds = 65,536 instances
    (SURVEY §8d lists 16 seeds, which gives 16,384; BASELINE.json names
    65,536, so the seed axis is 64).  The
    SLOs are stamped per request and used as global_slo (scenario.cpp:142-143).
    Instances are dealt round-robin to `n_shards` shards (multi-GPU)."""
    b = Batch()
    gen, scale = _gen(gen), _scale(scale)
    idx = 0
    for seed in range(seed0, seed0 + n_seeds):
        base = gen(
            fbgpu.burst_profile(2.0, 6.0, 1000.0, 2000.0, 892.0, 1776.0, 377.0, 742.0, 7 + seed),
            ms_to_us(horizon_ms))
        for sc in scales:
            scaled = scale(base, sc)
            for tt in ttfts:
                for tp in tpots:
                    rows = scaled.with_slo(ms_to_us(tt), ms_to_us(tp))
                    off = None
                    for pol, budget in policies:
                        if idx % n_shards == shard:
                            if off is None:
                                off = b.add_rows(rows)
                            b.add_instance(engine_config(pol, budget, MODEL_7B, tt, tp), off,
                                           len(rows), HORIZON_RUN_US, rows.offered_rps())
                        idx += 1
    return b


def c4_rows(n_req: int = 120_000, gap_us: int = 8, prompt: int = 64, output: int = 4000) -> Rows:
    """C4: decode-heavy, one arrival every 8 us (all within 0.96 s), fixed lengths."""
    arr = np.arange(n_req, dtype=np.int64) * gap_us
    return Rows(arr, np.full(n_req, prompt, np.int32), np.full(n_req, output, np.int32),
                np.full(n_req, ms_to_us(500.0), np.int64), np.full(n_req, ms_to_us(50.0), np.int64))


def c4_batch(n_inst: int = 64, n_req: int = 120_000, horizon_ms: float = 1500.0) -> Batch:
    b = Batch()
    rows = c4_rows(n_req)
    off = b.add_rows(rows)
    model = CostModel(5.0, 0.01, 1e-6)
    for _ in range(n_inst):
        b.add_instance(engine_config("fairbatch", 1 << 20, model, 500, 50), off, len(rows),
                       ms_to_us(horizon_ms), rows.offered_rps())
    return b
