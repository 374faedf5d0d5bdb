"""Seeded random engine corpus: instances whose traces and configurations are
drawn across the space the reference's `run_node` accepts (every policy,
token budgets from 16 to 8192, chunk caps, scheduler and truth cost models of
different magnitudes including c = 0, truth noise, max_active, per-request or
uniform SLOs), so the engines' fast paths -- repeated plans, all-fit
shortcuts, rank reuse, the memory path -- are checked against the oracle /
reference on configurations no named scenario holds.  Test infrastructure.
"""
from __future__ import annotations

import numpy as np

from paper_2510_14392_b200.batch import Batch, CostModel, Rows, engine_config, ms_to_us

POLICIES = ("prefill_first", "sarathi", "fairbatch", "fairbatch_pab")


def random_rows(rng: np.random.Generator, uniform_slo: bool, wide: bool = False) -> Rows:
    # wide: thousands of requests arriving faster than they drain, so more
    # than 512 are live at once (the grid-wide engine)
    n = int(rng.integers(600, 4000)) if wide else int(rng.integers(1, 400))
    rate_per_ms = float(rng.choice([2.0, 8.0])) if wide else float(rng.choice([0.005, 0.02, 0.08, 0.3]))
    gaps = rng.exponential(1.0 / rate_per_ms, size=n)
    if rng.random() < 0.3:  # bursts: runs of simultaneous arrivals
        gaps[rng.random(n) < 0.4] = 0.0
    arrival = np.cumsum(np.round(gaps * 1000.0)).astype(np.int64)
    prompt = rng.integers(1, int(rng.choice([64, 600, 3000])) + 1, size=n).astype(np.int32)
    output = rng.integers(1, int(rng.choice([8, 120, 600])) + 1, size=n).astype(np.int32)
    if uniform_slo:
        ttft = np.full(n, ms_to_us(float(rng.choice([200.0, 500.0, 2000.0]))), np.int64)
        tpot = np.full(n, ms_to_us(float(rng.choice([20.0, 50.0, 100.0]))), np.int64)
    else:
        ttft = rng.integers(ms_to_us(100.0), ms_to_us(3000.0), size=n).astype(np.int64)
        tpot = rng.integers(ms_to_us(10.0), ms_to_us(200.0), size=n).astype(np.int64)
    return Rows(arrival, prompt, output, ttft, tpot)


def random_model(rng: np.random.Generator) -> CostModel:
    return CostModel(float(rng.choice([0.5, 1.0, 5.0, 12.5])),
                     float(rng.choice([0.001, 0.01, 0.05, 0.2])),
                     float(rng.choice([0.0, 1e-6, 1e-4, 1e-3])))


def random_batch(seed: int, n_inst: int, wide: bool = False) -> Batch:
    rng = np.random.default_rng(seed)
    b = Batch()
    for _ in range(n_inst):
        rows = random_rows(rng, uniform_slo=rng.random() < 0.75, wide=wide)
        pol = POLICIES[int(rng.integers(0, 4))]
        budget = int(rng.choice([16, 64, 512, 2048, 8192]))
        max_chunk = int(rng.integers(1, budget + 1)) if rng.random() < 0.3 else None
        model = random_model(rng)
        truth = random_model(rng) if rng.random() < 0.3 else None
        noisy = rng.random() < 0.3
        cfg = engine_config(pol, budget, model, float(rng.choice([300.0, 500.0, 1000.0])),
                            float(rng.choice([30.0, 50.0, 80.0])), max_chunk=max_chunk,
                            noise_amplitude=0.1 if noisy else 0.0,
                            noise_seed=int(rng.integers(0, 1 << 31)),
                            max_active=int(rng.choice([0, 0, 0, 4, 16])), truth=truth)
        horizon = ms_to_us(float(rng.choice([2_000.0, 20_000.0, 120_000.0])))
        b.add(rows, cfg, horizon)
    return b


def random_cluster(seed: int):
    """(rows, node configs, LbConfig, horizon_us) of a random run_cluster case:
    1-64 nodes of one random policy, pab / count balancing, report interval
    1-3, report latency 0-50 ms, a quarter with retry_reroute."""
    from paper_2510_14392_b200 import cluster
    rng = np.random.default_rng(seed)
    rows = random_rows(rng, uniform_slo=rng.random() < 0.7)
    nodes = int(rng.choice([1, 2, 3, 5, 8, 16, 33, 64]))
    pol = POLICIES[int(rng.integers(0, 4))]
    cfgs = [engine_config(pol, int(rng.choice([64, 512, 2048])), random_model(rng),
                          float(rng.choice([300.0, 500.0])), float(rng.choice([30.0, 50.0])),
                          max_active=int(rng.choice([0, 0, 4])))
            for _ in range(nodes)]
    lb = cluster.LbConfig(str(rng.choice(["pab_lb", "count_lb"])), int(rng.choice([1, 1, 2, 3])),
                          float(rng.choice([0.0, 0.0, 5.0, 50.0])),
                          retry_reroute=bool(rng.random() < 0.25))
    hz = ms_to_us(float(rng.choice([5_000.0, 60_000.0])))
    return rows, cfgs, lb, hz
