"""Named parity scenarios shared by the golden-fixture generator and the tests.

Each scenario is a list of (profile, horizon_ms, scale, engine-config kwargs,
run horizon) built with a caller-supplied trace generator, so the same batch
can be materialised with the reference's generate_bursty (fixtures), the C
oracle's (CPU tests) or the product's (GPU tests).
"""
from __future__ import annotations

import hashlib

import numpy as np

from paper_2510_14392_b200 import _abi
from paper_2510_14392_b200.batch import Batch, CostModel, Rows, engine_config, ms_to_us

MODEL = CostModel(5.0, 0.05, 0.0001)
BUDGET = {"fairbatch": 2048, "fairbatch_pab": 2048, "sarathi": 512, "prefill_first": 8192}


def profile(base, burst, bms, ims, pm, p9, om, o9, seed, ttft=500.0, tpot=50.0):
    return _abi.BurstProfile(float(base), float(burst), ms_to_us(bms), ms_to_us(ims), float(pm),
                             float(p9), float(om), float(o9), ms_to_us(ttft), ms_to_us(tpot),
                             seed)


def qwen(seed, ttft=500.0, tpot=50.0):
    return profile(1.0, 10.0, 1500, 3500, 892, 1776, 377, 742, seed, ttft, tpot)


TRACE_PROFILES = {
    "c1_poisson": (profile(4.0, 4.0, 1500, 3500, 892, 1776, 377, 742, 33), 250_000.0),
    "qwen_33": (qwen(33), 40_000.0),
    "qwen_0": (qwen(0), 40_000.0),
    "qwen_7": (qwen(7), 40_000.0),
    "balanced_7": (profile(2.0, 6.0, 1000, 2000, 892, 1776, 377, 742, 7), 40_000.0),
    "short_bursty_11": (profile(2.0, 6.0, 1000, 2000, 688, 1599, 237, 470, 11), 40_000.0),
    "long_prompt_13": (profile(1.5, 5.0, 1500, 2500, 1604, 3561, 114, 392, 13, ttft=2000.0),
                       40_000.0),
    "cluster8_5": (profile(30.0, 90.0, 800, 1600, 892, 1776, 250, 500, 5), 30_000.0),
}


def rows_digest(rows) -> str:
    h = hashlib.sha256()
    for a in (rows.arrival_us, rows.prompt_len, rows.output_len, rows.ttft_us, rows.tpot_us):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _add(b: Batch, gen, prof, gen_h_ms, scale, pol, run_h_ms=3.6e6, **kw):
    rows = gen(prof, ms_to_us(gen_h_ms))
    if scale != 1.0:
        rows = rows.scaled(scale)
    tt = prof.ttft_us / 1000.0
    tp = prof.tpot_us / 1000.0
    cfg = engine_config(pol, kw.pop("budget", BUDGET[pol]), kw.pop("model", MODEL), tt, tp, **kw)
    b.add(rows, cfg, ms_to_us(run_h_ms))


def scenario_c1(gen) -> Batch:
    """C1 under every policy, plus noisy fair-batching variants."""
    b = Batch()
    prof, h = TRACE_PROFILES["c1_poisson"]
    for pol in ("fairbatch", "sarathi", "prefill_first", "fairbatch_pab"):
        _add(b, gen, prof, h, 1.0, pol)
    _add(b, gen, prof, h, 1.0, "fairbatch", noise_amplitude=0.052, noise_seed=12345)
    _add(b, gen, prof, h, 1.0, "fairbatch_pab", noise_amplitude=0.052, noise_seed=99)
    return b


def scenario_mixed(gen, n_seeds=24) -> Batch:
    """qwen-like bursts at 1x..3x load over every policy, with noise, max_active
    limits and short horizons (incomplete runs, arrivals past the horizon)."""
    b = Batch()
    pols = ("prefill_first", "sarathi", "fairbatch", "fairbatch_pab")
    for s in range(n_seeds):
        pol = pols[s % 4]
        _add(b, gen, qwen(s), 40_000.0, (1.0, 1.5, 2.0, 3.0)[(s // 4) % 4], pol,
             run_h_ms=3.6e6 if s % 7 else 20_000.0,
             noise_amplitude=0.05 if s % 3 == 0 else 0.0, noise_seed=7 * s + 1,
             max_active=(0, 0, 0, 8, 20)[s % 5])
    return b


def scenario_pab_overload(gen) -> Batch:
    """fairbatch_pab under 2x-4x overload: many admission rejects."""
    b = Batch()
    for s, sc in ((33, 2.0), (5, 3.0), (9, 4.0)):
        _add(b, gen, qwen(s), 40_000.0, sc, "fairbatch_pab")
        _add(b, gen, qwen(s), 40_000.0, sc, "fairbatch_pab", max_active=12)
    prof, h = TRACE_PROFILES["long_prompt_13"]
    _add(b, gen, prof, h, 2.8, "fairbatch_pab")
    return b


def scenario_large_live(gen) -> Batch:
    """Heavy overload where more than 64 tasks are visible at once (exercises
    the global-memory scratch path of the warp engine)."""
    b = Batch()
    prof, h = TRACE_PROFILES["balanced_7"]
    for pol in ("fairbatch", "sarathi", "prefill_first", "fairbatch_pab"):
        _add(b, gen, prof, 40_000.0, 12.0, pol, run_h_ms=8_000.0)
    _add(b, gen, prof, 40_000.0, 12.0, "fairbatch", run_h_ms=8_000.0,
         model=CostModel(5.0, 0.05, 0.001))
    _add(b, gen, prof, 40_000.0, 12.0, "sarathi", run_h_ms=8_000.0, max_active=100)
    return b


def wide_rows(n=5000, gap_us=8, seed=0):
    """C4-like decode-heavy burst: n arrivals every gap_us, varied lengths."""
    rng = np.random.default_rng(seed)
    arr = np.arange(n, dtype=np.int64) * gap_us
    prompt = rng.integers(16, 96, n).astype(np.int32)
    output = rng.integers(2, 40, n).astype(np.int32)
    return Rows(arr, prompt, output, np.full(n, 500_000, np.int64), np.full(n, 50_000, np.int64))


def scenario_wide(gen) -> Batch:
    """More than 512 live requests (the CTA-wide engine): selection windows,
    early scan termination, activation moves and completions at large A."""
    b = Batch()
    rows = wide_rows()
    m = CostModel(5.0, 0.01, 1e-6)  # SURVEY §8d C4 model
    for pol, budget in (("fairbatch", 1 << 20), ("sarathi", 512), ("prefill_first", 8192),
                        ("fairbatch_pab", 1 << 20)):
        b.add(rows, engine_config(pol, budget, m, 500, 50), ms_to_us(2_000.0))
    b.add(rows, engine_config("fairbatch", 1 << 20, m, 500, 50, noise_amplitude=0.05,
                              noise_seed=3, max_active=1500), ms_to_us(2_000.0))
    b.add(wide_rows(3000, 40, 1), engine_config("fairbatch", 4096, CostModel(5.0, 0.05, 1e-4),
                                                500, 50), ms_to_us(3_000.0))
    prof, h = TRACE_PROFILES["balanced_7"]
    _add(b, gen, prof, 40_000.0, 40.0, "fairbatch", run_h_ms=3_000.0)
    return b


def scenario_c2_subset(gen, seeds=range(0, 16)) -> Batch:
    """C2 (qwen x1.5, sarathi 512 vs fairbatch 2048) for a few seeds."""
    b = Batch()
    for s in seeds:
        _add(b, gen, qwen(s), 40_000.0, 1.5, "sarathi")
        _add(b, gen, qwen(s), 40_000.0, 1.5, "fairbatch")
    return b


SCENARIOS = {
    "c1": scenario_c1,
    "mixed": scenario_mixed,
    "pab_overload": scenario_pab_overload,
    "large_live": scenario_large_live,
    "c2_subset": scenario_c2_subset,
    "wide": scenario_wide,
}


def cluster_cases(gen):
    """run_cluster parity cases: (name, rows, node cfgs, LbConfig, horizon_us).
    The 8-node trace is cluster8.json's (acceptance.cpp:403-414); the last
    case is BASELINE config 5 (64 nodes)."""
    from paper_2510_14392_b200.cluster import LbConfig
    prof, h = TRACE_PROFILES["cluster8_5"]
    rows = gen(prof, ms_to_us(h))
    out = []
    for name, pol, lat, nn, hz in (("pab0_8", "pab_lb", 0.0, 8, 3.6e6),
                                   ("count0_8", "count_lb", 0.0, 8, 3.6e6),
                                   ("pab5000_8", "pab_lb", 5000.0, 8, 3.6e6),
                                   ("count37_3", "count_lb", 37.0, 3, 3.6e6),
                                   ("pab_hz10s_8", "pab_lb", 0.0, 8, 10_000.0),
                                   ("pab20_2", "pab_lb", 20.0, 2, 3.6e6)):
        node_pol = "fairbatch_pab" if pol == "pab_lb" else "fairbatch"
        cfgs = [engine_config(node_pol, 2048, MODEL, 500, 50) for _ in range(nn)]
        out.append((name, rows, cfgs, LbConfig(pol, 1, lat), ms_to_us(hz)))
    p5 = profile(240.0, 720.0, 800, 1600, 892, 1776, 250, 500, 5)
    rows5 = gen(p5, ms_to_us(30_000.0))
    cfgs5 = [engine_config("fairbatch_pab", 2048, MODEL, 500, 50) for _ in range(64)]
    out.append(("c5_pab0_64", rows5, cfgs5, LbConfig("pab_lb", 1, 0.0), ms_to_us(3.6e6)))
    return out


def reroute_cluster_cases(gen):
    """run_cluster with retry_reroute (cluster.cpp:222-237): the
    test_cluster.cpp:225-250 trace (a giant prompt saturates one node), and
    overloaded PAB clusters whose admission rejects (then reroutes) requests."""
    from paper_2510_14392_b200.batch import Rows
    from paper_2510_14392_b200.cluster import LbConfig
    t_model = CostModel(5.0, 0.01, 0.0001)
    out = []
    rows = Rows([0, 1000, 2000], [45_000, 45_000, 9000], [300, 300, 20],
                [500_000] * 3, [50_000] * 3)
    cfg = engine_config("fairbatch_pab", 8192, t_model, 500, 50)
    out.append(("rr_giant_2", rows, [cfg, cfg], LbConfig("pab_lb", 1, 0.0, retry_reroute=True),
                ms_to_us(3_600_000.0)))
    prof = profile(4.0, 40.0, 800, 1600, 2000, 6000, 120, 260, 11)
    rows_o = gen(prof, ms_to_us(20_000.0))
    for name, nn, lat, pol in (("rr_pab0_4", 4, 0.0, "pab_lb"), ("rr_pab30_3", 3, 30.0, "pab_lb"),
                               ("rr_count0_4", 4, 0.0, "count_lb")):
        cfgs = [engine_config("fairbatch_pab", 2048, MODEL, 500, 50) for _ in range(nn)]
        out.append((name, rows_o, cfgs, LbConfig(pol, 1, lat, retry_reroute=True),
                    ms_to_us(3.6e6)))
    # noise, max_active and a report interval of 2 under rerouting
    cfgs = [engine_config("fairbatch_pab", 2048, MODEL, 500, 50, noise_amplitude=0.04,
                          noise_seed=11 + i, max_active=(0, 12, 0, 20)[i]) for i in range(4)]
    out.append(("rr_mixed_4", rows_o, cfgs, LbConfig("pab_lb", 2, 10.0, retry_reroute=True),
                ms_to_us(3.6e6)))
    # the same overload without rerouting (rejected requests stay rejected)
    cfgs = [engine_config("fairbatch_pab", 2048, MODEL, 500, 50) for _ in range(4)]
    out.append(("rr_off_pab0_4", rows_o, cfgs, LbConfig("pab_lb", 1, 0.0), ms_to_us(3.6e6)))
    return out


def summarize(results: np.ndarray, records: np.ndarray) -> dict:
    """Compact, exact summary of a run for fixtures."""
    keys = ("steps", "plan_digest", "end_time_us", "n_arrived", "n_rejected", "sum_entries",
            "sum_new_tokens", "incomplete")
    return {
        "results": [{k: int(r[k]) for k in keys} for r in results],
        "records_sha256": hashlib.sha256(records.tobytes()).hexdigest(),
    }
