"""The reference acceptance suite's phenomenon criteria (acceptance.cpp:277-450)
as batched workloads: criteria 6-8 are sets of independent run_node runs (one
device batch each), criterion 9 is four 8-node cluster runs.  The same code
computes the metrics from any backend's records, so the reference library
(fixtures), the C oracle and the GPU are compared number for number.
"""
from __future__ import annotations

import numpy as np

from paper_2510_14392_b200 import reports
from paper_2510_14392_b200.batch import Batch, CostModel, engine_config, ms_to_us
from paper_2510_14392_b200.cluster import LbConfig

from catalog import profile, qwen

MODEL = CostModel(5.0, 0.05, 0.0001)  # acceptance.cpp:59
RUN_H = ms_to_us(3.6e6)


def _stats(rec, rows):
    """run_stats (acceptance.cpp:97-121)."""
    rep = reports.scenario_report(rec, rows.arrival_us, rows.offered_rps())
    return {"ttft_viol": rep.ttft_violations, "env_miss": rep.envelope_misses,
            "p99_ttft": rep.ttft.p99, "p99_tpot": rep.max_tpot.p99,
            "goodput": reports.goodput(rec, rows.offered_rps())}


def _run(batch, runner):
    res, rec = runner(batch)
    ro = batch.record_offsets()
    return res, [rec[ro[i]:ro[i + 1]] for i in range(batch.n_instances)]


def crit67(gen, runner):
    """Criteria 6 and 7 on qwen_profile(33) scaled x2 and x1.5."""
    base = gen(qwen(33), ms_to_us(40_000.0))
    out = {}
    b = Batch()
    plan = []
    for sc in (2.0, 1.5):
        rows = base.scaled(sc)
        off = b.add_rows(rows)
        for pol, budget in (("sarathi", 512), ("fairbatch", 2048), ("prefill_first", 8192)):
            b.add_instance(engine_config(pol, budget, MODEL, 500, 50), off, len(rows), RUN_H)
            plan.append((sc, pol, rows))
    res, recs = _run(b, runner)
    for (sc, pol, rows), r, rec in zip(plan, res, recs):
        s = _stats(rec, rows)
        s["incomplete"] = int(r["incomplete"])
        env = set(np.nonzero((rec["flags"] & 32) != 0)[0].tolist())
        s["env_set"] = sorted(env)
        out[f"x{sc}_{pol}"] = s
    return out


SHAPES = (  # acceptance.cpp:345-349
    ("short-bursty", 688, 1599, 237, 470, 500, 11, 2.0, 6.0, 1000, 2000),
    ("balanced", 892, 1776, 377, 742, 500, 7, 2.0, 6.0, 1000, 2000),
    ("long-prompt", 1604, 3561, 114, 392, 2000, 13, 1.5, 5.0, 1500, 2500),
)
SCALES = (0.7, 1.0, 1.4, 2.0, 2.8, 4.0)
SARATHI_BUDGETS = (256, 384, 512, 768)


def crit8(gen, runner):
    """Peak goodput over load sweeps on three trace shapes (acceptance.cpp:336-399),
    all 126 runs in one batch."""
    b = Batch()
    plan = []
    for name, pm, p9, om, o9, ttft, seed, base_r, burst_r, bms, ims in SHAPES:
        base = gen(profile(base_r, burst_r, bms, ims, pm, p9, om, o9, seed, ttft=ttft),
                   ms_to_us(40_000.0))
        for sc in SCALES:
            rows = base.scaled(sc)
            off = b.add_rows(rows)
            runs = [("sarathi", bb) for bb in SARATHI_BUDGETS] + [
                ("prefill_first", 8192), ("fairbatch", 2048), ("fairbatch_pab", 2048)]
            for pol, budget in runs:
                b.add_instance(engine_config(pol, budget, MODEL, ttft, 50), off, len(rows), RUN_H)
                plan.append((name, pol, rows))
    _, recs = _run(b, runner)
    peak = {}
    for (name, pol, rows), rec in zip(plan, recs):
        g = reports.goodput(rec, rows.offered_rps())
        key = (name, pol)
        peak[key] = max(peak.get(key, 0.0), g)
    return {name: {"pab": peak[(name, "fairbatch_pab")], "fb": peak[(name, "fairbatch")],
                   "sar": peak[(name, "sarathi")], "pf": peak[(name, "prefill_first")]}
            for name, *_ in SHAPES}


def crit9(gen, cluster_runner):
    """Budget-based vs count-based balancing, fresh and stale (acceptance.cpp:403-450)."""
    p = profile(30.0, 90.0, 800, 1600, 892, 1776, 250, 500, 5)
    rows = gen(p, ms_to_us(30_000.0))
    out = {}
    for lbp, lat in (("count_lb", 0.0), ("pab_lb", 0.0), ("count_lb", 5000.0), ("pab_lb", 5000.0)):
        node = "fairbatch_pab" if lbp == "pab_lb" else "fairbatch"
        cfgs = [engine_config(node, 2048, MODEL, 500, 50) for _ in range(8)]
        rec = cluster_runner(rows, cfgs, LbConfig(lbp, 1, lat), RUN_H)
        out[f"{lbp}_{int(lat)}"] = reports.goodput(rec, rows.offered_rps())
    return out
