"""Acceptance criteria 6-9 of the reference suite (acceptance.cpp:277-450):
the paper's phenomena, reproduced number for number.

Each criterion runs as one batch (criterion 8: 126 node runs; criterion 9:
four 8-node clusters).  CPU: the C oracle against the reference-generated
fixtures.  GPU: the device engines against the same fixtures, plus the
criteria's own pass conditions.
"""
from __future__ import annotations

import pytest

import acceptance_cases as ac


def _check_phenomena(c67, c8, c9):
    # 6: stall-free batching starves bursts; fair batching absorbs them
    sar, fair = c67["x2.0_sarathi"], c67["x2.0_fairbatch"]
    assert sar["ttft_viol"] >= 1 and 2 * fair["ttft_viol"] <= sar["ttft_viol"]
    assert not (set(fair["env_set"]) - set(sar["env_set"]))  # no net-new envelope misses
    assert not sar["incomplete"] and not fair["incomplete"]
    # 7: tail ordering
    assert c67["x1.5_fairbatch"]["p99_ttft"] < c67["x1.5_sarathi"]["p99_ttft"]
    assert c67["x1.5_fairbatch"]["p99_tpot"] <= 50.0
    assert c67["x1.5_prefill_first"]["p99_tpot"] > 50.0
    # 8: peak goodput fb-pab >= fb > best baseline on every shape
    for shape, v in c8.items():
        assert v["pab"] >= v["fb"] > max(v["sar"], v["pf"]), shape
    # 9: budget-based balancing beats counts and degrades less when stale
    assert c9["pab_lb_0"] >= c9["count_lb_0"]
    assert c9["count_lb_0"] - c9["count_lb_5000"] > c9["pab_lb_0"] - c9["pab_lb_5000"]


def test_acceptance_values_on_oracle(oracle, golden):
    def runner(b):
        o = oracle.run(b, nthreads=8)
        return o.results, o.records

    c67 = ac.crit67(oracle.generate_bursty, runner)
    c8 = ac.crit8(oracle.generate_bursty, runner)
    c9 = ac.crit9(oracle.generate_bursty,
                  lambda r, c, lb, h: oracle.run_cluster(r, c, lb, h).records)
    assert c67 == golden["acceptance"]["crit67"]
    assert c8 == golden["acceptance"]["crit8"]
    assert c9 == golden["acceptance"]["crit9"]
    _check_phenomena(c67, c8, c9)


@pytest.mark.gpu
def test_acceptance_values_on_gpu(fb, golden):
    from paper_2510_14392_b200.cluster import run_cluster

    def runner(b):
        a = fb.Arena(0)
        a.load(b)
        a.run()
        res, rec = a.results(), a.records()
        a.close()
        return res, rec

    c67 = ac.crit67(fb.generate_bursty, runner)
    c8 = ac.crit8(fb.generate_bursty, runner)
    c9 = ac.crit9(fb.generate_bursty, lambda r, c, lb, h: run_cluster(r, c, lb, h).records)
    assert c67 == golden["acceptance"]["crit67"]
    assert c8 == golden["acceptance"]["crit8"]
    assert c9 == golden["acceptance"]["crit9"]
    _check_phenomena(c67, c8, c9)


@pytest.mark.gpu
def test_scenario_drivers_on_gpu(fb, tmp_path):
    """run_scenario / sweep_scenario / tune_sarathi on the shipped demo scenario."""
    import json
    from paper_2510_14392_b200 import scenario
    sc_json = {
        "name": "single-node-demo",
        "trace": {"bursty": {"base_rate": 1.0, "burst_rate": 10.0, "burst_duration_ms": 1500,
                             "idle_duration_ms": 3500, "prompt_mean": 892, "prompt_p90": 1776,
                             "output_mean": 377, "output_p90": 742, "seed": 33,
                             "horizon_ms": 40000}, "scale": 1.5},
        "slo": {"ttft_ms": 500, "tpot_ms": 50},
        "scheduler": {"policy": "fairbatch", "token_budget": 2048},
        "cost_model": {"truth": {"a_ms": 5.0, "b_ms_per_token": 0.05,
                                 "c_ms_per_context_token": 0.0001}, "noise_amplitude": 0.0},
        "run": {"horizon_ms": 3600000, "seed": 42, "out_dir": "out/single"},
    }
    p = tmp_path / "s.json"
    p.write_text(json.dumps(sc_json))
    sc = scenario.load_scenario(str(p))
    rep = scenario.run_scenario(sc)
    assert rep.total_requests > 0 and rep.ttft.p99 == pytest.approx(444.204)
    rows = scenario.sweep_scenario(sc, [1.0, 2.0], ["fairbatch", "sarathi"])
    assert len(rows) == 4 and rows[0].effective_rps == pytest.approx(rep.effective_rps)
    tune, best = scenario.tune_sarathi(sc, [256, 512])
    assert best in (256, 512) and len(tune) == 2
