"""CPU suite: pins the C oracle (and, where built, the reference library) to the
reference's own known-answer tests and to the committed golden fixtures.

Known answers restate /root/reference/proj/tests/test_sched.cpp and
test_engine.cpp; fixtures come from tests/golden/make_golden.py.
"""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

from catalog import SCENARIOS, TRACE_PROFILES, rows_digest, summarize
from fuzz import (K_MODEL, Rng, acceptance_corpus, decode_task, fb_config, gen_pab_instance,
                  prefill_task, raw_to_views, views)
from paper_2510_14392_b200 import _abi
from paper_2510_14392_b200.batch import Batch, CostModel, Rows, engine_config, ms_to_us

LIBS = ["oracle", "ref"]


@pytest.fixture(params=LIBS)
def cpu(request, oracle):
    if request.param == "oracle":
        return oracle
    return request.getfixturevalue("ref")


# --------------------------------------------------------------- sched known answers

def test_init_time_budget_known_answers(cpu):
    # test_sched.cpp:57-78
    assert cpu.init_time_budget(views(decode_task(0, 30, 100), decode_task(1, 80, 100))) == 50_000
    assert cpu.init_time_budget(views(decode_task(0, 120, 100))) == 120_000
    assert cpu.init_time_budget(views(decode_task(0, -20, 100))) == 50_000
    assert cpu.init_time_budget(views(prefill_task(0, 300, 1000, 0, 80.0),
                                      prefill_task(1, 200, 500, 0, 60.0))) == 60_000
    with pytest.raises(RuntimeError):
        cpu.init_time_budget(views())


def test_single_urgent_decode(cpu):
    # test_sched.cpp:80-89
    plan, e = cpu.form_batch(views(decode_task(7, 40, 1000)), fb_config())
    assert len(e) == 1 and e[0]["request_id"] == 7 and e[0]["new_tokens"] == 1
    assert plan["predicted_ms"] == pytest.approx(5.11)
    assert plan["init_time_budget_ms"] == pytest.approx(50.0)


def test_prefill_chunked_ahead_of_relaxed_decode(cpu):
    # test_sched.cpp:91-131
    t = views(decode_task(0, 45, 100), decode_task(1, 400, 2000), prefill_task(2, 350, 30_000, 0))
    plan, e = cpu.form_batch(t, fb_config(8192))
    after = 45.0 - 0.02
    chunk = int(np.floor(min(8192 - 1, after / 0.01)))
    assert [int(x) for x in e["request_id"][:2]] == [0, 2] and e[1]["new_tokens"] == chunk
    resid = after - 0.01 * chunk
    assert len(e) == (3 if 0.01 + 0.0001 * 2000.0 <= resid else 2)
    plan, e = cpu.form_batch(t, fb_config(2048))
    assert len(e) == 2 and e[1]["request_id"] == 2 and e[1]["new_tokens"] == 2047
    t[2]["new_tokens"] = 3000
    plan, e = cpu.form_batch(t, fb_config(16_384))
    assert [int(x) for x in e["request_id"]] == [0, 2, 1] and e[1]["new_tokens"] == 3000


def test_order_tie_break_and_empty(cpu):
    # test_sched.cpp:133-166
    plan, e = cpu.form_batch(views(decode_task(0, 20, 500), decode_task(1, 10, 500),
                                   prefill_task(2, 100, 50_000, 0)), fb_config())
    assert [int(x) for x in e["request_id"][:2]] == [1, 0]
    plan, e = cpu.form_batch(views(decode_task(10, 30, 100, 50.0, 5),
                                   decode_task(11, 30, 100, 50.0, 2)), fb_config())
    assert e[0]["request_id"] == 11
    plan, e = cpu.form_batch(views(decode_task(0, 10, 600_000)), fb_config())
    assert len(e) == 0 and plan["predicted_ms"] == 0.0


def test_sarathi_and_prefill_first(cpu):
    # test_sched.cpp:268-361
    t = views(*[decode_task(i, 100 + i, 500) for i in range(48)], prefill_task(100, 300, 2000, 0))
    plan, e = cpu.form_batch(t, fb_config(512, _abi.POLICY_SARATHI, 512))
    assert len(e) == 49
    assert int(e["new_tokens"][e["request_id"] == 100].sum()) == 512 - 48
    plan, e = cpu.form_batch(views(decode_task(0, 40, 100), decode_task(1, 90, 100)),
                             fb_config(512, _abi.POLICY_SARATHI, 512))
    assert len(e) == 2 and plan["token_budget_used"] == 2
    plan, e = cpu.form_batch(views(prefill_task(0, 400, 10_000, 0)),
                             fb_config(512, _abi.POLICY_SARATHI, 256))
    assert len(e) == 1 and e[0]["new_tokens"] == 256
    t = views(prefill_task(0, 200, 5000, 0, 50.0, 0),
              *[decode_task(i, 100, 200, 50.0, i) for i in range(1, 11)])
    plan, e = cpu.form_batch(t, fb_config(4096, _abi.POLICY_PREFILL_FIRST, 4096))
    assert len(e) == 1 and e[0]["request_id"] == 0 and e[0]["new_tokens"] == 4096
    t = views(*[decode_task(i, 100, 200) for i in range(3)], prefill_task(9, 300, 1000, 0, 50.0, 9))
    plan, e = cpu.form_batch(t, fb_config(4096, _abi.POLICY_PREFILL_FIRST, 4096))
    assert len(e) == 4 and e[0]["request_id"] == 0 and e[3]["request_id"] == 9
    assert e[3]["new_tokens"] == 1000


def test_pab_known_answers(cpu):
    # test_sched.cpp:401-421
    assert cpu.pab(views(), K_MODEL, 500_000, 50_000) == 49_009
    assert cpu.pab(views(decode_task(0, 100, 2000)), K_MODEL, 500_000, 50_000) == 44_883
    assert cpu.pab(views(decode_task(0, 100, 2000), prefill_task(1, 500, 10_000, 0)), K_MODEL,
                   500_000, 50_000) == 34_883


def test_keyed_uniform_matches_reference(oracle, ref):
    for seed, k in ((0, 0), (1, 2), (0xdeadbeef, 12345), (2**64 - 1, 7)):
        assert oracle.keyed_uniform(seed, k) == ref.keyed_uniform(seed, k)


# --------------------------------------------------------------- fuzz corpora

@pytest.fixture(scope="module")
def corpus():
    return acceptance_corpus(10_000)


@pytest.mark.parametrize("policy", [2, 1, 0])
def test_acceptance_corpus_plans_match_golden(oracle, golden, corpus, policy):
    # acceptance.cpp:125-180 criterion 1, hashed against the reference's plans
    h = hashlib.sha256()
    for v, cfg in corpus:
        c = _abi.SchedulerConfig(policy, cfg.max_chunk, cfg.token_budget, cfg.model)
        plan, e = oracle.form_batch(v, c)
        h.update(plan.tobytes())
        h.update(e.tobytes())
    assert h.hexdigest() == golden["fuzz"][f"acceptance_policy{policy}"]


def test_degenerate_corpus_plans_match_golden(oracle, golden):
    """Zero-token tasks, negative contexts, tiny budgets, c = 0: the
    restatement's `consider` equals the reference's plans (fixture)."""
    from fuzz import degenerate_corpus
    h = hashlib.sha256()
    for v, cfg in degenerate_corpus():
        plan, e = oracle.form_batch(v, cfg)
        h.update(plan.tobytes())
        h.update(e.tobytes())
    assert h.hexdigest() == golden["fuzz"]["degenerate_77001"]


def test_pab_fuzz_matches_golden(oracle, golden):
    rng = Rng(424242)
    vals = []
    for _ in range(1000):
        raw, cfg, now = gen_pab_instance(rng, 8)
        v = raw_to_views(raw, now)
        tt = ms_to_us(rng.uniform(300.0, 2000.0))
        tp = ms_to_us(rng.uniform(25.0, 100.0))
        vals.append(oracle.pab(v, cfg.model, tt, tp))
    assert hashlib.sha256(np.asarray(vals, np.int64).tobytes()).hexdigest() == \
        golden["fuzz"]["pab_424242"]


# --------------------------------------------------------------- traces

@pytest.mark.parametrize("name", sorted(TRACE_PROFILES))
def test_oracle_traces_match_golden(oracle, golden, name):
    prof, h = TRACE_PROFILES[name]
    rows = oracle.generate_bursty(prof, ms_to_us(h))
    g = golden["traces"][name]
    assert len(rows) == g["n"] and rows_digest(rows) == g["sha256"]


def test_c1_trace_shape(oracle):
    prof, h = TRACE_PROFILES["c1_poisson"]
    assert len(oracle.generate_bursty(prof, ms_to_us(h))) == 931


# --------------------------------------------------------------- engine

def _single(prompt, output, arrival_ms=0.0, rid_rows=None):
    return Rows([ms_to_us(arrival_ms)], [prompt], [output], [500_000], [50_000])


ENGINE_MODEL = CostModel(5.0, 0.01, 0.0001)  # test_engine.cpp:19


def _run(cpu, rows, cfg, horizon_ms, log=True):
    b = Batch()
    b.add(rows, cfg, ms_to_us(horizon_ms))
    lo = _abi.LogOpts(1000, 10000, 100, 0) if log else None
    return cpu.run(b, lo)


def test_hand_traced_timeline(cpu):
    # test_engine.cpp:72-92: emits at 6000, 11020, 16040 us
    out = _run(cpu, _single(100, 3), engine_config("fairbatch", 8192, ENGINE_MODEL, 500, 50),
               60_000.0)
    r = out.results[0]
    assert r["steps"] == 3 and r["incomplete"] == 0
    st = out.steps[0][: out.counts[0]["steps"]]
    ends = (st["t_us"] + st["duration_us"]).tolist()
    assert ends == [6000, 11020, 16040]
    rec = out.records[0]
    assert rec["first_emit_us"] == 6000 and rec["tokens_emitted"] == 3
    assert rec["flags"] & _abi.REC_FINISHED


def test_pab_reject_logged(cpu):
    # test_engine.cpp:202-219: empty-node budget 49009 rejects a 60000 prompt
    rows = Rows([0, 0], [60_000, 100], [4, 4], [500_000] * 2, [50_000] * 2)
    out = _run(cpu, rows, engine_config("fairbatch_pab", 8192, ENGINE_MODEL, 500, 50), 60_000.0)
    assert out.counts[0]["rejects"] == 1
    rj = out.rejects[0][0]
    assert rj["req"] == 0 and rj["pab_tokens"] == 49_009
    assert out.records[0]["flags"] & _abi.REC_REJECTED
    assert out.records[0]["tokens_emitted"] == 0
    assert out.records[1]["flags"] & _abi.REC_FINISHED
    assert out.results[0]["incomplete"] == 0


def test_chunk_emission_pattern(cpu):
    # test_engine.cpp:221-243: 600-token prompt in 256-token chunks -> 256, 256, 88
    out = _run(cpu, _single(600, 3),
               engine_config("sarathi", 512, ENGINE_MODEL, 500, 50, max_chunk=256), 60_000.0)
    st = out.steps[0][: out.counts[0]["steps"]]
    assert len(st) == 5
    takes = [int(out.entries[0][s["entry_off"]]["new_tokens"]) for s in st]
    assert takes == [256, 256, 88, 1, 1]


def test_horizon_cut_flags_incomplete(cpu):
    # test_engine.cpp:174-182
    rows = Rows([0] * 32, [20_000] * 32, [50] * 32, [500_000] * 32, [50_000] * 32)
    out = _run(cpu, rows, engine_config("fairbatch", 8192, ENGINE_MODEL, 500, 50), 500.0)
    assert out.results[0]["incomplete"] == 1


def test_empty_trace(cpu):
    # test_engine.cpp:130-134
    out = _run(cpu, Rows.empty(), engine_config("fairbatch", 8192, ENGINE_MODEL, 500, 50), 1000.0)
    assert out.results[0]["steps"] == 0 and out.results[0]["incomplete"] == 0


@pytest.mark.parametrize("name", sorted(SCENARIOS))
def test_oracle_scenarios_match_golden(oracle, golden, name):
    batch = SCENARIOS[name](oracle.generate_bursty)
    out = oracle.run(batch, nthreads=4)
    assert summarize(out.results, out.records) == golden["scenarios"][name]


def test_oracle_equals_reference_with_logs(oracle, ref):
    """Step logs, entries and rejects agree field by field (not just digests)."""
    batch = SCENARIOS["pab_overload"](oracle.generate_bursty)
    lo = _abi.LogOpts(20_000, 400_000, 5_000, 0)
    a = oracle.run(batch, lo, nthreads=4)
    b = ref.run(batch, lo, nthreads=4, check=True)
    assert a.counts.tobytes() == b.counts.tobytes()
    for i in range(batch.n_instances):
        c = a.counts[i]
        assert a.steps[i][: c["steps"]].tobytes() == b.steps[i][: c["steps"]].tobytes()
        assert a.entries[i][: c["entries"]].tobytes() == b.entries[i][: c["entries"]].tobytes()
        assert a.rejects[i][: c["rejects"]].tobytes() == b.rejects[i][: c["rejects"]].tobytes()


# --------------------------------------------------------------- event logs

@pytest.mark.parametrize("name", ["c1", "pab_overload", "wide"])
def test_event_logs_from_plan_logs_match_reference_jsonl(oracle, golden, name):
    """save_event_log JSONL (engine.cpp:395-451) rebuilt from plan logs is
    byte-identical to the reference's own writer (hashes in golden.json)."""
    from paper_2510_14392_b200.events import event_log_jsonl
    batch = SCENARIOS[name](oracle.generate_bursty)
    lo = _abi.LogOpts(40_000, 600_000, 5_000, 0)
    out = oracle.run(batch, lo, nthreads=4)
    got = [hashlib.sha256(event_log_jsonl(batch.rows, batch.instance(i), out.results[i],
                                          out.counts[i], out.steps[i], out.entries[i],
                                          out.rejects[i]).encode()).hexdigest()
           for i in range(batch.n_instances)]
    assert got == golden["event_logs"][name]


@pytest.fixture(scope="module")
def overload_log_lines(oracle):
    from paper_2510_14392_b200.events import event_log_jsonl
    batch = SCENARIOS["pab_overload"](oracle.generate_bursty)
    lo = _abi.LogOpts(40_000, 600_000, 5_000, 0)
    out = oracle.run(batch, lo, nthreads=4)
    return [event_log_jsonl(batch.rows, batch.instance(i), out.results[i], out.counts[i],
                            out.steps[i], out.entries[i], out.rejects[i])
            for i in range(batch.n_instances)]


def test_replay_check_clean_logs(overload_log_lines):
    """Rebuilt event logs satisfy every replay_check invariant."""
    from paper_2510_14392_b200.events import load_event_log, replay_check
    for text in overload_log_lines:
        log = load_event_log(text)
        assert log.events and replay_check(log) == []


@pytest.mark.parametrize("name", ["clean", "drop_first_token", "drop_first_batch_end",
                                  "drop_first_arrival", "dup_arrival", "swap_2_3", "decrease_t",
                                  "bad_token_idx", "reject_after_activity", "truncated_complete",
                                  "done_early", "emit_outside", "unknown_request"])
def test_replay_check_known_answers(golden, overload_log_lines, name):
    """replay_check (engine.cpp:290-393) reports exactly the reference's
    violations, in its order, on mutated copies of a log (golden.json holds
    the reference's own answers on the same mutations)."""
    from paper_2510_14392_b200.events import load_event_log, replay_check
    from tests_golden_cases import REPLAY_MUTATIONS, replay_canonical
    base = overload_log_lines[0].rstrip("\n").split("\n")
    v = replay_canonical(replay_check(load_event_log("\n".join(REPLAY_MUTATIONS[name](base)))))
    g = golden["replay_check"][name]
    assert len(v) == g["n"] and v[:3] == g["head"]
    assert hashlib.sha256("\n".join(v).encode()).hexdigest() == g["sha256"]


def test_load_event_log_errors():
    from paper_2510_14392_b200.events import load_event_log
    from paper_2510_14392_b200.fbgpu import ParseError
    with pytest.raises(ParseError):
        load_event_log('{"t_ms":1.0,"kind":"teleport"}\n')
    with pytest.raises(ParseError):
        load_event_log('{"t_ms":1.0,\n')
    log = load_event_log('\n  \n{"kind":"log_end","node":3,"incomplete":1}\n')
    assert log.events == [] and log.node_id == 3 and log.incomplete


# --------------------------------------------------------------- cluster

@pytest.fixture(scope="module")
def cluster_case_list(oracle):
    from catalog import cluster_cases
    return {c[0]: c for c in cluster_cases(oracle.generate_bursty)}


@pytest.mark.parametrize("name", ["pab0_8", "count0_8", "pab5000_8", "count37_3", "pab_hz10s_8",
                                  "pab20_2", "c5_pab0_64"])
def test_oracle_cluster_matches_golden(oracle, golden, cluster_case_list, name):
    """run_cluster (cluster.cpp:134-251): per-node plan digests, routing
    decisions and per-request records equal the reference's."""
    from backends import cluster_summary
    _, rows, cfgs, lb, hz = cluster_case_list[name]
    assert cluster_summary(oracle.run_cluster(rows, cfgs, lb, hz)) == golden["clusters"][name]


@pytest.fixture(scope="module")
def reroute_case_list(oracle):
    from catalog import reroute_cluster_cases
    return {c[0]: c for c in reroute_cluster_cases(oracle.generate_bursty)}


@pytest.mark.parametrize("name", ["rr_giant_2", "rr_pab0_4", "rr_pab30_3", "rr_count0_4",
                                  "rr_mixed_4", "rr_off_pab0_4"])
def test_oracle_reroute_matches_golden(oracle, golden, reroute_case_list, name):
    """retry_reroute (cluster.cpp:222-237): a first rejection is routed once
    more at the same instant; digests, routing and records equal the reference's."""
    from backends import cluster_summary
    _, rows, cfgs, lb, hz = reroute_case_list[name]
    assert cluster_summary(oracle.run_cluster(rows, cfgs, lb, hz)) == golden["clusters"][name]


def test_oracle_reroute_giant_prompt(oracle, reroute_case_list):
    """test_cluster.cpp:225-250: request 2, rejected behind the giant prompts,
    finishes on the other node; it is routed at most twice."""
    _, rows, cfgs, lb, hz = reroute_case_list["rr_giant_2"]
    out = oracle.run_cluster(rows, cfgs, lb, hz)
    f = int(out.records["flags"][2])
    assert f & _abi.REC_FINISHED and not f & _abi.REC_REJECTED
    assert int(out.node_results["n_arrived"].sum()) <= len(rows) + 1


def test_route_known_answers(oracle):
    """test_cluster.cpp:76-113 through a 2-node cluster's first decisions:
    pab_lb prefers the roomiest node that fits, ties go to the lowest id."""
    from paper_2510_14392_b200.cluster import LbConfig
    rows = Rows([0, 0, 0], [800, 100, 50_000], [4, 4, 4], [500_000] * 3, [50_000] * 3)
    cfgs = [engine_config("fairbatch_pab", 8192, ENGINE_MODEL, 500, 50) for _ in range(2)]
    out = oracle.run_cluster(rows, cfgs, LbConfig("pab_lb", 1, 0.0), ms_to_us(60_000.0))
    # empty nodes report 49009 each: request 0 -> node 0 (tie, lowest id),
    # request 1 -> node 1 (node 0 decremented by 800), request 2 fits nowhere ->
    # best effort to the roomiest (node 0: 48209 vs node 1: 48909) -> node 1
    assert out.route_node.tolist() == [0, 1, 1]
