"""The C++ host API (paper_2510_14392_b200/host/fbsim_gpu.h): the reference's
fbsim interfaces over the C ABI.  Driven through its test program
(host/test_fbsim_gpu.cpp): host-only checks and loud failure without a GPU on
CPU; the reference's known answers and byte-identical event logs on the GPU."""
from __future__ import annotations

import hashlib
import os
import subprocess

import pytest

from catalog import SCENARIOS
from paper_2510_14392_b200.batch import Batch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2510_14392_b200", "host", "test_fbsim_gpu")


def _run(*args, timeout=600):
    if not os.path.exists(BIN):
        pytest.fail("host/test_fbsim_gpu not built (run __graft_entry__.build())")
    return subprocess.run([BIN, *args], capture_output=True, text=True, timeout=timeout)


def _gpu_present() -> bool:
    import torch
    return torch.cuda.is_available()


def test_host_api_without_gpu():
    """Trace generation and the JSONL writer work on the host; every device
    entry point throws CudaError (no CPU fallback)."""
    if _gpu_present():
        pytest.skip("a GPU is present: the no-device contract is checked on CPU hosts")
    p = _run("nogpu")
    assert p.returncode == 0, p.stderr


@pytest.mark.gpu
def test_host_api_known_answers():
    """test_sched.cpp / test_engine.cpp / test_cluster.cpp known answers through
    the C++ API: init budgets, plans, PAB 49009/44883/34883, the 6000 / 11020 /
    16040 us timeline, the 49009 reject, chunking, routing, reroute."""
    p = _run("kat")
    assert p.returncode == 0, p.stdout + p.stderr


def _instance_file(path, batch: Batch, i: int):
    inst = batch.instance(i)
    c = inst.cfg
    s = c.scheduler
    off, n = int(inst.trace_off), int(inst.n_req)
    r = batch.rows
    with open(path, "w") as f:
        f.write(f"{inst.horizon_us} {s.policy} {s.token_budget} {s.max_chunk} "
                f"{s.model.a_ms!r} {s.model.b_ms!r} {s.model.c_ms!r} "
                f"{c.truth_model.a_ms!r} {c.truth_model.b_ms!r} {c.truth_model.c_ms!r} "
                f"{c.noise_amplitude!r} {c.noise_seed} {c.global_ttft_us} {c.global_tpot_us} "
                f"{c.max_active}\n{n}\n")
        for k in range(off, off + n):
            f.write(f"{r.arrival_us[k]} {r.prompt_len[k]} {r.output_len[k]} {r.ttft_us[k]} "
                    f"{r.tpot_us[k]}\n")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["pab_overload", "c1"])
def test_host_api_event_logs_match_reference(golden, tmp_path, fb, name):
    """run_node on the single-instance path and run_nodes batched, each log
    written with save_event_log through the C++ API: byte-identical to the
    reference's own writer (sha256 per instance, golden.json)."""
    batch = SCENARIOS[name](fb.generate_bursty)
    src = tmp_path / "in0.txt"  # run_node on instance 0 (one process)
    _instance_file(src, batch, 0)
    p = _run("eventlog", str(src), str(tmp_path / "single.jsonl"))
    assert p.returncode == 0, p.stderr
    assert hashlib.sha256((tmp_path / "single.jsonl").read_bytes()).hexdigest() == \
        golden["event_logs"][name][0]
    hz = {int(batch.instance(i).horizon_us) for i in range(batch.n_instances)}
    groups = {h: [i for i in range(batch.n_instances) if int(batch.instance(i).horizon_us) == h]
              for h in hz}
    r = batch.rows
    for h, idx in groups.items():  # run_nodes per horizon group
        src = tmp_path / f"batch{h}.txt"
        with open(src, "w") as f:
            f.write(f"{len(idx)}\n")
            for i in idx:
                inst = batch.instance(i)
                off, n = int(inst.trace_off), int(inst.n_req)
                f.write(f"{inst.horizon_us}\n" + _cfg_line(inst.cfg) + f"{n}\n")
                for k in range(off, off + n):
                    f.write(f"{r.arrival_us[k]} {r.prompt_len[k]} {r.output_len[k]} "
                            f"{r.ttft_us[k]} {r.tpot_us[k]}\n")
        out = tmp_path / f"logs{h}"
        out.mkdir()
        p = _run("eventlogs", str(src), str(out))
        assert p.returncode == 0, p.stderr
        for j, i in enumerate(idx):
            got = hashlib.sha256((out / f"out{j}.jsonl").read_bytes()).hexdigest()
            assert got == golden["event_logs"][name][i], (name, i)


def _cfg_line(c):
    s = c.scheduler
    return (f"{s.policy} {s.token_budget} {s.max_chunk} {s.model.a_ms!r} {s.model.b_ms!r} "
            f"{s.model.c_ms!r} {c.truth_model.a_ms!r} {c.truth_model.b_ms!r} "
            f"{c.truth_model.c_ms!r} {c.noise_amplitude!r} {c.noise_seed} {c.global_ttft_us} "
            f"{c.global_tpot_us} {c.max_active}\n")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["pab0_8", "count37_3", "pab5000_8", "rr_giant_2", "rr_pab30_3"])
def test_host_api_cluster_logs_match_reference(golden, tmp_path, fb, name):
    """run_cluster through the C++ API: every node's EventLog and the routing
    log (view snapshots included), byte-identical to the reference's files --
    with retry_reroute too."""
    from catalog import cluster_cases, reroute_cluster_cases
    from paper_2510_14392_b200.cluster import node_configs_c
    cases = {c[0]: c for c in cluster_cases(fb.generate_bursty) +
             reroute_cluster_cases(fb.generate_bursty)}
    _, rows, cfgs, lb, hz = cases[name]
    lbc = lb.to_c()
    nc = node_configs_c(cfgs)
    src = tmp_path / "cluster.txt"
    with open(src, "w") as f:
        f.write(f"{len(cfgs)} {hz} {lbc.policy} {lbc.report_interval_steps} "
                f"{lbc.report_latency_us} {lbc.w_waiting!r} {lbc.w_running!r} "
                f"{lbc.retry_reroute}\n")
        for i in range(len(cfgs)):
            f.write(_cfg_line(nc[i]))
        f.write(f"{len(rows)}\n")
        for k in range(len(rows)):
            f.write(f"{rows.arrival_us[k]} {rows.prompt_len[k]} {rows.output_len[k]} "
                    f"{rows.ttft_us[k]} {rows.tpot_us[k]}\n")
    p = _run("clusterlogs", str(src), str(tmp_path))
    assert p.returncode == 0, p.stderr
    g = golden["cluster_logs"][name]
    assert hashlib.sha256((tmp_path / "routing.jsonl").read_bytes()).hexdigest() == g["routing"]
    got = [hashlib.sha256((tmp_path / f"node{i}.jsonl").read_bytes()).hexdigest()
           for i in range(len(cfgs))]
    assert got == g["nodes"]


def _scenario(nodes: int, policy: str) -> dict:
    return {
        "name": f"cpp_{policy}_{nodes}",
        "trace": {"bursty": {"base_rate": 2.0 * nodes, "burst_rate": 8.0 * nodes,
                             "burst_duration_ms": 1000, "idle_duration_ms": 2000,
                             "prompt_mean": 892, "prompt_p90": 1776, "output_mean": 120,
                             "output_p90": 260, "seed": 7, "horizon_ms": 20000},
                  "scale": 1.5},
        "slo": {"ttft_ms": 500, "tpot_ms": 50},
        "scheduler": {"policy": policy, "token_budget": 2048},
        "cost_model": {"truth": {"a_ms": 5.0, "b_ms_per_token": 0.05,
                                 "c_ms_per_context_token": 0.0001},
                       "noise_amplitude": 0.03},
        "cluster": {"nodes": nodes, "policy": "pab_lb"},
        "run": {"horizon_ms": 3600000, "seed": 42},
    }


def test_host_scenario_config_errors(tmp_path):
    """Schema violations are ConfigError (exit 1) before any device work --
    unknown keys, missing sections, bad policies (scenario.cpp:77-222)."""
    import json
    bad = _scenario(1, "fairbatch")
    bad["run"]["horizon"] = 5
    for j in (bad, {k: v for k, v in _scenario(1, "fairbatch").items() if k != "slo"},
              dict(_scenario(1, "fairbatch"), scheduler={"policy": "fifo"})):
        f = tmp_path / "bad.json"
        f.write_text(json.dumps(j))
        p = _run("scenario", str(f))
        assert p.returncode == 1 and "config error" in p.stderr, (p.returncode, p.stderr)


@pytest.mark.gpu
@pytest.mark.parametrize("nodes,policy", [(1, "fairbatch"), (1, "fairbatch_pab"), (4, "fairbatch_pab")])
def test_host_scenario_matches_python(tmp_path, fb, nodes, policy):
    """load_scenario + run_scenario through the C++ API report exactly what
    the Python driver (pinned against the reference's acceptance criteria)
    reports for the same scenario file."""
    import json
    from paper_2510_14392_b200.scenario import load_scenario, run_scenario
    f = tmp_path / "sc.json"
    f.write_text(json.dumps(_scenario(nodes, policy)))
    p = _run("scenario", str(f))
    assert p.returncode == 0, p.stderr
    got = json.loads(p.stdout.strip().splitlines()[-1])
    rep = run_scenario(load_scenario(str(f)))
    assert got["total"] == rep.total_requests and got["good"] == rep.good
    assert got["rejected"] == rep.rejected and got["finished"] == rep.finished
    assert got["offered"] == rep.offered_rps and got["effective"] == rep.effective_rps
    assert got["ttft"] == [rep.ttft.p50, rep.ttft.p95, rep.ttft.p99, rep.ttft.count]
    assert got["tpot"] == [rep.max_tpot.p50, rep.max_tpot.p95, rep.max_tpot.p99,
                           rep.max_tpot.count]


@pytest.mark.gpu
def test_host_node_batch_matches_arena(tmp_path, fb):
    """NodeBatch (the C++ step machine over many nodes) on C2 instances: every
    instance's step count, plan digest and reject count equal the Python
    arena's (which the oracle and golden fixtures pin)."""
    from paper_2510_14392_b200 import workloads
    batch = workloads.c2_batch(n_seeds=24, seed0=300)
    hz = {int(batch.instance(i).horizon_us) for i in range(batch.n_instances)}
    assert len(hz) == 1
    src = tmp_path / "batch.txt"
    r = batch.rows
    with open(src, "w") as f:
        f.write(f"{batch.n_instances}\n")
        for i in range(batch.n_instances):
            inst = batch.instance(i)
            off, n = int(inst.trace_off), int(inst.n_req)
            f.write(f"{inst.horizon_us}\n" + _cfg_line(inst.cfg) + f"{n}\n")
            for k in range(off, off + n):
                f.write(f"{r.arrival_us[k]} {r.prompt_len[k]} {r.output_len[k]} {r.ttft_us[k]} "
                        f"{r.tpot_us[k]}\n")
    p = _run("batch", str(src))
    assert p.returncode == 0, p.stderr
    got = [ln.split() for ln in p.stdout.strip().splitlines()]
    a = fb.Arena(0)
    a.load(batch)
    a.run()
    res = a.results()
    a.close()
    want = [[str(int(x["steps"])), "%016x" % int(x["plan_digest"]), str(int(x["n_rejected"]))]
            for x in res]
    assert got == want
