"""GPU parity suite: the CUDA path (through the C ABI) against the golden
fixtures of the unmodified reference and against the C oracle, bit-exact.

Batch composition (request rows, chunk sizes, predicted/actual step times) is
compared through the per-instance plan digest and, where logged, entry by
entry; per-request records (TTFT, TPOT, flags) byte for byte.
"""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

import test_oracle_cpu as kat
from backends import RunOutput
from catalog import SCENARIOS, summarize
from fuzz import Rng, acceptance_corpus, gen_pab_instance, raw_to_views
from paper_2510_14392_b200 import _abi, workloads
from paper_2510_14392_b200.batch import Batch, ms_to_us

pytestmark = pytest.mark.gpu


class GpuLib:
    """Single-set adapter over the batched device API, same shape as the CPU libs."""

    def __init__(self, fb):
        self.fb = fb

    def generate_bursty(self, prof, horizon_us):
        return self.fb.generate_bursty(prof, horizon_us)

    def init_time_budget(self, tasks):
        try:
            return int(self.fb.init_time_budget([tasks])[0])
        except self.fb.FbError as e:
            raise RuntimeError(str(e)) from e

    def form_batch(self, tasks, cfg):
        plans, entries = self.fb.form_batch([tasks], [cfg])
        p = plans[0].copy()
        p["entry_off"] = 0
        return p, entries[0]

    def pab(self, tasks, model, ttft_us, tpot_us):
        return int(self.fb.pab([tasks], [model], ttft_us, tpot_us)[0])

    def run(self, batch, log=None, nthreads=None, max_events=0):
        a = self.fb.Arena(0)
        a.load(batch, log)
        if max_events > 0:
            while a.run(max_events, sync=True) > 0:
                pass
        else:
            a.run()
        res, rec = a.results(), a.records()
        counts = steps = entries = rejects = None
        if log is not None:
            counts, steps, entries, rejects = a.logs()
        a.close()
        return RunOutput(res, rec, counts, steps, entries, rejects)


@pytest.fixture(scope="module")
def gpu(fb):
    return GpuLib(fb)


# ------------------------------------------------------------ known answers

@pytest.mark.parametrize("case", [
    "test_init_time_budget_known_answers", "test_single_urgent_decode",
    "test_prefill_chunked_ahead_of_relaxed_decode", "test_order_tie_break_and_empty",
    "test_sarathi_and_prefill_first", "test_pab_known_answers", "test_hand_traced_timeline",
    "test_pab_reject_logged", "test_chunk_emission_pattern", "test_horizon_cut_flags_incomplete",
    "test_empty_trace"])
def test_reference_known_answers_on_gpu(gpu, case):
    getattr(kat, case)(gpu)


# ------------------------------------------------------------ pure scheduler fuzz

@pytest.mark.parametrize("policy", [2, 1, 0])
def test_form_batch_acceptance_corpus(fb, golden, policy):
    """acceptance.cpp criterion 1 corpus (seed 20260808, 10^4 sets) in one launch."""
    corpus = acceptance_corpus(10_000)
    sets = [v for v, _ in corpus]
    cfgs = [_abi.SchedulerConfig(policy, c.max_chunk, c.token_budget, c.model) for _, c in corpus]
    plans, entries = fb.form_batch(sets, cfgs)
    h = hashlib.sha256()
    for p, e in zip(plans, entries):
        p = p.copy()
        p["entry_off"] = 0
        h.update(p.tobytes())
        h.update(e.tobytes())
    assert h.hexdigest() == golden["fuzz"][f"acceptance_policy{policy}"]


def test_form_batch_degenerate_corpus(fb, golden, oracle):
    """The pure scheduler boundary on sets the engines never produce:
    zero-token tasks (admitted as {id, 0} by fair batching even at token
    budget 0), negative contexts, tiny budgets, c = 0 -- plan for plan equal
    to the reference's form_batch (fixture) and to the oracle."""
    from fuzz import degenerate_corpus
    corpus = degenerate_corpus()
    plans, entries = fb.form_batch([v for v, _ in corpus], [c for _, c in corpus])
    h = hashlib.sha256()
    zero = 0
    for (v, c), p, e in zip(corpus, plans, entries):
        p = p.copy()
        p["entry_off"] = 0
        h.update(p.tobytes())
        h.update(e.tobytes())
        zero += int((e["new_tokens"] == 0).any())
    assert zero > 1000
    if h.hexdigest() != golden["fuzz"]["degenerate_77001"]:
        for (v, c), p, e in zip(corpus, plans, entries):
            op, oe = oracle.form_batch(v, c)
            p = p.copy()
            p["entry_off"] = 0
            assert p.tobytes() == op.tobytes() and e.tobytes() == oe.tobytes(), (v, c.policy)
        pytest.fail("degenerate corpus differs from the reference fixture")


def test_form_batch_large_sets_match_oracle(fb, oracle):
    """Sets beyond the shared-memory scratch (global scratch path)."""
    rng = Rng(99)
    from fuzz import gen_instance
    sets, cfgs = [], []
    for i in range(60):
        raw, cfg, now = gen_instance(rng, 400)
        cfg.policy = i % 3
        sets.append(raw_to_views(raw, now))
        cfgs.append(cfg)
    plans, entries = fb.form_batch(sets, cfgs)
    assert max(len(s) for s in sets) > 64
    for s, c, p, e in zip(sets, cfgs, plans, entries):
        op, oe = oracle.form_batch(s, c)
        p = p.copy()
        p["entry_off"] = 0
        assert p.tobytes() == op.tobytes() and e.tobytes() == oe.tobytes()


def test_pab_fuzz(fb, golden):
    rng = Rng(424242)
    sets, models, tt, tp = [], [], [], []
    for _ in range(1000):
        raw, cfg, now = gen_pab_instance(rng, 8)
        sets.append(raw_to_views(raw, now))
        models.append(cfg.model)
        tt.append(ms_to_us(rng.uniform(300.0, 2000.0)))
        tp.append(ms_to_us(rng.uniform(25.0, 100.0)))
    vals = fb.pab(sets, models, tt, tp)
    assert hashlib.sha256(np.asarray(vals, np.int64).tobytes()).hexdigest() == \
        golden["fuzz"]["pab_424242"]


def test_empty_fair_set_is_usage_error(fb):
    with pytest.raises(fb.UsageError):
        fb.form_batch([np.zeros(0, _abi.TASKVIEW_DTYPE)],
                      [_abi.SchedulerConfig(2, 2048, 2048, _abi.CostModel(5, 0.05, 1e-4))])


# ------------------------------------------------------------ engine vs fixtures

@pytest.mark.parametrize("name", sorted(SCENARIOS))
def test_engine_scenarios_match_golden(gpu, golden, name):
    batch = SCENARIOS[name](gpu.generate_bursty)
    out = gpu.run(batch)
    assert summarize(out.results, out.records) == golden["scenarios"][name]


@pytest.mark.parametrize("name", ["c1", "pab_overload", "large_live", "mixed", "wide"])
def test_engine_logs_match_oracle(gpu, oracle, name):
    """Every step: time, duration, predicted/actual ms, totals and each plan
    entry (request row, new tokens) in admission order; every PAB reject."""
    batch = SCENARIOS[name](oracle.generate_bursty)
    lo = _abi.LogOpts(40_000, 600_000, 5_000, 0)
    a = gpu.run(batch, lo)
    b = oracle.run(batch, lo, nthreads=4)
    assert a.counts.tobytes() == b.counts.tobytes()
    assert not a.counts["truncated"].any()
    for i in range(batch.n_instances):
        c = a.counts[i]
        assert a.steps[i][: c["steps"]].tobytes() == b.steps[i][: c["steps"]].tobytes(), i
        assert a.entries[i][: c["entries"]].tobytes() == b.entries[i][: c["entries"]].tobytes(), i
        assert a.rejects[i][: c["rejects"]].tobytes() == b.rejects[i][: c["rejects"]].tobytes(), i
    assert a.results.tobytes() == b.results.tobytes()
    assert a.records.tobytes() == b.records.tobytes()


@pytest.mark.parametrize("name,want", [("c2_subset", 1), ("large_live", 2), ("wide", 4),
                                       ("c2_subset", 8), ("large_live", 16)])
def test_engine_paths_exercised(fb, gpu, name, want):
    """The scenarios really drive the register, memory and CTA-wide paths,
    and the repeated-plan steps of the register and memory paths."""
    batch = SCENARIOS[name](gpu.generate_bursty)
    a = fb.Arena(0)
    a.load(batch)
    a.run()
    paths = a.paths()
    a.close()
    assert (paths & want).any(), paths


@pytest.mark.parametrize("name", ["c1", "pab_overload", "wide"])
def test_gpu_event_logs_match_reference_jsonl(gpu, golden, name):
    """The reference's JSONL event log (save_event_log) rebuilt from the
    device plan logs, byte for byte (sha256 per instance)."""
    from paper_2510_14392_b200.events import event_log_jsonl
    batch = SCENARIOS[name](gpu.generate_bursty)
    lo = _abi.LogOpts(40_000, 600_000, 5_000, 0)
    out = gpu.run(batch, lo)
    got = [hashlib.sha256(event_log_jsonl(batch.rows, batch.instance(i), out.results[i],
                                          out.counts[i], out.steps[i], out.entries[i],
                                          out.rejects[i]).encode()).hexdigest()
           for i in range(batch.n_instances)]
    assert got == golden["event_logs"][name]


@pytest.mark.parametrize("name", ["pab_overload", "wide"])
def test_gpu_event_logs_pass_replay_check(gpu, name):
    """replay_check (engine.cpp:290-393) on the device-built event logs:
    no violation in any instance."""
    from paper_2510_14392_b200.events import event_log_jsonl, load_event_log, replay_check
    batch = SCENARIOS[name](gpu.generate_bursty)
    lo = _abi.LogOpts(40_000, 600_000, 5_000, 0)
    out = gpu.run(batch, lo)
    for i in range(batch.n_instances):
        log = load_event_log(event_log_jsonl(batch.rows, batch.instance(i), out.results[i],
                                             out.counts[i], out.steps[i], out.entries[i],
                                             out.rejects[i]))
        assert log.events and replay_check(log) == [], i


def test_stepwise_api_matches_one_shot(gpu):
    """Node-style incremental driving (fb_arena_run with an event budget)."""
    batch = SCENARIOS["mixed"](gpu.generate_bursty)
    one = gpu.run(batch)
    inc = gpu.run(batch, max_events=97)
    assert summarize(one.results, one.records) == summarize(inc.results, inc.records)


def test_run_batch_e2e_equals_arena(fb, gpu):
    batch = SCENARIOS["c2_subset"](gpu.generate_bursty)
    res, rec, ms = fb.run_batch(batch)
    out = gpu.run(batch)
    assert res.tobytes() == out.results.tobytes() and rec.tobytes() == out.records.tobytes()
    assert ms > 0


def test_arena_reset_reruns_identically(fb):
    batch = workloads.c2_batch(n_seeds=64)
    a = fb.Arena(0)
    a.load(batch)
    a.run()
    r1, c1 = a.results().copy(), a.records().copy()
    a.reset()
    a.run()
    assert a.results().tobytes() == r1.tobytes() and a.records().tobytes() == c1.tobytes()
    a.close()


def test_validation_errors(fb):
    b = Batch()
    from paper_2510_14392_b200.batch import CostModel, Rows, engine_config
    rows = Rows([0], [0], [5], [500_000], [50_000])  # prompt_len 0
    b.add(rows, engine_config("fairbatch", 2048, CostModel(5, 0.05, 1e-4), 500, 50), 10**9)
    a = fb.Arena(0)
    with pytest.raises(fb.ValidationError):
        a.load(b)
    b2 = Batch()
    b2.add(Rows([0], [10], [5], [500_000], [50_000]),
           engine_config("fairbatch", 100, CostModel(5, 0.05, 1e-4), 500, 50, max_chunk=200),
           10**9)
    with pytest.raises(fb.ValidationError):
        a.load(b2)
    a.close()


# ------------------------------------------------------------ C2 at scale

def test_c2_sample_matches_oracle(gpu, oracle):
    """512 C2 instances: per-instance digest and records identical to the oracle."""
    batch = workloads.c2_batch(n_seeds=256, seed0=1000)
    a = gpu.run(batch)
    b = oracle.run(batch, nthreads=8)
    assert a.results.tobytes() == b.results.tobytes()
    assert a.records.tobytes() == b.records.tobytes()


def test_c2_full_size_properties(fb):
    """The bench workload (4096 instances): every instance quiescent, record
    invariants hold, and a rerun is bit-identical (determinism)."""
    batch = workloads.c2_batch()
    a = fb.Arena(0)
    a.load(batch)
    a.run()
    res = a.results()
    rec = a.records()
    assert (res["status"] == 0).all() and (res["incomplete"] == 0).all()
    assert int(res["steps"].sum()) > 10_000_000
    assert (rec["flags"] & _abi.REC_ARRIVED).all()
    fin = (rec["flags"] & _abi.REC_FINISHED) != 0
    assert fin.all()
    a.reset()
    a.run()
    assert a.results().tobytes() == res.tobytes()
    a.close()


# ------------------------------------------------------------ cluster (C5)

@pytest.fixture(scope="module")
def gpu_cluster_cases(fb):
    from catalog import cluster_cases
    return {c[0]: c for c in cluster_cases(fb.generate_bursty)}


@pytest.mark.parametrize("name", ["pab0_8", "count0_8", "pab5000_8", "count37_3", "pab_hz10s_8",
                                  "pab20_2", "c5_pab0_64"])
def test_cluster_matches_golden(golden, gpu_cluster_cases, name):
    """fb_run_cluster: per-node plan digests, routing decisions and records
    equal the reference run_cluster's (cluster.cpp:134-251)."""
    from backends import cluster_summary
    from paper_2510_14392_b200.cluster import run_cluster
    _, rows, cfgs, lb, hz = gpu_cluster_cases[name]
    out = run_cluster(rows, cfgs, lb, hz)
    assert cluster_summary(out) == golden["clusters"][name]


@pytest.fixture(scope="module")
def gpu_reroute_cases(fb):
    from catalog import reroute_cluster_cases
    return {c[0]: c for c in reroute_cluster_cases(fb.generate_bursty)}


@pytest.mark.parametrize("name", ["rr_giant_2", "rr_pab0_4", "rr_pab30_3", "rr_count0_4",
                                  "rr_mixed_4", "rr_off_pab0_4"])
def test_cluster_reroute_matches_golden(golden, gpu_reroute_cases, name):
    """retry_reroute (cluster.cpp:222-237) on the serial cluster engine:
    digests, routing (last target) and merged records equal the reference's."""
    from backends import cluster_summary
    from paper_2510_14392_b200.cluster import run_cluster
    _, rows, cfgs, lb, hz = gpu_reroute_cases[name]
    out = run_cluster(rows, cfgs, lb, hz)
    assert cluster_summary(out) == golden["clusters"][name]


def test_clusters_side_by_side_match_golden(golden, gpu_cluster_cases, gpu_reroute_cases):
    """run_clusters: concurrent shards (epoch-decomposed and serial reroute
    engines mixed) give each case's golden run_cluster output."""
    from backends import cluster_summary
    from paper_2510_14392_b200.cluster import run_clusters
    names = ["pab0_8", "count37_3", "rr_giant_2", "pab5000_8", "rr_pab30_3", "count0_8"]
    cases = [(gpu_cluster_cases.get(n) or gpu_reroute_cases[n])[1:] for n in names]
    outs = run_clusters(cases)
    for n, out in zip(names, outs):
        assert cluster_summary(out) == golden["clusters"][n], n


def test_clusters_cooperative_fallback_match_golden(fb, golden, gpu_cluster_cases, monkeypatch):
    """The cooperative-grid path (global-memory epoch barrier) that runs when
    a one-cluster launch is not possible (forced with FB_NO_HW_CLUSTER), and
    the two-CTAs-per-SM cluster kernel run_clusters takes for more replicas
    than fit at one CTA per SM."""
    import ctypes as C
    from backends import cluster_summary
    from paper_2510_14392_b200.cluster import cluster_density, cluster_fit, run_cluster, run_clusters
    assert run_clusters([]) == []
    monkeypatch.setenv("FB_NO_HW_CLUSTER", "1")
    for n in ("c5_pab0_64", "pab5000_8", "count37_3"):
        _, rows, cfgs, lb, hz = gpu_cluster_cases[n]
        assert cluster_summary(run_cluster(rows, cfgs, lb, hz)) == golden["clusters"][n], n
    monkeypatch.delenv("FB_NO_HW_CLUSTER")
    fit = C.c_int32(0)
    fb._check(fb.lib().fb_cluster_max_hw_clusters(0, 64, C.byref(fit)), "max_hw_clusters")
    assert 1 <= fit.value <= 64
    fit1, fit2 = cluster_fit(64, 1), cluster_fit(64, 2)
    assert fit1 == fit.value and fit2 >= fit1
    case = gpu_cluster_cases["c5_pab0_64"][1:]
    # one copy more than fit at one CTA per SM: every copy at two per SM
    assert cluster_density(fit1 + 1, 64) == (2 if fit1 + 1 <= fit2 else 0)
    outs = run_clusters([case] * (fit1 + 1))
    assert len(outs) == fit1 + 1
    for out in outs:
        assert cluster_summary(out) == golden["clusters"]["c5_pab0_64"]


@pytest.mark.parametrize("name", ["pab0_8", "count37_3", "pab5000_8", "pab_hz10s_8", "pab20_2",
                                  "rr_giant_2", "rr_pab30_3", "rr_mixed_4"])
def test_cluster_logs_match_reference(golden, gpu_cluster_cases, gpu_reroute_cases, name):
    """ClusterResult's logs from the device run: every node's EventLog
    (save_event_log) and the routing log with view snapshots
    (save_routing_log), byte-identical to the reference's files."""
    from paper_2510_14392_b200.cluster import run_cluster_logged
    from paper_2510_14392_b200.events import cluster_event_logs
    _, rows, cfgs, lb, hz = (gpu_cluster_cases.get(name) or gpu_reroute_cases[name])
    logs = run_cluster_logged(rows, cfgs, lb, hz)
    g = golden["cluster_logs"][name]
    nodes, routing = cluster_event_logs(rows, logs, lb.policy)
    assert hashlib.sha256(routing.encode()).hexdigest() == g["routing"]
    assert [hashlib.sha256(x.encode()).hexdigest() for x in nodes] == g["nodes"]


def test_cluster_reroute_is_single_rank(fb):
    """The reroute engine replays the global loop on one GPU: a multi-rank
    shard with retry_reroute is a usage error, not a silent divergence."""
    from paper_2510_14392_b200.cluster import ClusterShard, LbConfig
    from paper_2510_14392_b200.batch import CostModel, Rows, engine_config
    rows = Rows([0, 0], [10, 10], [5, 5], [500_000] * 2, [50_000] * 2)
    cfgs = [engine_config("fairbatch_pab", 2048, CostModel(5, 0.05, 1e-4), 500, 50)] * 2
    with pytest.raises(fb.UsageError):
        ClusterShard(rows, cfgs, LbConfig("pab_lb", 1, 0.0, retry_reroute=True), 10**9, 0, 2)


@pytest.mark.parametrize("name,world", [("pab0_8", 2), ("count37_3", 3), ("pab5000_8", 4),
                                        ("pab_hz10s_8", 2), ("c5_pab0_64", 8)])
def test_cluster_shards_in_process_match_golden(golden, gpu_cluster_cases, name, world):
    """The multi-rank protocol on one device: `world` shards (one persistent
    kernel each, on its own stream, running concurrently) exchange their
    node reports through each other's exchange buffers; the merged output
    equals run_cluster's golden summary."""
    from backends import cluster_summary
    from paper_2510_14392_b200.cluster import ClusterShard, merge_shards
    _, rows, cfgs, lb, hz = gpu_cluster_cases[name]
    shards = [ClusterShard(rows, cfgs, lb, hz, r, world, 0) for r in range(world)]
    try:
        ptrs = [s.exchange_ptr() for s in shards]
        for s in shards:
            s.connect_ptrs(ptrs)
        for s in shards:
            s.reset()
        for s in shards:
            s.launch()
        parts = [s.fetch(s.wait()) for s in shards]
    finally:
        for s in shards:
            s.close()
    out = merge_shards(parts, len(cfgs))
    assert cluster_summary(out) == golden["clusters"][name]


def _ipc_worker(rank, world, port, q, name):
    import os
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch.distributed as dist
    from backends import cluster_summary
    from catalog import cluster_cases
    from paper_2510_14392_b200 import fbgpu
    from paper_2510_14392_b200.cluster import run_cluster_dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    case = {c[0]: c for c in cluster_cases(fbgpu.generate_bursty)}[name]
    _, rows, cfgs, lb, hz = case
    rows = rows.truncated(120)  # processes time-slice one GPU: keep the epochs few
    out = run_cluster_dist(rows, cfgs, lb, hz, dist, device=0)
    if rank == 0:
        q.put(cluster_summary(out))
    dist.barrier()
    dist.destroy_process_group()


def test_cluster_two_processes_cuda_ipc(fb, oracle):
    """run_cluster_dist across two processes: exchange buffers opened with
    CUDA IPC (the multi-GPU path; here both processes share one device)."""
    import socket
    import torch.multiprocessing as mp
    from backends import cluster_summary
    from catalog import cluster_cases
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    name = "count37_3"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q, name)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, rows, cfgs, lb, hz = {c[0]: c for c in cluster_cases(oracle.generate_bursty)}[name]
    ref = oracle.run_cluster(rows.truncated(120), cfgs, lb, hz)
    assert got == cluster_summary(ref)


# ------------------------------------------------------- device aggregates


@pytest.mark.parametrize("name", sorted(SCENARIOS))
def test_device_summaries_match_host_reports(fb, gpu, name):
    """fb_arena_fetch_summaries (on-device scenario_report, metrics.cpp:171-205)
    equals the host aggregation of the byte-identical records, field for
    field: counts, and nearest-rank p50/p95/p99 as exact doubles (the wide
    scenario has > 2048 values per series: the radix-select path)."""
    from paper_2510_14392_b200 import reports
    batch = SCENARIOS[name](gpu.generate_bursty)
    a = fb.Arena(0)
    a.load(batch)
    a.run()
    summ = a.summaries()
    rec = a.records()
    a.close()
    off = batch.record_offsets()
    rows = batch.rows
    for i in range(batch.n_instances):
        x = batch.instance(i)
        r = rec[off[i]:off[i + 1]]
        arr = rows.arrival_us[x.trace_off:x.trace_off + x.n_req]
        host = reports.scenario_report(r, arr, 1.0, alt_tpot=True)
        dev = reports.summary_report(summ[i], 1.0, alt_tpot=True)
        assert dev == host, (name, i)


# ------------------------------------------------------- edge cases / API paths


def test_stepwise_wide_engine_matches_one_shot(gpu):
    """Event-budgeted driving of escalated (> 512 live) nodes: the grid-wide
    engine releases a node mid-run and picks it up in the next launch, with
    its view records, marks and takes persisting across launches."""
    batch = SCENARIOS["wide"](gpu.generate_bursty)
    one = gpu.run(batch)
    for budget in (13, 64):
        inc = gpu.run(batch, max_events=budget)
        assert summarize(one.results, one.records) == summarize(inc.results, inc.records), budget


def test_summaries_mid_run_do_not_perturb(fb, gpu):
    """fb_arena_fetch_summaries between event-budgeted runs (its scratch is
    separate from the engines' persistent state)."""
    batch = SCENARIOS["wide"](gpu.generate_bursty)
    ref = gpu.run(batch)
    a = fb.Arena(0)
    a.load(batch)
    while a.run(29, sync=True) > 0:
        a.summaries()
    assert a.results().tobytes() == ref.results.tobytes()
    assert a.records().tobytes() == ref.records.tobytes()
    a.close()


def test_empty_and_degenerate_batches(fb, oracle):
    """No instances; instances with zero requests next to normal and wide ones;
    a horizon of zero (no step may begin)."""
    from paper_2510_14392_b200.batch import CostModel, Rows, engine_config
    a = fb.Arena(0)
    a.load(Batch())
    a.run()
    assert len(a.results()) == 0 and len(a.records()) == 0 and len(a.summaries()) == 0
    cfg = engine_config("fairbatch", 2048, CostModel(5, 0.05, 1e-4), 500, 50)
    b = Batch()
    b.add(Rows.empty(), cfg, 10**9)
    b.extend(SCENARIOS["c2_subset"](fb.generate_bursty).subset([0, 1]))
    b.add(Rows([0, 10], [64, 64], [4, 4], [500_000] * 2, [50_000] * 2), cfg, 0)
    b.add(Rows.empty(), cfg, 0)
    a.load(b)
    a.run()
    got_r, got_c = a.results(), a.records()
    want = oracle.run(b)
    assert got_r.tobytes() == want.results.tobytes()
    assert got_c.tobytes() == want.records.tobytes()
    s = a.summaries()
    assert s[0]["total_requests"] == 0 and s[0]["ttft_ms"]["count"] == 0
    a.close()


def test_pinned_buffers_match_pageable(fb):
    """Uploads from fb_host_alloc memory and records into a pinned buffer
    (direct DMA) equal the staged pageable path byte for byte."""
    batch = workloads.c2_batch(n_seeds=32)
    a = fb.Arena(0)
    a.load(batch)
    a.run()
    r1, c1 = a.results().copy(), a.records().copy()
    batch.pin()
    out = fb.pinned_empty(a.record_rows(), _abi.RECORD_DTYPE)
    a.load(batch)
    a.run()
    assert a.results().tobytes() == r1.tobytes()
    assert a.records(out=out).tobytes() == c1.tobytes()
    a.close()


def test_run_batch_cached_arena_resizes(fb, gpu):
    """fb_run_batch reuses one arena per device: a large batch, then a small
    one, then the large one again, each equal to a fresh arena's run."""
    big = SCENARIOS["c2_subset"](gpu.generate_bursty)
    small = big.subset([3])
    for b in (big, small, big):
        res, rec, _ = fb.run_batch(b)
        out = gpu.run(b)
        assert res.tobytes() == out.results.tobytes() and rec.tobytes() == out.records.tobytes()


@pytest.mark.parametrize("name", ["c1", "pab_overload", "wide", "c2_subset"])
def test_lead_series_matches_reference(fb, gpu, golden, name):
    """Envelope-lead series on the device (run-time emission histograms +
    post-run envelope sums) equals the reference's envelope_lead_series
    (metrics.cpp:137-169) point for point, for every instance; the engine's
    decisions are unaffected by the accounting."""
    import hashlib
    from tests_golden_cases import LEAD_CASES
    batch = SCENARIOS[name](gpu.generate_bursty)
    a = fb.Arena(0)
    a.set_lead(ms_to_us(LEAD_CASES[name]), 1 << 14)
    a.load(batch)
    a.run()
    series = a.lead()
    res = a.results()
    a.close()
    assert [hashlib.sha256(s.tobytes()).hexdigest() for s in series] == golden["lead"][name]
    plain = gpu.run(batch)
    assert res.tobytes() == plain.results.tobytes()


def test_lead_capacity_overflow_reported(fb, gpu):
    batch = SCENARIOS["c1"](gpu.generate_bursty)
    a = fb.Arena(0)
    a.set_lead(ms_to_us(500.0), 8)  # far too few points for a 250 s run
    a.load(batch)
    a.run()
    assert all(s is None for s in a.lead())
    a.close()


# ------------------------------------------------------------ interactive node set

@pytest.mark.parametrize("name", ["pab0_8", "count0_8", "count37_3", "pab5000_8", "pab_hz10s_8",
                                  "pab20_2", "c5_pab0_64", "rr_giant_2", "rr_pab30_3",
                                  "rr_count0_4", "rr_mixed_4", "rr_off_pab0_4"])
def test_host_dispatcher_over_node_set_matches_golden(golden, gpu_cluster_cases,
                                                      gpu_reroute_cases, name):
    """run_cluster's loop (cluster.cpp:134-251) on the host, over the batched
    Node surface (fb_nodes_*: advance / enqueue / begin / drain_rejects with
    the report hook): routing, per-node plan digests and records equal the
    reference's run_cluster -- including retry_reroute, where the host
    visits every event time and begins node by node."""
    from backends import cluster_summary
    from paper_2510_14392_b200.cluster import run_cluster_host
    _, rows, cfgs, lb, hz = (gpu_cluster_cases.get(name) or gpu_reroute_cases[name])
    out = run_cluster_host(rows, cfgs, lb, hz)
    assert cluster_summary(out) == golden["clusters"][name]


def test_node_set_queries(fb, gpu_cluster_cases):
    """current_pab / state / drain_rejects against the same nodes' reports,
    visiting every global event time (step ends and arrivals): a node that
    completes at t reports at t, and its PAB / waiting / running queried at t
    equal the report."""
    from paper_2510_14392_b200.cluster import HostRouter, NodeSet
    _, rows, cfgs, lb, hz = gpu_cluster_cases["pab0_8"]
    ns = NodeSet(rows, cfgs, hz, lb)
    view = HostRouter(len(cfgs), lb)
    checked, arr = 0, 0
    try:
        for _ in range(1500):
            st = ns.state()
            busy = st["busy"] != 0
            t = int(st["step_end"][busy].min()) if busy.any() else 1 << 62
            t = min(t, int(rows.arrival_us[arr]))
            rep = ns.advance(t)
            st = ns.state()
            pab = ns.current_pab(t)
            for i in range(len(cfgs)):
                assert st["busy"][i] == 0 or st["step_end"][i] > t
                if rep["fresh"][i]:
                    view.apply(i, int(rep["emitted_at"][i]), int(rep["pab_tokens"][i]),
                               int(rep["waiting"][i]), int(rep["running"][i]))
                    if rep["emitted_at"][i] == t:  # completed and reported at this instant
                        assert pab[i] == rep["pab_tokens"][i]
                        assert (st["waiting"][i], st["running"][i]) == (rep["waiting"][i],
                                                                        rep["running"][i])
                        checked += 1
            q = arr
            while arr < len(rows) and rows.arrival_us[arr] == t:
                arr += 1
            ns.enqueue(t, [view.route(int(rows.prompt_len[k])) for k in range(q, arr)],
                       np.arange(q, arr))
            ns.begin(t)
        assert checked > 100
        assert isinstance(ns.drain_rejects(), list)
        with pytest.raises(fb.UsageError):
            ns.enqueue(0, [len(cfgs)], [0])
    finally:
        ns.close()
