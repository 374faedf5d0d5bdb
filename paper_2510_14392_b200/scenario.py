"""Scenario files and experiment drivers on the device (the reference's
scenario.cpp / commands.cpp, re-hosted over the batched engine).

* `load_scenario` / `scenario_from_dict`: the JSON schema of scenario.cpp:77-222
  (unknown keys rejected, same defaults, ConfigError on bad values);
* `materialize_trace` (scenario.cpp:298-308), `engine_config`
  (scenario.cpp:310-319; truth-noise seed = derive_seed(seed, 3));
* `run_scenario` (commands.cpp:59-85): one node -> Arena, several -> cluster;
* `sweep_scenario` / `tune_sarathi` (commands.cpp:100-190): every
  (policy, scale) or budget point becomes one instance of ONE device batch
  instead of a serial loop of runs.
"""
from __future__ import annotations

import copy
import json
from dataclasses import dataclass, field

import numpy as np

from . import _abi, cluster, fbgpu, reports
from .batch import Batch, CostModel, EngineConfig, Rows, SchedulerConfig, ms_to_us, us_to_ms

M64 = (1 << 64) - 1


def _splitmix(s: int):
    s = (s + 0x9E3779B97F4A7C15) & M64
    z = s
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return s, z ^ (z >> 31)


def derive_seed(base: int, stream: int) -> int:
    """rng.h:33-37."""
    s = (base ^ ((0x9E3779B97F4A7C15 * (stream + 1)) & M64)) & M64
    s, _ = _splitmix(s)
    _, z = _splitmix(s)
    return z


class ConfigError(fbgpu.ConfigError):
    pass


@dataclass
class Scenario:
    """scenario.h:31-61."""

    name: str = "scenario"
    trace_file: str | None = None
    trace_format: str = "jsonl"
    bursty: dict | None = None
    max_requests: int = 0
    scale: float = 1.0
    ttft_ms: float = 0.0
    tpot_ms: float = 0.0
    scheduler: SchedulerConfig = field(default_factory=SchedulerConfig)
    truth: CostModel = field(default_factory=CostModel)
    noise_amplitude: float = 0.0
    nodes: int = 1
    lb: cluster.LbConfig = field(default_factory=cluster.LbConfig)
    horizon_ms: float = 0.0
    seed: int = 0
    out_dir: str = "out"
    max_active: int = 0
    lead_bucket_ms: float = 1000.0
    alt_tpot: bool = False


def _keys(d, section, allowed):
    for k in d:
        if k not in allowed:
            raise ConfigError(f"unknown key '{(section + '.') if section else ''}{k}'")


def _num(d, section, key, default=None):
    if key not in d:
        if default is None:
            raise ConfigError(f"missing required key '{section}.{key}'")
        return default
    v = d[key]
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        raise ConfigError(f"'{section}.{key}' must be a number")
    return float(v)


def _model(d, section):
    _keys(d, section, {"a_ms", "b_ms_per_token", "c_ms_per_context_token"})
    return CostModel(_num(d, section, "a_ms"), _num(d, section, "b_ms_per_token"),
                     _num(d, section, "c_ms_per_context_token"))


def scenario_from_dict(j: dict) -> Scenario:
    """scenario_from_json, scenario.cpp:77-222."""
    _keys(j, "", {"name", "trace", "slo", "scheduler", "cost_model", "cluster", "run"})
    sc = Scenario(name=j.get("name", "scenario"))
    if "trace" not in j:
        raise ConfigError("missing section 'trace'")
    jt = j["trace"]
    _keys(jt, "trace", {"file", "format", "bursty", "max_requests", "scale"})
    if "file" in jt:
        sc.trace_file = jt["file"]
        sc.trace_format = jt.get("format", "jsonl")
        if sc.trace_format not in ("jsonl", "csv"):
            raise ConfigError(f"trace.format must be 'jsonl' or 'csv', got '{sc.trace_format}'")
    if "bursty" in jt:
        jb = jt["bursty"]
        _keys(jb, "trace.bursty", {"base_rate", "burst_rate", "burst_duration_ms",
                                   "idle_duration_ms", "prompt_mean", "prompt_p90",
                                   "output_mean", "output_p90", "seed", "horizon_ms"})
        sc.bursty = {k: _num(jb, "trace.bursty", k) for k in
                     ("base_rate", "burst_rate", "burst_duration_ms", "idle_duration_ms",
                      "prompt_mean", "prompt_p90", "output_mean", "output_p90", "horizon_ms")}
        if "seed" not in jb:
            raise ConfigError("missing required key 'trace.bursty.seed'")
        sc.bursty["seed"] = int(jb["seed"])
    if (sc.trace_file is not None) == (sc.bursty is not None):
        raise ConfigError("trace must name exactly one of 'file' or 'bursty'")
    sc.max_requests = int(_num(jt, "trace", "max_requests", 0.0))
    sc.scale = _num(jt, "trace", "scale", 1.0)
    if not sc.scale > 0.0:
        raise ConfigError("trace.scale must be > 0")
    if "slo" not in j:
        raise ConfigError("missing section 'slo'")
    js = j["slo"]
    _keys(js, "slo", {"ttft_ms", "tpot_ms"})
    sc.ttft_ms, sc.tpot_ms = _num(js, "slo", "ttft_ms"), _num(js, "slo", "tpot_ms")
    if ms_to_us(sc.ttft_ms) <= 0 or ms_to_us(sc.tpot_ms) <= 0:
        raise ConfigError("slo targets must be positive")
    if "cost_model" not in j:
        raise ConfigError("missing section 'cost_model'")
    jc = j["cost_model"]
    _keys(jc, "cost_model", {"truth", "noise_amplitude"})
    if "truth" not in jc:
        raise ConfigError("missing required key 'cost_model.truth'")
    sc.truth = _model(jc["truth"], "cost_model.truth")
    sc.noise_amplitude = _num(jc, "cost_model", "noise_amplitude", 0.0)
    if not 0.0 <= sc.noise_amplitude < 1.0:
        raise ConfigError("cost_model.noise_amplitude must be in [0, 1)")
    if "scheduler" not in j:
        raise ConfigError("missing section 'scheduler'")
    jsch = j["scheduler"]
    _keys(jsch, "scheduler", {"policy", "token_budget", "max_chunk", "model"})
    pol = jsch.get("policy", "")
    if pol not in _abi.POLICY_NAMES:
        raise ConfigError("scheduler.policy must be one of prefill_first, sarathi, fairbatch, "
                          f"fairbatch_pab; got '{pol}'")
    tb = int(_num(jsch, "scheduler", "token_budget", 2048.0))
    mc = int(_num(jsch, "scheduler", "max_chunk", float(tb)))
    model = _model(jsch["model"], "scheduler.model") if "model" in jsch else sc.truth
    sc.scheduler = SchedulerConfig(pol, tb, mc, model)
    jcl = j.get("cluster", {})
    _keys(jcl, "cluster", {"nodes", "policy", "report_interval_steps", "report_latency_ms",
                           "w_waiting", "w_running", "retry_reroute"})
    sc.nodes = int(_num(jcl, "cluster", "nodes", 1.0))
    if sc.nodes < 1:
        raise ConfigError("cluster.nodes must be >= 1")
    lbp = jcl.get("policy", "pab_lb")
    if lbp not in ("pab_lb", "count_lb"):
        raise ConfigError(f"cluster.policy must be count_lb or pab_lb; got '{lbp}'")
    sc.lb = cluster.LbConfig(lbp, int(_num(jcl, "cluster", "report_interval_steps", 1.0)),
                             _num(jcl, "cluster", "report_latency_ms", 0.0),
                             _num(jcl, "cluster", "w_waiting", 1.0),
                             _num(jcl, "cluster", "w_running", 1.0),
                             bool(jcl.get("retry_reroute", False)))
    if sc.lb.report_latency_ms < 0:
        raise ConfigError("cluster.report_latency_ms must be >= 0")
    if "run" not in j:
        raise ConfigError("missing section 'run'")
    jr = j["run"]
    _keys(jr, "run", {"horizon_ms", "seed", "out_dir", "max_active", "lead_bucket_ms", "alt_tpot"})
    sc.horizon_ms = _num(jr, "run", "horizon_ms")
    if ms_to_us(sc.horizon_ms) <= 0:
        raise ConfigError("run.horizon_ms must be > 0")
    if "seed" not in jr:
        raise ConfigError("missing required key 'run.seed' (seeds are explicit)")
    sc.seed = int(jr["seed"])
    sc.out_dir = jr.get("out_dir", "out")
    sc.max_active = int(_num(jr, "run", "max_active", 0.0))
    sc.lead_bucket_ms = _num(jr, "run", "lead_bucket_ms", 1000.0)
    sc.alt_tpot = bool(jr.get("alt_tpot", False))
    s = sc.scheduler  # validate_scheduler_config, sched.cpp:81-88
    if s.max_chunk < 1 or s.token_budget < s.max_chunk or s.model.a_ms < 0 or s.model.b_ms <= 0 \
            or s.model.c_ms < 0:
        raise fbgpu.ValidationError("invalid scheduler configuration")
    return sc


def load_scenario(path: str) -> Scenario:
    """load_scenario, scenario.cpp:280-289."""
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError as e:
        raise ConfigError(f"cannot open scenario file: {path}") from e
    except json.JSONDecodeError as e:
        raise ConfigError(f"scenario {path}: {e}") from e
    return scenario_from_dict(j)


def _load_trace_file(path: str, fmt: str, ttft_us: int, tpot_us: int) -> Rows:
    """load_trace (workload.cpp:185-209): records re-sorted by arrival (stable)."""
    recs = []
    with open(path) as f:
        if fmt == "jsonl":
            for line in f:
                if line.strip():
                    recs.append(json.loads(line))
        else:
            import csv
            recs = [{k: float(v) for k, v in r.items() if v != ""} for r in csv.DictReader(f)]
    arr = [ms_to_us(float(r["arrival_ms"])) for r in recs]
    order = sorted(range(len(recs)), key=lambda i: arr[i])
    return Rows([arr[i] for i in order], [int(recs[i]["prompt_tokens"]) for i in order],
                [int(recs[i]["output_tokens"]) for i in order],
                [ms_to_us(recs[i]["ttft_slo_ms"]) if "ttft_slo_ms" in recs[i] else ttft_us
                 for i in order],
                [ms_to_us(recs[i]["tpot_slo_ms"]) if "tpot_slo_ms" in recs[i] else tpot_us
                 for i in order])


def materialize_trace(sc: Scenario) -> Rows:
    """scenario.cpp:298-308."""
    tt, tp = ms_to_us(sc.ttft_ms), ms_to_us(sc.tpot_ms)
    if sc.trace_file is not None:
        rows = _load_trace_file(sc.trace_file, sc.trace_format, tt, tp)
    else:
        b = sc.bursty
        rows = fbgpu.generate_bursty(
            fbgpu.burst_profile(b["base_rate"], b["burst_rate"], b["burst_duration_ms"],
                                b["idle_duration_ms"], b["prompt_mean"], b["prompt_p90"],
                                b["output_mean"], b["output_p90"], b["seed"], sc.ttft_ms,
                                sc.tpot_ms), ms_to_us(b["horizon_ms"]))
    if sc.scale != 1.0:
        rows = fbgpu.scale_trace(rows, sc.scale)
    return rows.truncated(sc.max_requests)


def engine_config(sc: Scenario) -> EngineConfig:
    """scenario.cpp:310-319."""
    return EngineConfig(scheduler=copy.deepcopy(sc.scheduler), truth_model=sc.truth,
                        noise_amplitude=sc.noise_amplitude, noise_seed=derive_seed(sc.seed, 3),
                        global_ttft_us=ms_to_us(sc.ttft_ms), global_tpot_us=ms_to_us(sc.tpot_ms),
                        max_active=sc.max_active)


def run_scenario(sc: Scenario, device: int = 0) -> reports.ScenarioReport:
    """run_scenario (commands.cpp:59-85) without the file writers."""
    rows = materialize_trace(sc)
    cfg = engine_config(sc)
    if sc.nodes == 1:
        b = Batch()
        b.add(rows, cfg, ms_to_us(sc.horizon_ms))
        a = fbgpu.Arena(device)
        a.load(b)
        a.run()
        rec = a.records()
        a.close()
    else:
        out = cluster.run_cluster(rows, [cfg] * sc.nodes, sc.lb, ms_to_us(sc.horizon_ms), device)
        rec = out.records
    return reports.scenario_report(rec, rows.arrival_us, rows.offered_rps(), sc.name, sc.alt_tpot)


@dataclass
class SweepRow:
    """commands.h:45-51."""

    policy: str
    scale: float
    offered_rps: float
    effective_rps: float
    violation_rate: float


def _run_points(points, device=0):
    """points: list of (rows, EngineConfig, horizon_us) -> ScenarioReports, one batch."""
    b = Batch()
    offs = []
    cache = {}
    for rows, cfg, hz in points:
        key = id(rows)
        if key not in cache:
            cache[key] = b.add_rows(rows)
        b.add_instance(cfg, cache[key], len(rows), hz, rows.offered_rps())
        offs.append(rows)
    a = fbgpu.Arena(device)
    a.load(b)
    a.run()
    summ = a.summaries()  # aggregated on the device: no per-request records shipped
    a.close()
    return [reports.summary_report(summ[i], offs[i].offered_rps()) for i in range(b.n_instances)]


def sweep_scenario(sc: Scenario, scales, policies, device: int = 0) -> list[SweepRow]:
    """sweep_scenario (commands.cpp:100-116) as ONE device batch."""
    base = materialize_trace(sc)
    scaled = {s: fbgpu.scale_trace(base, s) if s != 1.0 else base for s in scales}
    pts, meta = [], []
    for pol in policies:
        for s in scales:
            cfg = engine_config(sc)
            cfg.scheduler.policy = pol
            pts.append((scaled[s], cfg, ms_to_us(sc.horizon_ms)))
            meta.append((pol, s))
    return [SweepRow(p, s, r.offered_rps, r.effective_rps, r.slo_violation_rate)
            for (p, s), r in zip(meta, _run_points(pts, device))]


def tune_sarathi(sc: Scenario, budgets, device: int = 0):
    """tune_sarathi (commands.cpp:169-190): rows + best budget (ties -> smallest)."""
    rows = materialize_trace(sc)
    pts = []
    for b in budgets:
        cfg = engine_config(sc)
        cfg.scheduler.policy = "sarathi"
        cfg.scheduler.token_budget = int(b)
        cfg.scheduler.max_chunk = int(min(int(b), sc.scheduler.max_chunk))
        pts.append((rows, cfg, ms_to_us(sc.horizon_ms)))
    res = _run_points(pts, device)
    out = [(int(b), r.effective_rps) for b, r in zip(budgets, res)]
    best, best_rps = 0, -1.0
    for b, e in out:  # strict > keeps the first maximum in scan order
        if e > best_rps:
            best, best_rps = b, e
    return out, best
