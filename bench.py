"""Benchmark: FairBatching per-iteration scheduling on B200.

Workload (BASELINE.json configs[1]): Sarathi (512) vs
FairBatching (2048) A/B on the qwen-like bursty trace x1.5, 2048 seeds ->
4096 concurrent Node instances, each run to quiescence.  One bench "step" is
one pass of the hot path over the whole sweep: arena reset + every instance's
run_node event loop (arrival injection, PAB/none admission, views, slack
ordering, capacity scan, ground-truth step, completion, online records).

metric: scheduler iterations/sec = sum over instances of begin_step launches
(steps incl. spin steps, engine.h:139) / device time.  Multi-GPU: one process
per GPU, each runs its own 2048-seed shard (weak scaling, no data-path
collective); value = all ranks' steps / max-over-ranks time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
# 32 hardware work queues: the C5 replica item runs 16 cluster simulations
# on their own streams (must be set before the CUDA context exists)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "scheduler iterations/sec (instances·steps/s) at 1/2/4/8 B200 vs CPU ref"
UNIT = "instance-steps/s"
SEEDS_PER_GPU = 2048
L2_FLUSH_BYTES = 256 << 20


def workload_config(n_gpus: int) -> dict:
    return {
        "workload": "C2: sarathi-512 vs fairbatch-2048 A/B, qwen bursty x1.5, 40 s trace, "
                    f"{SEEDS_PER_GPU} seeds x 2 policies = {2 * SEEDS_PER_GPU} instances per GPU",
        "instances": 2 * SEEDS_PER_GPU * n_gpus,
        "cost_model": "a=5.0 b=0.05 c=0.0001 ms (scheduler and truth)",
        "slo_ms": [500, 50],
        "parallelism": f"instance-sharded x{n_gpus}",
        "l2": "flushed between timed iterations (256 MiB write)",
    }


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[3:7]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def measured_peak_hbm() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def ncu_summary() -> dict:
    """The committed ncu --set full summary of the engine kernel."""
    path = os.path.join(ROOT, "profiles", "engine_ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def ncu_traffic():
    """DRAM bytes per engine launch from the committed ncu --set full summary."""
    return ncu_summary().get("dram_bytes_per_launch")


def ref_lib():
    """The reference's own CPU implementation (oracle/_ref, compiled unmodified
    from /root/reference), else the C oracle port (kind "port")."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from backends import REF_SO, OracleLib, RefLib
    if os.path.exists(REF_SO):
        return RefLib(), "reference"
    return OracleLib(), "port"


def ref_batch_runner(lib, kind, n_threads):
    if kind == "reference":
        return lambda b: lib.run_node_batch(b, nthreads=n_threads)  # stock run_node
    return lambda b: lib.run(b, nthreads=n_threads)


def cpu_baseline(batch, n_threads: int, budget_s: float = 15.0, lib=None) -> dict:
    """The reference's own CPU run_node + request_reports (oracle/_ref) on the
    same instances with `n_threads` host threads: the whole batch when it fits
    `budget_s`, else an evenly strided sample sized to it.  Returns the line
    plus the run's outputs (`_out`, `_sel`) for the parity check."""
    if lib is None:
        lib = ref_lib()
    lib, kind = lib
    runner = ref_batch_runner(lib, kind, n_threads)
    n_total = batch.n_instances
    take = min(n_total, max(2 * n_threads, 64))
    while True:
        sel = list(range(0, n_total, max(1, n_total // take)))[:take]
        sub = batch if len(sel) == n_total else batch.subset(sel)
        t0 = time.perf_counter()
        out = runner(sub)
        dt = time.perf_counter() - t0
        steps = int(out.results["steps"].sum())
        if dt >= budget_s / 3 or take >= n_total:
            break
        take = min(n_total, int(take * max(2.0, (budget_s / 2) / max(dt, 1e-3))))
    return {"value": steps / dt, "unit": UNIT, "cores": n_threads, "kind": kind,
            "sample": f"{len(sel)} of {n_total} instances ({steps} instance-steps) in {dt:.2f} s, "
                      f"{n_threads} threads, {os.cpu_count()} host CPUs",
            "cpu_model": cpu_model(), "_out": out, "_sel": sel}


def live_parity(gpu_res, gpu_rec, batch, out, sel) -> dict:
    """Per-instance step / arrival / reject counts, incomplete flags and the
    per-request records of the GPU run against the reference's stock
    run_node + request_reports on the same instances."""
    keys = ("steps", "n_arrived", "n_rejected", "incomplete")
    off = batch.record_offsets()
    g = gpu_res[sel]
    ok = {k: bool(np.array_equal(g[k].astype(np.int64), out.results[k].astype(np.int64)))
          for k in keys}
    rec = np.concatenate([gpu_rec[off[i]:off[i + 1]] for i in sel]) if sel else gpu_rec[:0]
    ok["records"] = bool(rec.tobytes() == out.records.tobytes())
    return {"instances": len(sel), "equal": all(ok.values()), "fields": ok,
            "against": "reference run_node + request_reports (oracle/_ref), live on this host"}


def fixture_parity(name: str, batch, res, rec=None) -> dict:
    """Per-instance plan digests (every step's batch composition, chunk sizes
    and step times) against the committed reference fixture
    tests/golden/full_size.json (made by tests/golden/make_golden_full.py from
    oracle/_ref, checked against the real run_node)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from full_size import CONFIGS, canonical_results, chunk_digests
    with open(os.path.join(ROOT, "tests", "golden", "full_size.json")) as f:
        gold = json.load(f)[name]
    chunk = CONFIGS[name]["chunk"]
    if rec is not None:
        got = chunk_digests(batch, res, rec, chunk)
        rec_eq = got["records_sha256"] == gold["records_sha256"]
    else:
        import hashlib
        can = canonical_results(res)
        got = {"results_sha256": [hashlib.sha256(can[c:c + chunk].tobytes()).hexdigest()
                                  for c in range(0, len(res), chunk)],
               "total_steps": int(res["steps"].sum())}
        rec_eq = None
    eq = got["results_sha256"] == gold["results_sha256"]
    return {"fixture": f"tests/golden/full_size.json:{name}", "instances": len(res),
            "plan_digests_equal": bool(eq), "records_equal": rec_eq,
            "total_steps": got["total_steps"], "reference_total_steps": gold["total_steps"],
            "equal": bool(eq and rec_eq is not False and got["total_steps"] == gold["total_steps"])}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def bench_c4(peak: float, peak_kind: str, reps: int = 3, cpu: bool = True) -> dict:
    """Secondary line item: BASELINE config 4 (decode-heavy, 64 nodes x 120k
    requests, > 77k visible tasks per step), the only configuration whose
    per-step working set exceeds L2, so the one whose slack/selection passes
    are HBM-bound.  Runs on the grid-wide wide engine; roofline over the
    whole pass (both engine kernels, device events).  Parity: plan digests
    against the reference fixture; with `cpu`, the reference's run_node on
    all 64 instances with every host thread (measured, and compared)."""
    from paper_2510_14392_b200 import fbgpu, workloads
    batch = workloads.c4_batch(n_inst=64)
    arena = fbgpu.Arena(0)
    arena.load(batch)
    arena.run()
    arena.synchronize()
    tot, wide, phases = [], [], []
    for _ in range(reps):
        arena.reset()
        arena.run()
        arena.synchronize()
        w, g = arena.last_run_split_ms()
        tot.append(w + g)
        wide.append(g)
        phases.append(arena.wide_phases()[0])
    r = arena.results()
    rec = arena.records()
    arena.close()
    ph = {k: statistics.median(p[k] for p in phases) for k in phases[0]}
    try:
        with open(os.path.join(ROOT, "profiles", "wide_ncu_summary.json")) as f:
            wide_ncu = json.load(f)
    except (OSError, ValueError):
        wide_ncu = {}
    # the slack/selection kernels proper: K1 views (envelope slack, key
    # stems) + K2 histogram + K2 gather, each phase timed on the device up to
    # and including its closing grid barrier; algorithmic bytes 32 per
    # visible task
    sel_ms = ph["k1_views"] + ph["k2_hist"] + ph["k2_gather"]
    sel_bytes = 32 * int(r["sum_visible"].sum())
    sel_ach = sel_bytes / (sel_ms / 1000.0) / 1e9
    k1_ach = sel_bytes / (ph["k1_views"] / 1000.0) / 1e9
    steps = int(r["steps"].sum())
    alg = int(32 * r["sum_visible"].sum() + 64 * r["sum_entries"].sum()
              + 64 * r["n_arrived"].sum())
    ms = statistics.median(tot)
    ach = alg / (ms / 1000.0) / 1e9
    line = {"workload": "C4: decode-heavy, 64 nodes x 120,000 requests, horizon 1.5 s",
            "value": steps / (ms / 1000.0), "unit": UNIT, "ms_per_pass": ms,
            "wide_engine_ms": statistics.median(wide), "instance_steps": steps,
            "mean_visible": float(r["sum_visible"].sum()) / max(steps, 1),
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak, "traffic": wide_ncu.get("dram_bytes_per_launch"),
                         "traffic_source": "profiles/wide_ncu_summary.json (" +
                                           str(wide_ncu.get("tag")) +
                                           ": wide_grid_kernel, one C4 pass)",
                         "kernel": "engine_kernel+wide_grid_kernel (whole pass)",
                         "alg_bytes_per_launch": alg, "peak_source": peak_kind},
            "phases_ms": ph,
            "roofline_slack_selection": {
                "bound": "hbm", "achieved": sel_ach, "peak": peak, "unit": "GB/s",
                "frac": sel_ach / peak, "phases": "K1 views + K2a histogram + K2b gather",
                "alg_bytes": sel_bytes, "ms": sel_ms,
                "k1_views_achieved": k1_ach, "k1_views_frac": k1_ach / peak},
            "parity": {"fixture": fixture_parity("c4_full", batch, r, rec)}}
    if cpu:
        lib = ref_lib()
        nt = os.cpu_count() or 1
        cb = cpu_baseline(batch, nt, budget_s=1e9, lib=lib)  # all 64 instances
        out, sel = cb.pop("_out"), cb.pop("_sel")
        line["cpu_reference"] = cb
        line["parity"]["live"] = live_parity(r, rec, batch, out, sel)
    return line


def bench_c5(reps: int = 3, cpu: bool = True) -> dict:
    """Secondary line item: BASELINE config 5, the 64-node cluster (one GPU;
    the grid is one thread-block cluster), next to the reference's own
    single-threaded run_cluster on this host; plus as many copies side by
    side as fit the GPU as one-cluster grids (replicas, the multi-simulation
    throughput form: each copy is bound by its per-epoch latency, so the GPU
    runs many at once) next to the reference running the same copies on
    every host thread."""
    import ctypes as C
    from paper_2510_14392_b200 import cluster, fbgpu
    rows, cfgs, lb, hz = cluster.c5()
    fit1 = cluster.cluster_fit(len(cfgs), 1)
    fit2 = cluster.cluster_fit(len(cfgs), 2)
    # as many copies as fit as one-cluster grids at two CTAs per SM (more
    # would push every copy off the hardware-cluster path), one stream each,
    # at most one per hardware work queue (CUDA_DEVICE_MAX_CONNECTIONS, 32:
    # a 33rd stream would queue behind another copy)
    queues = int(os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8"))
    n_rep = max(1, min(max(fit1, fit2), queues))
    mode = cluster.cluster_density(n_rep, len(cfgs))
    best, out = 1e30, None
    for _ in range(reps):
        out = cluster.run_cluster(rows, cfgs, lb, hz)
        best = min(best, out.device_ms)
    steps = int(out.node_results["steps"].sum())
    line = {"workload": "C5: 64-node cluster, pab_lb, 11,694 requests, 11,690 dispatch epochs",
            "value": steps / (best / 1000.0), "unit": "node-steps/s", "ms_per_pass": best,
            "node_steps": steps}
    # replicas: one launch per copy on its own stream, all copies at once
    cases = [(rows, cfgs, lb, hz)] * n_rep
    cluster.run_clusters(cases)
    t_rep = []
    for _ in range(reps):
        span = {}
        outs = cluster.run_clusters(cases, span=span)
        t_rep.append(span["ms"] / 1000.0)
    rep_steps = sum(int(o.node_results["steps"].sum()) for o in outs)
    line["replicas"] = {"copies": n_rep, "fit_as_hw_clusters": {"1_cta_per_sm": fit1,
                                                                  "2_ctas_per_sm": fit2},
                        "ctas_per_sm": mode,
                        "value": rep_steps / min(t_rep), "unit": "node-steps/s",
                        "ms_per_pass": 1000.0 * min(t_rep),
                        "timing": "host clock from the first launch to the last copy's "
                                  "completion (inputs resident)"}
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from backends import REF_SO, RefLib, cluster_summary
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        gold = json.load(f)["clusters"]["c5_pab0_64"]
    line["parity"] = {"fixture": {"fixture": "tests/golden/golden.json:clusters.c5_pab0_64",
                                  "equal": cluster_summary(out) == gold and
                                  all(cluster_summary(o) == gold for o in outs)}}
    if cpu and os.path.exists(REF_SO):
        ref = RefLib()
        t0 = time.perf_counter()
        res1, rec1 = ref.run_cluster_stock(rows, cfgs, lb, hz, 1, 1, records=True)
        dt = time.perf_counter() - t0
        line["cpu_reference"] = {"value": steps / dt, "unit": "node-steps/s", "cores": 1,
                                 "kind": "reference",
                                 "sample": f"the whole C5 run_cluster in {dt:.2f} s "
                                           "(sequential by construction)"}
        keys = ("steps", "n_arrived", "n_rejected", "incomplete")
        line["parity"]["live"] = {
            "equal": bool(all(np.array_equal(res1[0][k].astype(np.int64),
                                             out.node_results[k].astype(np.int64)) for k in keys)
                          and rec1.tobytes() == out.records.tobytes()),
            "against": "reference run_cluster (stock) + request_reports, live on this host"}
        nt = min(n_rep, os.cpu_count() or 1)
        t0 = time.perf_counter()
        ref.run_cluster_stock(rows, cfgs, lb, hz, n_rep, nt)
        dt = time.perf_counter() - t0
        line["replicas"]["cpu_reference"] = {
            "value": rep_steps / dt, "unit": "node-steps/s", "cores": nt, "kind": "reference",
            "sample": f"{n_rep} copies of run_cluster on {nt} threads in {dt:.2f} s"}
    return line


def bench_c3(ws: int, rank: int, dev: int, stream, reps: int = 3) -> dict:
    """BASELINE config 3, the capacity-search grid, at its stated size:
    65,536 instances (64 trace seeds x 16 scales x 16 SLO pairs x 4
    policies), dealt round-robin over the ranks (strong scaling: the total is
    fixed).  Device time per pass, max over ranks; per-instance results
    gathered to every rank over NCCL and checked against the reference
    fixture (plan digests of all 65,536 instances; records too at N=1)."""
    import torch
    from paper_2510_14392_b200 import dist as fdist
    from paper_2510_14392_b200 import fbgpu, workloads
    batch = workloads.c3_batch(shard=rank, n_shards=ws)
    arena = fbgpu.Arena(dev, stream=stream.cuda_stream)
    arena.load(batch)
    arena.run()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        _barrier(ws)
        a.record(stream)
        arena.reset()
        arena.run()
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    res = arena.results()
    rec = arena.records() if ws == 1 else None
    arena.close()
    t = torch.tensor([statistics.median(ms), float(res["steps"].sum())], dtype=torch.float64,
                     device="cuda")
    if ws > 1:
        tmax = t[:1].clone()
        torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
        tsum = t[1:].clone()
        torch.distributed.all_reduce(tsum, op=torch.distributed.ReduceOp.SUM)
        t = torch.cat([tmax, tsum])
        idx = np.asarray(fdist.shard_indices(65536, rank, ws), np.int64)
        res = fdist.gather_results(res, idx, 65536, torch.distributed, device="cuda")
    max_ms, steps = float(t[0].item()), float(t[1].item())
    line = {"workload": "C3: balanced bursty trace, 64 seeds x 16 scales x 16 (TTFT, TPOT) SLO "
                        "pairs x 4 policies = 65,536 instances",
            "value": steps / (max_ms / 1000.0), "unit": UNIT, "ms_per_pass": max_ms,
            "instance_steps": steps, "n_gpus": ws, "scaling": "strong",
            "instances_per_gpu": batch.n_instances}
    if rank == 0:  # at N=1 `batch` is the whole grid; at N>1 results only
        line["parity"] = {"fixture": fixture_parity("c3_full", batch, res, rec)}
    return line


def _barrier(ws: int) -> None:
    import torch
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()


def repo_so_loaded() -> list[str]:
    """The repo's product libraries mapped into this process."""
    try:
        with open("/proc/self/maps") as f:
            return sorted({ln.split()[-1] for ln in f
                           if ln.rstrip().endswith(".so") and "paper_2510_14392_b200" in ln})
    except OSError:
        return []


def run_reference(args) -> None:
    """The reference arm: the reference's own CPU implementation (oracle/_ref:
    stock run_node + request_reports, compiled unmodified from /root/reference)
    on the C2 workload, all host threads.  Inputs are generated with the
    reference's own generate_bursty / scale_trace, so nothing of the product
    (libfbgpu.so) is loaded into this process.  Under torchrun only rank 0
    runs."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2510_14392_b200 import workloads
    lib = ref_lib()
    ref, kind = lib

    def scale(rows, f):
        from paper_2510_14392_b200.batch import Rows
        return Rows(ref.scale_trace(rows.arrival_us, f), rows.prompt_len, rows.output_len,
                    rows.ttft_us, rows.tpot_us)
    batch = workloads.c2_batch(n_seeds=SEEDS_PER_GPU, gen=ref.generate_bursty, scale=scale)
    n_threads = os.cpu_count() or 1
    vals = []
    cb = None
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(batch, n_threads, budget_s=args.ref_budget_s, lib=lib)
        r.pop("_out"), r.pop("_sel")
        if i >= args.warmup:
            vals.append(r["value"])
            cb = r
    v = statistics.median(vals)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64+fp64", "data": "synthetic",
            "config": workload_config(1), "impl": "reference",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cb["cores"], "kind": cb["kind"],
                             "sample": cb["sample"], "cpu_model": cb["cpu_model"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "inputs": "generate_bursty / scale_trace of the reference library",
            "repo_so_loaded": repo_so_loaded()}
    print(json.dumps(line), flush=True)


def run_ours(args) -> None:
    import torch
    ws, rank, local = dist_env()
    if ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    from paper_2510_14392_b200 import _abi, fbgpu, workloads

    batch = workloads.c2_batch(n_seeds=SEEDS_PER_GPU, seed0=rank * SEEDS_PER_GPU)
    # a dedicated (non-default) stream shared by torch events and the arena
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0
    arena = fbgpu.Arena(dev, stream=stream.cuda_stream)
    arena.load(batch)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")

    def barrier():
        _barrier(ws)

    # warm-up (full passes)
    for _ in range(args.warmup):
        arena.reset()
        arena.run()
    torch.cuda.synchronize()
    res = arena.results()
    rec0 = arena.records()
    steps_per_pass = int(res["steps"].sum())
    assert (res["status"] == 0).all() and (res["incomplete"] == 0).all()
    # algorithmic bytes per engine launch: 32 A + 64 E + 64 N_arr
    alg_bytes = int(32 * res["sum_visible"].sum() + 64 * res["sum_entries"].sum()
                    + 64 * res["n_arrived"].sum())

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    engine_ms = []
    barrier()
    with ClockSampler(dev) as clocks:
        for k in range(args.steps):
            flush.fill_(k)  # L2 flush outside the timed events
            starts[k].record(stream)
            arena.reset()
            arena.run()
            ends[k].record(stream)
            torch.cuda.synchronize()
            engine_ms.append(arena.last_run_ms())
        barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    n = torch.tensor([steps_per_pass * args.steps], dtype=torch.float64, device="cuda")
    per_rank = torch.tensor([float(steps_per_pass)], dtype=torch.float64, device="cuda")
    rank_steps = [per_rank]
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(n, op=torch.distributed.ReduceOp.SUM)
        rank_steps = [torch.empty_like(per_rank) for _ in range(ws)]
        torch.distributed.all_gather(rank_steps, per_rank)
    max_ms = float(t.item())
    all_steps = float(n.item())
    value = all_steps / (max_ms / 1000.0)

    # end to end through the C ABI with host buffers: the trace rows live in
    # pinned host memory (fb_host_alloc) and every step uploads them plus the
    # instance table (validated + packed on the host), runs, and downloads
    # per-instance results and per-request records into a pinned buffer
    batch.pin()
    rec_out = fbgpu.pinned_empty(arena.record_rows(), _abi.RECORD_DTYPE)
    import ctypes as C
    h2d = batch.rows.nbytes + C.sizeof(_abi.Instance) * batch.n_instances
    # (a) serial: one arena, each step load -> run -> fetch
    e2e_ms = []
    for k in range(max(1, min(args.steps, 5))):
        flush.fill_(k)
        barrier()
        t0 = time.perf_counter()
        arena.load(batch)
        arena.run()
        r2 = arena.results()
        rec = arena.records(out=rec_out)
        e2e_ms.append((time.perf_counter() - t0) * 1000.0)
    d2h = r2.nbytes + rec.nbytes
    assert r2.tobytes() == res.tobytes()
    # (b) pipelined (the e2e figure): two arenas on their own streams; step
    # k+1's host validation/packing and H2D upload overlap step k's device
    # run, then step k's results and records come back.  Every step still
    # uploads its inputs from pinned memory and downloads its outputs.
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    arenas = [fbgpu.Arena(dev, stream=st_.cuda_stream) for st_ in streams]
    outs = [fbgpu.pinned_empty(arena.record_rows(), _abi.RECORD_DTYPE) for _ in range(2)]
    n_pipe = max(2, args.steps)
    for a_ in arenas:  # one-time device allocation outside the timed region
        a_.load(batch)
        a_.run()
        a_.records(out=outs[0])
    # Step k+1 is enqueued before step k's outputs are fetched: its upload
    # overlaps step k's run, and its L2 flush + run (ordered after step k's
    # run by an event) overlap step k's download.
    evs = [torch.cuda.Event(), torch.cuda.Event()]
    barrier()
    t0 = time.perf_counter()
    arenas[0].load(batch)
    with torch.cuda.stream(streams[0]):
        flush.fill_(0)
    arenas[0].run()
    evs[0].record(streams[0])
    for k in range(n_pipe):
        cur, nxt = k % 2, (k + 1) % 2
        if k + 1 < n_pipe:
            arenas[nxt].load(batch)
            streams[nxt].wait_event(evs[cur])
            with torch.cuda.stream(streams[nxt]):
                flush.fill_(k + 1)
            arenas[nxt].run()
            evs[nxt].record(streams[nxt])
        r3 = arenas[cur].results()
        arenas[cur].records(out=outs[cur])
    pipe_ms = (time.perf_counter() - t0) * 1000.0 / n_pipe
    assert r3.tobytes() == res.tobytes() and outs[(n_pipe - 1) % 2].tobytes() == rec.tobytes()
    for a_ in arenas:
        a_.close()
    te = torch.tensor([statistics.median(e2e_ms), pipe_ms], dtype=torch.float64, device="cuda")
    if ws > 1:
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
    serial_ms, pipe_ms = float(te[0].item()), float(te[1].item())
    e2e_value = (all_steps / args.steps) / (pipe_ms / 1000.0)
    e2e_serial = (all_steps / args.steps) / (serial_ms / 1000.0)
    arena.close()

    c3 = None if args.no_c3 else bench_c3(ws, rank, dev, stream)

    if rank == 0:
        peak, peak_kind = measured_peak_hbm()
        eng = statistics.mean(engine_ms)
        achieved = alg_bytes / (eng / 1000.0) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64+fp64", "data": "synthetic",
            "config": workload_config(ws),
            "instance_steps_per_pass": all_steps / args.steps,
            "instance_steps_per_rank": [float(x.item()) for x in rank_steps],
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(),
                         "kernel": "engine_kernel", "kernel_ms": eng,
                         "alg_bytes_per_launch": alg_bytes, "peak_source": peak_kind,
                         # the working set is L2-resident: the binding limit is
                         # instruction issue (ncu, profiles/engine_ncu_summary.json)
                         "issue_active_pct": ncu_summary().get("issue_active_pct"),
                         "l2_hit_rate_pct": ncu_summary().get("lts_hit_rate_pct")},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": pipe_ms,
                    "mode": "pipelined: 2 arenas; step k+1's upload overlaps step k's run, "
                            "its run overlaps step k's download",
                    "serial_value": e2e_serial, "serial_ms_per_step": serial_ms},
            # per step: reset_kernel, engine_kernel (warp engine), wide_kernel
            # (CTA-wide engine; exits at once when no instance escalated)
            "gpu_launches": 3 * args.steps,
            "clocks": clocks.summary(),
            # rank 0's shard is seeds 0..2047, the fixture's batch
            "parity": {"fixture": fixture_parity("c2_full", batch, res, rec0)},
        }
        if c3 is not None:
            line["c3"] = c3
        if ws == 1 and not args.no_c4:
            line["c4"] = bench_c4(peak, peak_kind, cpu=not args.no_cpu_baseline)
            line["c5"] = bench_c5(cpu=not args.no_cpu_baseline)
        if ws == 1 and not args.no_cpu_baseline:
            # the reference on the whole C2 batch (all host threads): the
            # CPU baseline and a live parity check of every instance
            lib = ref_lib()
            cb = cpu_baseline(batch, os.cpu_count() or 1, args.ref_budget_s, lib=lib)
            out, sel = cb.pop("_out"), cb.pop("_sel")
            line["parity"]["live"] = live_parity(res, rec0, batch, out, sel)
            line["cpu_baseline"] = cb
            # the single-core figure beside the all-cores one
            one = cpu_baseline(batch, 1, args.ref_budget_s / 3, lib=lib)
            line["cpu_baseline"]["one_core"] = {"value": one["value"], "sample": one["sample"]}
        line["parity"]["equal"] = all(v.get("equal", True) for v in line["parity"].values()
                                      if isinstance(v, dict))
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def relaunch(args) -> int:
    """`python bench.py --gpus N` (N > 1) outside torchrun: start N ranks
    (one process per GPU) through torch.distributed.run on 127.0.0.1."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_dry(args) -> None:
    """CPU dry run of the multi-rank plumbing (tests/test_dist_cpu.py): gloo
    instead of NCCL, no device work.  Each rank builds its C2 and C3 shards,
    and the same reductions as the GPU run produce the line's n_gpus,
    per-rank steps (here: instances) and the gathered C3 coverage."""
    import torch
    import torch.distributed as dist
    ws, rank, _ = dist_env()
    if ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    dist.init_process_group("gloo")
    from paper_2510_14392_b200 import _abi, workloads
    from paper_2510_14392_b200 import dist as fdist
    c2 = workloads.c2_batch(n_seeds=args.dry_seeds, seed0=rank * args.dry_seeds)
    c3 = workloads.c3_batch(n_seeds=1, shard=rank, n_shards=ws)
    per = torch.tensor([float(c2.n_instances)], dtype=torch.float64)
    parts = [torch.empty_like(per) for _ in range(ws)]
    dist.all_gather(parts, per)
    res = np.zeros(c3.n_instances, _abi.RESULT_DTYPE)
    res["steps"] = [c3.instance(i).n_req for i in range(c3.n_instances)]
    res["plan_digest"] = np.asarray(fdist.shard_indices(1024, rank, ws), np.uint64)
    idx = np.asarray(fdist.shard_indices(1024, rank, ws), np.int64)
    allres = fdist.gather_results(res, idx, 1024, dist)
    if rank == 0:
        print(json.dumps({"n_gpus": ws, "dry_run": True,
                          "instances_per_rank": [float(p.item()) for p in parts],
                          "c3_gathered_in_order": bool(np.array_equal(
                              allres["plan_digest"], np.arange(1024, dtype=np.uint64))),
                          "c3_instances": int(len(allres))}), flush=True)
    dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the config-4/5 line items")
    ap.add_argument("--no-c3", action="store_true", help="skip the config-3 line item")
    ap.add_argument("--ref-budget-s", type=float, default=15.0)
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU-only check of the multi-rank launcher and reductions (gloo)")
    ap.add_argument("--dry-seeds", type=int, default=4)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.dry_run:
        run_dry(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
