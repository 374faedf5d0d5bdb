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


def cpu_baseline(batch, n_threads: int, budget_s: float = 15.0) -> dict:
    """The reference's own CPU run_node + request_reports (oracle/_ref, the
    unmodified library) on a bounded sample of the same instances, all host
    threads; falls back to the C oracle port when the reference was not built."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from backends import REF_SO, OracleLib, RefLib

    if os.path.exists(REF_SO):
        lib, kind = RefLib(), "reference"
        runner = lambda b: lib.run_node_batch(b, nthreads=n_threads)  # noqa: E731
    else:
        lib, kind = OracleLib(), "port"
        runner = lambda b: lib.run(b, nthreads=n_threads)  # noqa: E731
    # probe with a few instances, then size the sample to ~budget_s
    n_total = batch.n_instances
    take = min(n_total, max(2 * n_threads, 64))
    best = None
    while True:
        sel = list(range(0, n_total, max(1, n_total // take)))[:take]
        sub = batch.subset(sel)
        t0 = time.perf_counter()
        out = runner(sub)
        dt = time.perf_counter() - t0
        steps = int(out.results["steps"].sum())
        best = (steps, dt, len(sel))
        if dt >= budget_s / 3 or take >= n_total:
            break
        take = min(n_total, int(take * max(2.0, (budget_s / 2) / max(dt, 1e-3))))
    steps, dt, n = best
    return {"value": steps / dt, "unit": UNIT, "cores": n_threads, "kind": kind,
            "sample": f"{n} of {n_total} C2 instances ({steps} instance-steps) in {dt:.2f} s, "
                      f"{n_threads} threads, {os.cpu_count()} host CPUs",
            "cpu_model": cpu_model()}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def bench_c4(peak: float, peak_kind: str, reps: int = 3) -> dict:
    """Secondary line item: BASELINE config 4 (decode-heavy, 64 nodes x 120k
    requests, > 77k visible tasks per step), the only configuration whose
    per-step working set exceeds L2, so the one whose slack/selection passes
    are HBM-bound.  Runs on the grid-wide wide engine; roofline over the
    whole pass (both engine kernels, device events)."""
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
    arena.close()
    ph = {k: statistics.median(p[k] for p in phases) for k in phases[0]}
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
    return {"workload": "C4: decode-heavy, 64 nodes x 120,000 requests, horizon 1.5 s",
            "value": steps / (ms / 1000.0), "unit": UNIT, "ms_per_pass": ms,
            "wide_engine_ms": statistics.median(wide), "instance_steps": steps,
            "mean_visible": float(r["sum_visible"].sum()) / max(steps, 1),
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak, "traffic": None,
                         "kernel": "engine_kernel+wide_grid_kernel (whole pass)",
                         "alg_bytes_per_launch": alg, "peak_source": peak_kind},
            "phases_ms": ph,
            "roofline_slack_selection": {
                "bound": "hbm", "achieved": sel_ach, "peak": peak, "unit": "GB/s",
                "frac": sel_ach / peak, "phases": "K1 views + K2a histogram + K2b gather",
                "alg_bytes": sel_bytes, "ms": sel_ms,
                "k1_views_achieved": k1_ach, "k1_views_frac": k1_ach / peak}}


def bench_c5(reps: int = 3) -> dict:
    """Secondary line item: BASELINE config 5, the 64-node cluster (one GPU;
    the grid is one thread-block cluster), next to the reference's
    single-threaded run_cluster on this host."""
    from paper_2510_14392_b200 import cluster
    rows, cfgs, lb, hz = cluster.c5()
    best, out = 1e30, None
    for _ in range(reps):
        out = cluster.run_cluster(rows, cfgs, lb, hz)
        best = min(best, out.device_ms)
    steps = int(out.node_results["steps"].sum())
    line = {"workload": "C5: 64-node cluster, pab_lb, 11,694 requests, 11,690 dispatch epochs",
            "value": steps / (best / 1000.0), "unit": "node-steps/s", "ms_per_pass": best,
            "node_steps": steps}
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from backends import REF_SO, RefLib
    if os.path.exists(REF_SO):
        t0 = time.perf_counter()
        RefLib().run_cluster(rows, cfgs, lb, hz)
        dt = time.perf_counter() - t0
        line["cpu_reference"] = {"value": steps / dt, "unit": "node-steps/s", "cores": 1,
                                 "kind": "reference",
                                 "sample": f"the whole C5 run_cluster in {dt:.2f} s (sequential)"}
    return line


def run_reference(args) -> None:
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2510_14392_b200 import workloads
    batch = workloads.c2_batch(n_seeds=SEEDS_PER_GPU)
    n_threads = os.cpu_count() or 1
    vals = []
    cb = None
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(batch, n_threads, budget_s=args.ref_budget_s)
        if i >= args.warmup:
            vals.append(r["value"])
            cb = r
    v = statistics.median(vals)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64+fp64", "data": "synthetic",
            "config": workload_config(1), "impl": "reference",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cb["cores"], "kind": cb["kind"],
                             "sample": cb["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args) -> None:
    import torch
    ws, rank, local = dist_env()
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
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # warm-up (full passes)
    for _ in range(args.warmup):
        arena.reset()
        arena.run()
    torch.cuda.synchronize()
    res = arena.results()
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
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(n, op=torch.distributed.ReduceOp.SUM)
    max_ms = float(t.item())
    all_steps = float(n.item())
    value = all_steps / (max_ms / 1000.0)

    # end to end through the C ABI with host buffers: the trace rows live in
    # pinned host memory (fb_host_alloc) and every step uploads them plus the
    # instance table (validated + packed on the host), runs, and downloads
    # per-instance results and per-request records into a pinned buffer
    batch.pin()
    rec_out = fbgpu.pinned_empty(arena.record_rows(), _abi.RECORD_DTYPE)
    rows = batch.rows
    import ctypes as C
    h2d = rows.nbytes + C.sizeof(_abi.Instance) * batch.n_instances
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
        }
        if ws == 1 and not args.no_c4:
            line["c4"] = bench_c4(peak, peak_kind)
            line["c5"] = bench_c5()
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(batch, os.cpu_count() or 1, args.ref_budget_s)
            # the single-core figure beside the all-cores one
            one = cpu_baseline(batch, 1, args.ref_budget_s / 3)
            line["cpu_baseline"]["one_core"] = {"value": one["value"], "sample": one["sample"]}
        print(json.dumps(line), flush=True)
    arena.close()
    if ws > 1:
        torch.distributed.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the config-4 line item")
    ap.add_argument("--ref-budget-s", type=float, default=15.0)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
