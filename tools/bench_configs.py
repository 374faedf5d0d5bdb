"""Per-config measurements (C1, C3 sample, C4, C5) on one B200 next to the
reference CPU code on this host.  Prints one JSON object per config.

    python tools/bench_configs.py [c1 c3 c4 c5]
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2510_14392_b200 import cluster, fbgpu, workloads  # noqa: E402

NCPU = os.cpu_count() or 1


def ref_lib():
    from backends import REF_SO, RefLib
    return RefLib() if os.path.exists(REF_SO) else None


def gpu_batch(batch, reps=3):
    a = fbgpu.Arena(0)
    a.load(batch)
    ms = []
    for _ in range(reps):
        a.reset()
        a.run()
        a.synchronize()
        ms.append(a.last_run_ms())
    r = a.results()
    paths = np.bitwise_or.reduce(a.paths())
    a.close()
    return min(ms), r, int(paths)


def cpu_batch(ref, batch, budget_s=20.0):
    """Reference run_node on all host threads over a bounded sample."""
    n = batch.n_instances
    take = min(n, max(NCPU, 8))
    while True:
        sub = batch.subset(list(range(0, n, max(1, n // take)))[:take])
        t0 = time.perf_counter()
        out = ref.run_node_batch(sub, nthreads=NCPU, records=True)
        dt = time.perf_counter() - t0
        if dt > budget_s / 4 or take >= n:
            return int(out.results["steps"].sum()) / dt, take
        take = min(n, take * 4)


def report(name, steps, ms, cpu=None, extra=None):
    d = {"config": name, "instance_steps": steps, "device_ms": ms,
         "gpu_steps_per_s": steps / (ms / 1000.0)}
    if cpu:
        d["cpu_ref_steps_per_s"], d["cpu_sample_instances"] = cpu
        d["cpu_threads"] = NCPU
        d["speedup_vs_cpu_ref"] = d["gpu_steps_per_s"] / cpu[0]
    d.update(extra or {})
    print(json.dumps(d), flush=True)


def main(which):
    ref = ref_lib()
    if "c1" in which:
        b = workloads.c1_batch(("fairbatch", "sarathi", "prefill_first", "fairbatch_pab"))
        ms, r, p = gpu_batch(b)
        report("C1 (931-request Poisson trace, 4 policies)", int(r["steps"].sum()), ms,
               cpu_batch(ref, b) if ref else None, {"paths": p})
    if "c3" in which:
        b = workloads.c3_batch(n_seeds=8)  # 8 of 64 seeds: 8,192 instances
        ms, r, p = gpu_batch(b, reps=2)
        report("C3 sample (8 trace seeds x 16 scales x 16 SLO pairs x 4 policies)",
               int(r["steps"].sum()), ms, cpu_batch(ref, b) if ref else None,
               {"instances": b.n_instances, "paths": p})
    if "c4" in which:
        b = workloads.c4_batch(n_inst=64)
        ms, r, p = gpu_batch(b)
        alg = 32 * r["sum_visible"].sum() + 64 * r["sum_entries"].sum() + 64 * r["n_arrived"].sum()
        cpu = None
        if ref:
            sub = b.subset([0])
            t0 = time.perf_counter()
            o = ref.run_node_batch(sub, nthreads=1)
            dt = time.perf_counter() - t0
            cpu = (int(o.results["steps"].sum()) / dt * min(NCPU, 64), 1)
        report("C4 (64 instances x 120k requests, decode-heavy)", int(r["steps"].sum()), ms, cpu,
               {"mean_visible": float((r["sum_visible"] / r["steps"]).mean()),
                "alg_GBps": float(alg / (ms / 1e3) / 1e9), "paths": p,
                "cpu_note": "1 instance single-thread x min(threads, 64) (instances independent)"})
    if "c5" in which:
        rows, cfgs, lb, hz = cluster.c5()
        best = 1e30
        for _ in range(3):
            out = cluster.run_cluster(rows, cfgs, lb, hz)
            best = min(best, out.device_ms)
        steps = int(out.node_results["steps"].sum())
        cpu = None
        if ref:
            t0 = time.perf_counter()
            ref.run_cluster(rows, cfgs, lb, hz)
            dt = time.perf_counter() - t0
            cpu = (steps / dt, 1)
        report("C5 (64-node cluster, pab_lb, 11,694 requests)", steps, best, cpu,
               {"epochs": int(len(np.unique(rows.arrival_us))),
                "cpu_note": "reference run_cluster is single-threaded by construction"})
    if "c5x" in which:
        # C5 replicas side by side (run_clusters): R seeds of the 64-node
        # cluster, one shard + stream each; device time = first launch to last
        # completion (host clock around launch-all / wait-all)
        R = 16
        cases = []
        for i in range(R):
            _, cfgs, lb, hz = cluster.c5()
            cases.append((cluster.c5_rows(seed=5 + i), cfgs, lb, hz))
        best, steps = 1e30, 0
        for _ in range(3):
            shards = [cluster.ClusterShard(r, c, l, h, 0, 1) for r, c, l, h in cases]
            fit = C.c_int32(0)
            fbgpu.lib().fb_cluster_max_hw_clusters(0, len(cases[0][1]), C.byref(fit))
            for sh in shards:  # as run_clusters: one-cluster grids only if all fit
                fbgpu.lib().fb_cluster_shard_allow_hw_cluster(sh._h, int(R <= fit.value))
                sh.reset()
            t0 = time.perf_counter()
            for sh in shards:
                sh.launch()
            for sh in shards:
                sh.wait()
            best = min(best, (time.perf_counter() - t0) * 1e3)
            steps = sum(int(sh.fetch().node_results["steps"].sum()) for sh in shards)
            for sh in shards:
                sh.close()
        cpu = None
        if ref:
            from concurrent.futures import ThreadPoolExecutor
            t0 = time.perf_counter()
            with ThreadPoolExecutor(min(R, NCPU)) as ex:
                list(ex.map(lambda c: ref.run_cluster(*c), cases))
            cpu = (steps / (time.perf_counter() - t0), min(R, NCPU))
        report(f"C5 x{R} replicas side by side (run_clusters, 64 nodes each)", steps, best, cpu,
               {"replicas": R, "cpu_note": "reference run_cluster, one replica per host thread"})


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c3", "c4", "c5", "c5x"])
