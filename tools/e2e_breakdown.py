"""Where the end-to-end (host buffers) C2 time goes (dev tool).
    python tools/e2e_breakdown.py [reps]"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14392_b200 import fbgpu, workloads  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
batch = workloads.c2_batch(n_seeds=2048)
pinned = len(sys.argv) > 2 and sys.argv[2] == "pinned"
a = fbgpu.Arena(0)
a.load(batch)
a.run()
a.synchronize()
out = None
if pinned:
    batch.pin()
    out = fbgpu.pinned_empty(a.record_rows(), fbgpu._abi.RECORD_DTYPE)
ph = {k: [] for k in ("instances_c", "load", "run", "results", "records", "total", "run_batch")}
for _ in range(reps):
    t0 = time.perf_counter()
    inst = batch.instances_c()
    t1 = time.perf_counter()
    a.load(batch)
    t2 = time.perf_counter()
    a.run()
    a.synchronize()
    t3 = time.perf_counter()
    r = a.results()
    t4 = time.perf_counter()
    rec = a.records(out=out)
    t5 = time.perf_counter()
    for k, v in zip(("instances_c", "load", "run", "results", "records", "total"),
                    (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t5 - t1)):
        ph[k].append(v * 1e3)
    t6 = time.perf_counter()
    fbgpu.run_batch(batch)
    ph["run_batch"].append((time.perf_counter() - t6) * 1e3)
print("pinned" if pinned else "pageable", {k: round(statistics.median(v), 3) for k, v in ph.items()}, "device ms", a.last_run_ms())
