"""BASELINE config 3 at full size on one GPU: 65,536 instances (64 trace seeds x
16 load scales x 16 SLO pairs x 4 policies).  Prints device time, steps/s and
the summary-based capacity search result (max load scale per policy and SLO
pair with attainment >= 90%), with per-request records never leaving the GPU."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14392_b200 import fbgpu, workloads  # noqa: E402

t0 = time.time()
batch = workloads.c3_batch(n_seeds=int(sys.argv[1]) if len(sys.argv) > 1 else 64)
t1 = time.time()
a = fbgpu.Arena(0)
a.load(batch)
a.run()
a.synchronize()
ms = a.last_run_ms()
a.reset()
a.run()
a.synchronize()
ms2 = a.last_run_ms()
r = a.results()
t2 = time.time()
s = a.summaries()
t3 = time.time()
steps = int(r["steps"].sum())
att = s["good"] / np.maximum(1, s["total_requests"])
print(f"C3 full: {batch.n_instances} instances, {len(batch.rows)} trace rows, "
      f"{steps} instance-steps, device {ms2:.1f} ms ({steps / ms2 / 1e3:.1f} M steps/s), "
      f"summaries {1e3 * (t3 - t2):.1f} ms, mean attainment {att.mean():.3f}, "
      f"gen {t1 - t0:.1f} s, paths {np.bitwise_or.reduce(a.paths())}, incomplete {int(r['incomplete'].sum())}")
