"""A/B timing of one workload pass (dev tool): FBGPU_LIB=... python tools/ab_time.py c2|c3|c4 [reps]
Prints ms per pass (median of reps, device events) and a digest of results."""
import hashlib
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14392_b200 import fbgpu, workloads  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
if which == "c2":
    batch = workloads.c2_batch(n_seeds=2048)
elif which == "c3":
    batch = workloads.c3_batch(n_seeds=8)
elif which == "c4":
    batch = workloads.c4_batch(n_inst=64)
elif which == "c1":
    batch = workloads.c1_batch(("fairbatch", "fairbatch_pab", "sarathi", "prefill_first"))
else:
    raise SystemExit(which)
a = fbgpu.Arena(0)
a.load(batch)
ms = []
for k in range(reps + 2):
    a.reset()
    a.run()
    a.synchronize()
    if k >= 2:
        ms.append(a.last_run_ms())
r = a.results()
h = hashlib.sha1(r.tobytes() + a.records().tobytes()).hexdigest()[:12]
steps = int(r["steps"].sum())
med = statistics.median(ms)
print(f"{os.environ.get('FBGPU_LIB', 'default')} {which} {batch.n_instances} inst {steps} steps "
      f"{med:.3f} ms (min {min(ms):.3f}) {steps / med / 1e3:.1f} M steps/s digest {h}")
