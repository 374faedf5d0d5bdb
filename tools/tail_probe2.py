"""Is the C2 pass bound by its longest instances?  Pass time of the batch
without its top-k instances (by step count), and of the top-k alone."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14392_b200 import fbgpu, workloads  # noqa: E402


def timed(b, reps=3):
    a = fbgpu.Arena(0)
    a.load(b)
    ms = []
    for _ in range(reps + 1):
        a.reset()
        a.run()
        a.synchronize()
        ms.append(a.last_run_ms())
    r = a.results()
    a.close()
    return min(ms[1:]), r


batch = workloads.c2_batch()
full, r = timed(batch)
steps = r["steps"].astype(np.int64)
order = np.argsort(-steps)
print(f"full {full:.2f} ms, {steps.sum()} steps, max {steps.max()}")
for k in (8, 64, 256, 1024):
    rest = batch.subset(sorted(order[k:].tolist()))
    ms, rr = timed(rest)
    top = batch.subset(sorted(order[:k].tolist()))
    ms2, _ = timed(top)
    print(f"without top{k}: {ms:.2f} ms ({int(rr['steps'].sum())} steps, max {int(rr['steps'].max())});"
          f" top{k} alone: {ms2:.2f} ms")
