"""Probes the tail: how long do the longest C2 instances take alone?"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14392_b200 import fbgpu, workloads  # noqa: E402

batch = workloads.c2_batch()
a = fbgpu.Arena(0)
a.load(batch)
a.run()
a.synchronize()
full_ms = a.last_run_ms()
r = a.results()
steps = r["steps"].astype(np.int64)
order = np.argsort(-steps)
print("full", full_ms, "ms; steps max", steps.max(), "p99", np.percentile(steps, 99), "mean", steps.mean())
for k in (1, 8, 64, 512):
    sub = batch.subset(order[:k].tolist())
    b = fbgpu.Arena(0)
    b.load(sub)
    b.run()
    b.synchronize()
    b.reset()
    b.run()
    b.synchronize()
    ms = b.last_run_ms()
    rs = b.results()
    print(f"top{k}: {ms:.2f} ms, max steps {rs['steps'].max()}, us/step(max) {1000*ms/rs['steps'].max():.3f}")
# longest-first ordering of the full batch
lpt = batch.subset(order.tolist())
c = fbgpu.Arena(0)
c.load(lpt)
c.run(); c.synchronize(); c.reset(); c.run(); c.synchronize()
print("longest-first full:", c.last_run_ms(), "ms")
