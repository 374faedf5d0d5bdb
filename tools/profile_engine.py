"""One engine pass over a workload, for ncu (kernel-only capture).

    ncu --set full -k regex:engine_kernel -c 1 -o out python tools/profile_engine.py [c2|c1|c3]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14392_b200 import fbgpu, workloads  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
if which == "c2":
    batch = workloads.c2_batch(n_seeds=n or 2048)
elif which == "c1":
    batch = workloads.c1_batch(("fairbatch",))
elif which == "c3":
    batch = workloads.c3_batch(n_seeds=n or 4)
else:
    raise SystemExit(which)
a = fbgpu.Arena(0)
a.load(batch)
a.run()
a.synchronize()
r = a.results()
print(which, batch.n_instances, "instances", int(r["steps"].sum()), "steps", a.last_run_ms(), "ms")

if which == "c2" and len(sys.argv) > 3 and sys.argv[3] == "top":
    import numpy as np
    order = np.argsort(-r["steps"].astype(np.int64))
    sub = batch.subset(order[: int(sys.argv[4]) if len(sys.argv) > 4 else 1].tolist())
    b = fbgpu.Arena(0)
    b.load(sub)
    b.run()
    b.synchronize()
    print("top subset", sub.n_instances, b.last_run_ms(), "ms")
