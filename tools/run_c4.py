"""C4 (decode-heavy, 120k live requests per instance) on the GPU."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14392_b200 import fbgpu, workloads  # noqa: E402

n_inst = int(sys.argv[1]) if len(sys.argv) > 1 else 64
batch = workloads.c4_batch(n_inst=n_inst)
a = fbgpu.Arena(0)
a.load(batch)
for rep in range(3):
    a.reset()
    a.run()
    a.synchronize()
    print(f"rep {rep}: {a.last_run_ms():.2f} ms")
r = a.results()
print("steps", r["steps"][:4], "total", int(r["steps"].sum()), "paths", np.unique(a.paths()))
print("mean A", (r["sum_visible"] / r["steps"]).mean(), "mean E", (r["sum_entries"] / r["steps"]).mean())
alg = 32 * r["sum_visible"].sum() + 64 * r["sum_entries"].sum() + 64 * r["n_arrived"].sum()
ms = a.last_run_ms()
print(f"steps/s {r['steps'].sum() / (ms / 1e3):.3e}  alg GB/s {alg / (ms / 1e3) / 1e9:.1f}")
np.save("gpurun_out/c4_results.npy", r)
