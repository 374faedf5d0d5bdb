"""One C4 pass for ncu: ncu -k regex:wide_kernel python tools/profile_c4.py [n_inst]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14392_b200 import fbgpu, workloads  # noqa: E402

batch = workloads.c4_batch(n_inst=int(sys.argv[1]) if len(sys.argv) > 1 else 64)
a = fbgpu.Arena(0)
a.load(batch)
a.run()
a.synchronize()
print("c4", a.last_run_ms(), "ms", int(a.results()["steps"].sum()), "steps")
