"""C4 pass time and wide-engine phase split (dev tool):
FBGPU_LIB=... python tools/c4_phases.py [reps]"""
import hashlib
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14392_b200 import fbgpu, workloads  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
batch = workloads.c4_batch(n_inst=64)
a = fbgpu.Arena(0)
a.load(batch)
tot, ph = [], []
for k in range(reps + 1):
    a.reset()
    a.run()
    a.synchronize()
    if k:
        w, g = a.last_run_split_ms()
        tot.append(w + g)
        ph.append(a.wide_phases()[0])
r = a.results()
h = hashlib.sha1(r.tobytes()).hexdigest()[:12]
med = {k: statistics.median(p[k] for p in ph) for k in ph[0]}
print(f"{os.environ.get('FBGPU_LIB', 'default')}: {statistics.median(tot):.3f} ms "
      + " ".join(f"{k}={v:.3f}" for k, v in med.items()) + f" digest {h} {a.wide_selection()}")
