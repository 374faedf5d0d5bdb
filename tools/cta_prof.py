"""Per-CTA busy time of the wide engine's phases on C4 (dev tool):
tools/build_variant.sh prof -DFB_WIDE_PROF && FBGPU_LIB=build/variants/prof/libfbgpu.so \
    python tools/cta_prof.py
Prints, per phase (K1 views, K2a histogram, K2b gather, owner), the busy
clocks per CTA summed over one pass: min / median / max and the sum, next to
the phase wall time (CTA 0's phase clock)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14392_b200 import fbgpu, workloads  # noqa: E402

batch = workloads.c4_batch(n_inst=64)
a = fbgpu.Arena(0)
a.load(batch)
a.run()
a.synchronize()
L = fbgpu.lib()
buf = (C.c_ulonglong * 1024)()
sub = (C.c_ulonglong * 2048)()
L.fb_debug_cta_prof(buf, 1)
L.fb_debug_sub_prof(sub, 1)
a.reset()
a.run()
a.synchronize()
L.fb_debug_cta_prof(buf, 1)
L.fb_debug_sub_prof(sub, 1)
y = np.frombuffer(sub, np.uint64).reshape(256, 8)[:148].astype(np.float64) / 1.965e6
x = np.frombuffer(buf, np.uint64).reshape(256, 4)[:148].astype(np.float64) / 1.965e6  # ms @1965MHz
ph, it = a.wide_phases()
print("phases (CTA0 wall, ms):", {k: round(v, 3) for k, v in ph.items()}, "iterations", it)
for k, name in enumerate(("k1", "k2a_hist", "k2b_gather", "owner")):
    v = x[:, k]
    print(f"{name:11s} busy ms per CTA: min {v.min():.3f} med {np.median(v):.3f} "
          f"max {v.max():.3f} (argmax {int(v.argmax())})")
names = ("k2a setup", "k2a loop", "k2a flush", "k2a window", "k2b setup", "k2b loop")
for k, name in enumerate(names):
    v = y[:, k]
    print(f"{name:11s} ms per CTA: min {v.min():.3f} med {np.median(v):.3f} max {v.max():.3f}")
