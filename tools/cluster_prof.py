"""Per-epoch phase split of the C5 cluster kernel (dev tool; CTA 0 thread 0 clock):
    tools/build_variant.sh cprof -DFB_CLUSTER_PROF
    FBGPU_LIB=build/variants/cprof/libfbgpu.so python tools/cluster_prof.py"""
import ctypes as C, sys
sys.path.insert(0, '.')
from paper_2510_14392_b200 import cluster, fbgpu
rows, cfgs, lb, hz = cluster.c5()
out = cluster.run_cluster(rows, cfgs, lb, hz)
b = (C.c_ulonglong * 8)()
fbgpu.lib().fb_debug_cluster_prof(b)
out = cluster.run_cluster(rows, cfgs, lb, hz)
fbgpu.lib().fb_debug_cluster_prof(b)
e = b[5]
names = ["phase A (own node)", "barrier wait", "reports + stop test", "routing", "phase C (own node)"]
print("device ms", out.device_ms, "epochs", e)
for k, n in enumerate(names):
    print(f"  {n:22s} {b[k] / 1e6:8.2f} ms  {b[k] / max(e, 1) / 1000:6.2f} us/epoch")
# per epoch: the slowest node's work since the previous routing (phase C of
# the previous epoch + phase A of this one), against the mean node's
b7 = b[7]
em = (C.c_ulonglong * 32768)()
fbgpu.lib().fb_debug_epoch_max(em)   # first run's values: reset
out = cluster.run_cluster(rows, cfgs, lb, hz)
fbgpu.lib().fb_debug_cluster_prof(b)
fbgpu.lib().fb_debug_epoch_max(em)
import numpy as np
m = np.array(em[:min(e, 16384)], dtype=np.float64)
mc = np.array(em[16384:16384 + min(e, 16384)], dtype=np.float64)
print(f"  slowest phase C per epoch: mean {mc.mean()/1000:6.2f} us, p50 {np.median(mc)/1000:6.2f}, p90 {np.percentile(mc, 90)/1000:6.2f}")
print(f"  slowest node per epoch: mean {m.mean()/1000:6.2f} us, p50 {np.median(m)/1000:6.2f}, "
      f"p90 {np.percentile(m, 90)/1000:6.2f}, max {m.max()/1000:8.2f}; "
      f"mean node {b[7] / max(e, 1) / 64 / 1000:6.2f} us/epoch")
