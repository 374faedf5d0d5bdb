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
