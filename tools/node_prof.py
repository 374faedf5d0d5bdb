"""Per-node phase costs of the C5 cluster kernel (dev tool):
    tools/build_variant.sh nprof -DFB_CLUSTER_PROF -DFB_CLUSTER_NODE_PROF
    FBGPU_LIB=build/variants/nprof/libfbgpu.so python tools/node_prof.py"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14392_b200 import cluster, fbgpu  # noqa: E402

rows, cfgs, lb, hz = cluster.c5()
L = fbgpu.lib()
buf = (C.c_ulonglong * (512 * 8))()
cluster.run_cluster(rows, cfgs, lb, hz)
L.fb_debug_node_prof(buf)
cb = (C.c_ulonglong * 8)()
L.fb_debug_cluster_prof(cb)
out = cluster.run_cluster(rows, cfgs, lb, hz)
L.fb_debug_node_prof(buf)
L.fb_debug_cluster_prof(cb)
a = np.frombuffer(buf, dtype=np.uint64).reshape(512, 8)[: len(cfgs)].astype(np.float64) / 1965.0
ep = cb[5]
print(f"device {out.device_ms:.1f} ms, {ep} epochs")
for k, nm in enumerate(["phase A (own node)", "barrier wait", "reports + stop", "routing", "phase C"]):
    print(f"  CTA0 {nm:20s} {cb[k] / max(ep, 1) / 1000:6.2f} us/epoch")
steps = out.node_results["steps"].astype(np.float64)
print(f"per node (us): phase A total mean {a[:, 0].mean():.0f} max {a[:, 0].max():.0f}; "
      f"max single phase A {a[:, 7].max():.1f}")
nrep = a[:, 5] * 1965.0
nc = a[:, 6] * 1965.0
print(f"  report (node_pab): {a[:, 1].sum() / nrep.sum():.2f} us each, {nrep.sum():.0f} reports")
print(f"  complete: {a[:, 2].sum() / steps.sum():.2f} us per step; begin (phase A): "
      f"{a[:, 3].sum() / steps.sum():.2f} us per step")
print(f"  phase C: {a[:, 4].sum() / max(nc.sum(), 1):.2f} us each, {nc.sum():.0f}")
print(f"  per epoch, summed over nodes: phase A {a[:, 0].sum() / ep:.2f} us")
