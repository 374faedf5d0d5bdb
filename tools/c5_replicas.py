"""C5 replica throughput for several copy counts (dev tool):
FBGPU_LIB=... python tools/c5_replicas.py 1 16 24 33"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
from paper_2510_14392_b200 import cluster  # noqa: E402

rows, cfgs, lb, hz = cluster.c5()
for n in [int(x) for x in sys.argv[1:]] or [16]:
    cases = [(rows, cfgs, lb, hz)] * n
    cluster.run_clusters(cases)
    best = 1e30
    for _ in range(2):
        span = {}
        outs = cluster.run_clusters(cases, span=span)
        best = min(best, span["ms"])
    steps = sum(int(o.node_results["steps"].sum()) for o in outs)
    print(f"{os.environ.get('FBGPU_LIB', 'default')}: {n} copies {best:.1f} ms "
          f"{steps / best / 1e3:.2f} M node-steps/s")
