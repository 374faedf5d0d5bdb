"""One C5 cluster run for ncu (-k regex:cluster_kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_14392_b200 import cluster  # noqa: E402

rows, cfgs, lb, hz = cluster.c5()
out = cluster.run_cluster(rows, cfgs, lb, hz)
print("c5", out.device_ms, "ms", int(out.node_results["steps"].sum()), "node-steps")
