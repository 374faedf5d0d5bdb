"""Randomized cluster stress (dev tool): random traces, node counts, node
policies / budgets / cost models, load balancers, report intervals and
latencies, with and without retry_reroute -- the device run_cluster against
the C oracle's run_cluster (pinned to the reference), node results, records
and routing compared exactly.  python tools/random_cluster_stress.py [seed0] [n]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from backends import OracleLib, cluster_summary  # noqa: E402  (test infrastructure)
from random_corpus import random_cluster  # noqa: E402
from paper_2510_14392_b200 import cluster  # noqa: E402

s0 = int(sys.argv[1]) if len(sys.argv) > 1 else 300
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
oracle = OracleLib()
bad = 0
t0 = time.time()
steps = 0
for seed in range(s0, s0 + n):
    rows, cfgs, lb, hz = random_cluster(seed)
    got = cluster.run_cluster(rows, cfgs, lb, hz)
    want = oracle.run_cluster(rows, cfgs, lb, hz)
    steps += int(got.node_results["steps"].sum())
    if cluster_summary(got) != cluster_summary(want):
        bad += 1
        print("MISMATCH seed", seed, len(cfgs), lb, flush=True)
print(f"random cluster stress: seeds {s0}..{s0 + n - 1}, {steps} node-steps, mismatches {bad}, "
      f"{time.time() - t0:.0f} s")
