"""Randomized engine stress (dev tool): tests/random_corpus.py batches for many
seeds, GPU (C ABI) against the C oracle (pinned to the reference), results and
records byte for byte.  python tools/random_stress.py [first_seed] [n_seeds] [n_inst] [wide]
(wide: thousands of live requests per instance -- the grid-wide engine)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from backends import OracleLib  # noqa: E402  (test infrastructure: the checker)
from random_corpus import random_batch  # noqa: E402
from paper_2510_14392_b200 import fbgpu  # noqa: E402

s0 = int(sys.argv[1]) if len(sys.argv) > 1 else 100
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ni = int(sys.argv[3]) if len(sys.argv) > 3 else 150
wide = len(sys.argv) > 4 and sys.argv[4] == "wide"
oracle = OracleLib()
bad = 0
tot_inst = tot_steps = 0
paths_or = 0
t0 = time.time()
for seed in range(s0, s0 + ns):
    b = random_batch(seed, ni, wide=wide)
    a = fbgpu.Arena(0)
    a.load(b)
    a.run()
    res, rec, paths = a.results(), a.records(), a.paths()
    a.close()
    want = oracle.run(b, nthreads=16)
    ok = res.tobytes() == want.results.tobytes() and rec.tobytes() == want.records.tobytes()
    bad += not ok
    tot_inst += b.n_instances
    tot_steps += int(res["steps"].sum())
    paths_or |= int(paths.max()) if len(paths) else 0
    for p in paths:
        paths_or |= int(p)
    if not ok:
        print("MISMATCH seed", seed, flush=True)
print(f"random stress{' (wide)' if wide else ''}: seeds {s0}..{s0 + ns - 1}, {tot_inst} instances, {tot_steps} steps, "
      f"paths used {paths_or:#x}, mismatches {bad}, {time.time() - t0:.0f} s")
