"""Full-size parity fixtures: the UNMODIFIED reference (oracle/_ref) on the
BASELINE.json configurations at their stated sizes, written to
tests/golden/full_size.json.  TEST INFRASTRUCTURE ONLY.

    python tests/golden/make_golden_full.py [--only c2_full,c3_sample,...]

Traces are materialised with the reference's own generate_bursty /
scale_trace (workload.cpp:211-298).  Every run goes through
ref_run_instances, the Node-API mirror of run_node (engine.cpp:266-288) that
records each plan for the per-instance digest; `--check` additionally
verifies every mirrored event log against the real run_node (slow: C3 full
takes ~10 min on 8 host threads with it, ~5 min without).

Fixture layout per config: instances are cut into chunks of `chunk`
instances; per chunk the sha256 of the canonical results array (the
RESULT_KEYS columns as int64, instance order) and of the chunk's packed
per-request records, plus totals.  A mismatch therefore names the chunk (for
C3: the trace seed), and the GPU test re-runs only that chunk on the
reference to name the instance.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from backends import RefLib  # noqa: E402
from full_size import CONFIGS, chunk_digests  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    ref = RefLib()
    path = os.path.join(HERE, "full_size.json")
    gold = {}
    if os.path.exists(path):
        with open(path) as f:
            gold = json.load(f)
    gold["source"] = "oracle/_ref/libfbsim_ref.so (unmodified /root/reference/proj/src)"
    only = [x for x in args.only.split(",") if x]
    for name, spec in CONFIGS.items():
        if only and name not in only:
            continue
        t0 = time.time()
        batch = spec["build"](ref)
        out = ref.run(spec["ref_batch"](batch) if "ref_batch" in spec else batch,
                      nthreads=args.threads, check=args.check)
        res, rec = out.results, out.records
        if "expand" in spec:  # identical instances: the reference runs one
            res, rec = spec["expand"](batch, res, rec)
        gold[name] = chunk_digests(batch, res, rec, spec["chunk"])
        gold[name]["description"] = spec["description"]
        gold[name]["checked_against_run_node"] = bool(args.check)
        print(f"{name}: {batch.n_instances} instances, {gold[name]['total_steps']} steps, "
              f"{time.time() - t0:.1f} s", flush=True)
        with open(path, "w") as f:
            json.dump(gold, f, indent=1, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
