"""Full-size parity: the CUDA path on the BASELINE.json configurations at their
stated sizes against fixtures of the unmodified reference
(tests/golden/full_size.json, made by tests/golden/make_golden_full.py).

Per chunk of instances the canonical per-instance outcome (step count, the
64-bit plan digest of every step's batch composition and step times, end
time, arrivals, rejects, entry and token totals, incomplete flag) and the
per-request records (TTFT, TPOT flags, max-TPOT bit patterns) must be
byte-identical.  A mismatching chunk is re-run on the reference (oracle/_ref,
when present) to name the first differing instance.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from backends import RefLib
from full_size import CONFIGS, canonical_results, chunk_digests

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "full_size.json")) as _f:
    GOLD = json.load(_f)


def _explain(name, batch, res, rec, chunk_idx, chunk):
    if not RefLib.available():
        return ""
    c0 = chunk_idx * chunk
    c1 = min(batch.n_instances, c0 + chunk)
    sub = batch.subset(range(c0, c1))
    ref = RefLib().run(sub, nthreads=os.cpu_count() or 1)
    can_g = canonical_results(res[c0:c1])
    can_r = canonical_results(ref.results)
    for i in range(c1 - c0):
        if not np.array_equal(can_g[i], can_r[i]):
            return f"; first differing instance {c0 + i}: gpu {can_g[i]} ref {can_r[i]}"
    return "; results equal on re-run, records differ"


@pytest.mark.gpu
@pytest.mark.parametrize("name", [n for n in CONFIGS])
def test_full_size_matches_reference(fb, name):
    if name not in GOLD:
        pytest.fail(f"fixture {name} missing: run tests/golden/make_golden_full.py")
    spec = CONFIGS[name]
    gold = GOLD[name]
    batch = spec["build"](fb)
    a = fb.Arena(0)
    try:
        a.load(batch)
        a.run()
        res, rec = a.results(), a.records()
    finally:
        a.close()
    assert (res["status"] == 0).all()
    got = chunk_digests(batch, res, rec, spec["chunk"])
    if "rows_sha256" in gold:
        assert got["rows_sha256"] == gold["rows_sha256"], "trace rows differ from the reference's"
    assert got["n_instances"] == gold["n_instances"]
    for k in ("total_steps", "total_rejected", "total_incomplete"):
        assert got[k] == gold[k], f"{name}: {k} {got[k]} != reference {gold[k]}"
    for c, (g, r) in enumerate(zip(got["results_sha256"], gold["results_sha256"])):
        if g != r:
            pytest.fail(f"{name}: chunk {c} results differ"
                        + _explain(name, batch, res, rec, c, spec["chunk"]))
    for c, (g, r) in enumerate(zip(got["records_sha256"], gold["records_sha256"])):
        assert g == r, f"{name}: chunk {c} per-request records differ"


def test_full_size_fixtures_present():
    """CPU: every full-size config has its reference fixture, made by the
    run_node-checked mirror, at the stated size."""
    sizes = {"c2_full": 4096, "c3_sample": 1024, "c3_full": 65536, "c4_full": 64}
    for name in CONFIGS:
        assert name in GOLD, name
        assert GOLD[name]["checked_against_run_node"], name
        if name in sizes:
            assert GOLD[name]["n_instances"] == sizes[name]
