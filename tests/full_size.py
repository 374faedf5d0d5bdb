"""BASELINE.json configurations at their stated sizes, for full-size parity
(TEST INFRASTRUCTURE ONLY).  Shared by the fixture generator
(tests/golden/make_golden_full.py, which runs the unmodified reference) and
the GPU tests (tests/test_full_size.py, which run the CUDA path).

Each config builds its batch from a trace library `lib` that has
`generate_bursty(profile, horizon_us) -> Rows` and `scale_trace(arrival,
factor)`: RefLib for the fixtures, the product's fbgpu for the GPU runs (the
two generators are pinned equal by the trace fixtures of golden.json).
"""
from __future__ import annotations

import hashlib

import numpy as np

from catalog import wide_rows
from paper_2510_14392_b200 import workloads
from paper_2510_14392_b200.batch import Batch, CostModel, Rows, engine_config, ms_to_us

# the exact per-instance outcome fields every backend computes (the
# reference's mirror does not count visible tasks: sum_visible is -1 there)
RESULT_KEYS = ("steps", "plan_digest", "end_time_us", "n_arrived", "n_rejected", "sum_entries",
               "sum_new_tokens", "incomplete")


def canonical_results(res: np.ndarray) -> np.ndarray:
    return np.stack([res[k].astype(np.int64) for k in RESULT_KEYS], axis=1)


def chunk_digests(batch: Batch, res: np.ndarray, rec: np.ndarray, chunk: int) -> dict:
    """sha256 per `chunk` instances of the canonical results and of the
    chunk's per-request records, plus totals."""
    off = batch.record_offsets()
    can = canonical_results(res)
    n = batch.n_instances
    r = batch.rows
    h = hashlib.sha256()
    for a in (r.arrival_us, r.prompt_len, r.output_len, r.ttft_us, r.tpot_us):
        h.update(np.ascontiguousarray(a).tobytes())
    out = {"n_instances": n, "chunk": chunk, "rows_sha256": h.hexdigest(),
           "total_steps": int(res["steps"].sum()),
           "total_rejected": int(res["n_rejected"].sum()),
           "total_incomplete": int(res["incomplete"].sum()), "results_sha256": [],
           "records_sha256": []}
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        out["results_sha256"].append(hashlib.sha256(can[c0:c1].tobytes()).hexdigest())
        out["records_sha256"].append(
            hashlib.sha256(rec[off[c0]:off[c1]].tobytes()).hexdigest())
    return out


def _gen(lib):
    return lib.generate_bursty


def _scale(lib):
    def scale(rows: Rows, f: float) -> Rows:
        if hasattr(lib, "scale_trace") and not hasattr(lib, "Arena"):  # RefLib: arrays
            arr = lib.scale_trace(rows.arrival_us, f)
            return Rows(arr, rows.prompt_len, rows.output_len, rows.ttft_us, rows.tpot_us)
        return lib.scale_trace(rows, f)  # fbgpu: Rows
    return scale


def c2_full(lib) -> Batch:
    """C2 as benchmarked: seeds 0..2047 x {sarathi 512, fairbatch 2048}."""
    return workloads.c2_batch(n_seeds=2048, gen=_gen(lib), scale=_scale(lib))


def c3_sample(lib) -> Batch:
    """One trace seed of C3: every scale x SLO pair x policy (1,024 instances)."""
    return workloads.c3_batch(n_seeds=1, gen=_gen(lib), scale=_scale(lib))


def c3_full(lib) -> Batch:
    """C3 at its stated size: 64 trace seeds x 16 scales x 16 SLO pairs x 4
    policies = 65,536 instances."""
    return workloads.c3_batch(n_seeds=64, gen=_gen(lib), scale=_scale(lib))


def c4_full(lib) -> Batch:
    """C4 as benchmarked: 64 nodes x 120,000 requests (identical instances)."""
    return workloads.c4_batch(n_inst=64)


def _c4_expand(batch: Batch, res: np.ndarray, rec: np.ndarray):
    n = batch.n_instances
    return np.repeat(res[:1], n), np.tile(rec, n)


def c4_variants(lib) -> Batch:
    """120,000 live requests per instance under every policy and engine
    option: PAB admission, Sarathi chunking, prefill-first, noise,
    max_active, a binding token budget, and varied lengths."""
    b = Batch()
    rows = workloads.c4_rows()
    m = CostModel(5.0, 0.01, 1e-6)
    hz = ms_to_us(1500.0)
    for cfg in (engine_config("fairbatch_pab", 1 << 20, m, 500, 50),
                engine_config("sarathi", 512, m, 500, 50),
                engine_config("prefill_first", 8192, m, 500, 50),
                engine_config("fairbatch", 1 << 20, m, 500, 50, noise_amplitude=0.05,
                              noise_seed=3),
                engine_config("fairbatch", 1 << 20, m, 500, 50, max_active=50_000),
                engine_config("fairbatch", 8192, m, 500, 50)):
        b.add(rows, cfg, hz)
    vr = wide_rows(120_000, 8, 4)
    b.add(vr, engine_config("fairbatch", 1 << 20, m, 500, 50), hz)
    b.add(vr, engine_config("fairbatch_pab", 1 << 20, m, 300, 30), hz)
    return b


CONFIGS = {
    "c2_full": {"build": c2_full, "chunk": 256,
                "description": "C2 at 4,096 instances (the bench workload)"},
    "c3_sample": {"build": c3_sample, "chunk": 64,
                  "description": "C3 trace seed 0: 16 scales x 16 SLO pairs x 4 policies"},
    "c3_full": {"build": c3_full, "chunk": 1024,
                "description": "C3 at 65,536 instances (chunk = one trace seed)"},
    "c4_full": {"build": c4_full, "chunk": 64,
                "ref_batch": lambda b: b.subset([0]), "expand": _c4_expand,
                "description": "C4 at 64 x 120,000 requests (identical instances: the "
                               "reference runs one, the fixture repeats it)"},
    "c4_variants": {"build": c4_variants, "chunk": 1,
                    "description": "120,000-request instances under every policy/option"},
}
