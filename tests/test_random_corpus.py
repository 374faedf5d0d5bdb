"""Randomized engine corpus (tests/random_corpus.py): the C oracle against the
compiled reference on CPU, and the CUDA engines against the oracle on the GPU
-- per-instance plan digests, counters and per-request records byte for byte,
and with event logs every step and plan entry.
"""
from __future__ import annotations

import pytest

from backends import cluster_summary
from full_size import canonical_results
from random_corpus import random_batch, random_cluster
from paper_2510_14392_b200 import _abi


@pytest.mark.parametrize("seed", [11, 12])
def test_oracle_matches_reference_on_random_corpus(oracle, ref, seed):
    batch = random_batch(seed, 40)
    a = oracle.run(batch, nthreads=4)
    b = ref.run(batch, nthreads=4, check=True)  # mirrored plans checked against run_node
    assert (canonical_results(a.results) == canonical_results(b.results)).all()
    assert a.records.tobytes() == b.records.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_gpu_matches_oracle_on_random_corpus(fb, oracle, seed):
    """No logs: the register / memory paths with runs of repeated plans."""
    batch = random_batch(seed, 150)
    arena = fb.Arena(0)
    arena.load(batch)
    arena.run()
    res, rec, paths = arena.results(), arena.records(), arena.paths()
    arena.close()
    want = oracle.run(batch, nthreads=8)
    for i in range(batch.n_instances):
        assert res[i].tobytes() == want.results[i].tobytes(), i
    assert rec.tobytes() == want.records.tobytes()
    assert (paths & 8).any()  # FB_PATH_REPEAT_REGISTER: the repeated-plan runs did run


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [5, 6])
def test_gpu_logs_match_oracle_on_random_corpus(fb, oracle, seed):
    """With event logs: every step and plan entry (the per-event lanes)."""
    batch = random_batch(seed, 60)
    lo = _abi.LogOpts(40_000, 200_000, 1_000, 0)
    arena = fb.Arena(0)
    arena.load(batch, lo)
    arena.run()
    res, rec = arena.results(), arena.records()
    counts, steps, entries, rejects = arena.logs()
    arena.close()
    want = oracle.run(batch, lo, nthreads=8)
    assert counts.tobytes() == want.counts.tobytes()
    assert not counts["truncated"].any()
    for i in range(batch.n_instances):
        c = counts[i]
        assert steps[i][: c["steps"]].tobytes() == want.steps[i][: c["steps"]].tobytes(), i
        assert entries[i][: c["entries"]].tobytes() == want.entries[i][: c["entries"]].tobytes(), i
        assert rejects[i][: c["rejects"]].tobytes() == want.rejects[i][: c["rejects"]].tobytes(), i
    assert res.tobytes() == want.results.tobytes()
    assert rec.tobytes() == want.records.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [7, 8])
def test_gpu_wide_random_corpus_matches_oracle(fb, oracle, seed):
    """Thousands of live requests per instance: the grid-wide engine."""
    batch = random_batch(seed, 8, wide=True)
    arena = fb.Arena(0)
    arena.load(batch)
    arena.run()
    res, rec, paths = arena.results(), arena.records(), arena.paths()
    arena.close()
    want = oracle.run(batch, nthreads=8)
    for i in range(batch.n_instances):
        assert res[i].tobytes() == want.results[i].tobytes(), i
    assert rec.tobytes() == want.records.tobytes()
    assert (paths & 4).any()  # FB_PATH_WIDE


@pytest.mark.parametrize("seed", [300, 301, 302, 303, 305, 306])
def test_oracle_cluster_matches_reference_on_random_cases(oracle, ref, seed):
    rows, cfgs, lb, hz = random_cluster(seed)
    assert cluster_summary(oracle.run_cluster(rows, cfgs, lb, hz)) == \
        cluster_summary(ref.run_cluster(rows, cfgs, lb, hz, check=True))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(300, 312))
def test_gpu_cluster_matches_oracle_on_random_cases(oracle, seed):
    from paper_2510_14392_b200 import cluster
    rows, cfgs, lb, hz = random_cluster(seed)
    assert cluster_summary(cluster.run_cluster(rows, cfgs, lb, hz)) == \
        cluster_summary(oracle.run_cluster(rows, cfgs, lb, hz))
