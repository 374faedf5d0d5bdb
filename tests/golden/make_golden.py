"""Generates tests/golden/golden.json from the UNMODIFIED reference library.

Run in a container that has /root/reference (the library is built by
`make -C oracle ref` into oracle/_ref/libfbsim_ref.so):

    python tests/golden/make_golden.py

The fixtures pin the C oracle (CPU tests) and the CUDA path (GPU tests):
trace checksums of generate_bursty, exact run summaries (plan digest, step
counts, per-request record hashes) of the catalogue scenarios, and hashes of
the batch plans / PAB values over the reference test-suite fuzz corpora.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

from backends import RefLib, cluster_summary  # noqa: E402
from catalog import (SCENARIOS, TRACE_PROFILES, cluster_cases, reroute_cluster_cases,  # noqa: E402
                     rows_digest, summarize)
from fuzz import Rng, acceptance_corpus, gen_pab_instance, raw_to_views  # noqa: E402
from tests_golden_cases import (CLUSTER_LOG_CASES, LEAD_CASES, REPLAY_MUTATIONS,  # noqa: E402
                                replay_canonical)
from paper_2510_14392_b200.batch import ms_to_us  # noqa: E402


def plans_digest(lib, corpus) -> str:
    h = hashlib.sha256()
    for v, cfg in corpus:
        plan, entries = lib.form_batch(v, cfg)
        h.update(plan.tobytes())
        h.update(entries.tobytes())
    return h.hexdigest()


def pab_values(lib, n=1000, seed=424242):
    rng = Rng(seed)
    out = []
    for _ in range(n):
        raw, cfg, now = gen_pab_instance(rng, 8)
        v = raw_to_views(raw, now)
        tt = ms_to_us(rng.uniform(300.0, 2000.0))
        tp = ms_to_us(rng.uniform(25.0, 100.0))
        out.append(lib.pab(v, cfg.model, tt, tp))
    return out


def main() -> None:
    ref = RefLib()
    gold = {"source": "oracle/_ref/libfbsim_ref.so (unmodified /root/reference/proj/src)"}
    gold["traces"] = {}
    for name, (prof, h_ms) in TRACE_PROFILES.items():
        rows = ref.generate_bursty(prof, ms_to_us(h_ms))
        gold["traces"][name] = {"n": len(rows), "sha256": rows_digest(rows),
                                "head_arrival_us": rows.arrival_us[:4].tolist(),
                                "head_prompt": rows.prompt_len[:4].tolist()}
    gold["scenarios"] = {}
    for name, fn in SCENARIOS.items():
        batch = fn(ref.generate_bursty)
        out = ref.run(batch, nthreads=8, check=True)
        gold["scenarios"][name] = summarize(out.results, out.records)
    gold["event_logs"] = {}
    for name in ("c1", "pab_overload", "wide"):
        batch = SCENARIOS[name](ref.generate_bursty)
        gold["event_logs"][name] = [
            hashlib.sha256(ref.event_log(batch, i, "/tmp/_golden_ev.jsonl").encode()).hexdigest()
            for i in range(batch.n_instances)]
    # the reference's replay_check on mutations of its own event log
    batch = SCENARIOS["pab_overload"](ref.generate_bursty)
    base = ref.event_log(batch, 0, "/tmp/_golden_ev.jsonl").rstrip("\n").split("\n")
    gold["replay_check"] = {}
    for name, fn in REPLAY_MUTATIONS.items():
        v = replay_canonical(ref.replay_check("\n".join(fn(base)) + "\n", "/tmp/_golden_rc.jsonl"))
        gold["replay_check"][name] = {"n": len(v), "head": v[:3],
                                      "sha256": hashlib.sha256("\n".join(v).encode()).hexdigest()}
    gold["lead"] = {}
    for name, bucket_ms in LEAD_CASES.items():
        batch = SCENARIOS[name](ref.generate_bursty)
        gold["lead"][name] = [
            hashlib.sha256(ref.lead_series(batch, i, ms_to_us(bucket_ms)).tobytes()).hexdigest()
            for i in range(batch.n_instances)]
    import acceptance_cases as ac

    def ref_runner(b):
        o = ref.run_node_batch(b, nthreads=8)
        return o.results, o.records

    gold["acceptance"] = {
        "crit67": ac.crit67(ref.generate_bursty, ref_runner),
        "crit8": ac.crit8(ref.generate_bursty, ref_runner),
        "crit9": ac.crit9(ref.generate_bursty,
                          lambda r, c, lb, h: ref.run_cluster(r, c, lb, h).records),
    }
    gold["clusters"] = {}
    for name, rows, cfgs, lb, hz in (cluster_cases(ref.generate_bursty) +
                                     reroute_cluster_cases(ref.generate_bursty)):
        gold["clusters"][name] = cluster_summary(ref.run_cluster(rows, cfgs, lb, hz, check=True))
    cl = {c[0]: c for c in cluster_cases(ref.generate_bursty) +
          reroute_cluster_cases(ref.generate_bursty)}
    gold["cluster_logs"] = {}
    for name in CLUSTER_LOG_CASES:
        _, rows, cfgs, lb, hz = cl[name]
        nodes, routing = ref.cluster_logs(rows, cfgs, lb, hz, "/tmp/_golden_cl.jsonl")
        gold["cluster_logs"][name] = {
            "nodes": [hashlib.sha256(x.encode()).hexdigest() for x in nodes],
            "routing": hashlib.sha256(routing.encode()).hexdigest()}
    corpus = acceptance_corpus(10_000)
    gold["fuzz"] = {}
    for pol in (2, 1, 0):
        for _, cfg in corpus:
            cfg.policy = pol
        gold["fuzz"][f"acceptance_policy{pol}"] = plans_digest(ref, corpus)
    from fuzz import degenerate_corpus
    gold["fuzz"]["degenerate_77001"] = plans_digest(ref, degenerate_corpus())
    gold["fuzz"]["pab_424242"] = hashlib.sha256(
        np.asarray(pab_values(ref), np.int64).tobytes()).hexdigest()
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(gold, f, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
