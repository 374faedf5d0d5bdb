"""Fuzz corpora of the reference test suite, regenerated bit-for-bit in Python.

`Rng` restates fbsim's splitmix64 generator (rng.h:25-86) and `gen_instance`
/ `gen_pab_instance` restate testutil.h:23-82 / raw_to_views
(reference_alg.cpp:22-39), so the acceptance corpus (seed 20260808,
acceptance.cpp:125-180) is reproduced exactly without the C++ test harness.
"""
from __future__ import annotations

import numpy as np

from paper_2510_14392_b200 import _abi
from paper_2510_14392_b200.batch import ms_to_us

M64 = (1 << 64) - 1


class Rng:
    def __init__(self, seed: int):
        self.s = seed & M64

    def next_u64(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def next_double(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.next_double()

    def uniform_int(self, lo: int, hi: int) -> int:
        span = ((hi - lo) & M64) + 1
        return lo + (self.next_u64() % span)


def gen_instance(rng: Rng, max_tasks: int):
    """testutil.h:23-63 -> (raw task dicts, scheduler config dict, now)."""
    now = ms_to_us(10_000.0)
    n = rng.uniform_int(1, max_tasks)
    raw = []
    for i in range(n):
        t = {"id": i, "seq": i}
        t["ttft"] = ms_to_us(rng.uniform(200.0, 2000.0))
        t["tpot"] = ms_to_us(rng.uniform(20.0, 200.0))
        t["decode"] = rng.next_double() < 0.5
        if t["decode"]:
            t["nidx"] = rng.uniform_int(1, 200)
            t["new"] = 1
            t["ctx"] = rng.uniform_int(50, 4000)
        else:
            t["nidx"] = 0
            t["new"] = rng.uniform_int(1, 30_000)
            t["ctx"] = rng.uniform_int(0, 4000)
        target = ms_to_us(rng.uniform(-300.0, 800.0))
        t["arrival"] = now + target - t["ttft"] - t["tpot"] * t["nidx"]
        t["first"] = -1
        if t["decode"]:
            fe = t["arrival"] + t["ttft"] + ms_to_us(rng.uniform(-400.0, 200.0))
            t["first"] = max(fe, t["arrival"])
        raw.append(t)
    a = rng.uniform(1.0, 10.0)
    b = rng.uniform(0.005, 0.03)
    c = rng.uniform(0.00003, 0.0003)
    budget = (256, 512, 2048, 8192)[rng.uniform_int(0, 3)]
    cfg = _abi.SchedulerConfig(_abi.POLICY_FAIRBATCH, budget, budget, _abi.CostModel(a, b, c))
    return raw, cfg, now


def gen_pab_instance(rng: Rng, max_tasks: int):
    """testutil.h:68-82."""
    raw, cfg, now = gen_instance(rng, max_tasks)
    cfg.model.a_ms = rng.uniform(3.0, 8.0)
    cfg.model.b_ms = rng.uniform(0.01, 0.03)
    cfg.model.c_ms = rng.uniform(0.00002, 0.0001)
    for t in raw:
        t["ctx"] = rng.uniform_int(0, 2000)
        target = ms_to_us(rng.uniform(-100.0, 700.0))
        t["arrival"] = now + target - t["ttft"] - t["tpot"] * t["nidx"]
        if t["decode"]:
            t["first"] = t["arrival"] + t["ttft"]
    return raw, cfg, now


def raw_to_views(raw, now) -> np.ndarray:
    """reference_alg.cpp:22-39 (anchor: reference_alg.cpp:14-18)."""
    v = np.zeros(len(raw), _abi.TASKVIEW_DTYPE)
    for i, t in enumerate(raw):
        anchor = t["arrival"] + t["ttft"]
        if t["decode"] and t["first"] >= 0:
            anchor = min(anchor, t["first"])
        v[i]["request_id"] = t["id"]
        v[i]["phase"] = _abi.PHASE_DECODE if t["decode"] else _abi.PHASE_PREFILL
        v[i]["slack_us"] = anchor + t["tpot"] * t["nidx"] - now
        v[i]["new_tokens"] = t["new"]
        v[i]["context"] = t["ctx"]
        v[i]["arrival_seq"] = t["seq"]
        v[i]["tpot_us"] = t["tpot"]
    return v


def acceptance_corpus(n: int = 10_000, seed: int = 20260808, max_tasks: int = 32,
                      policy: int | None = None):
    """Criterion 1's corpus (acceptance.cpp:127-134): list of (views, cfg)."""
    rng = Rng(seed)
    out = []
    for _ in range(n):
        raw, cfg, now = gen_instance(rng, max_tasks)
        if policy is not None:
            cfg.policy = policy
        out.append((raw_to_views(raw, now), cfg))
    return out


def decode_task(tid, slack_ms, context, tpot_ms=50.0, seq=-1):
    """test_sched.cpp:17-28."""
    v = np.zeros(1, _abi.TASKVIEW_DTYPE)[0]
    v["request_id"] = tid
    v["phase"] = _abi.PHASE_DECODE
    v["slack_us"] = ms_to_us(slack_ms)
    v["new_tokens"] = 1
    v["context"] = context
    v["arrival_seq"] = tid if seq < 0 else seq
    v["tpot_us"] = ms_to_us(tpot_ms)
    return v


def prefill_task(tid, slack_ms, tokens, context=0, tpot_ms=50.0, seq=-1):
    """test_sched.cpp:30-42."""
    v = np.zeros(1, _abi.TASKVIEW_DTYPE)[0]
    v["request_id"] = tid
    v["phase"] = _abi.PHASE_PREFILL
    v["slack_us"] = ms_to_us(slack_ms)
    v["new_tokens"] = tokens
    v["context"] = context
    v["arrival_seq"] = tid if seq < 0 else seq
    v["tpot_us"] = ms_to_us(tpot_ms)
    return v


def views(*tasks) -> np.ndarray:
    return np.array(list(tasks), dtype=_abi.TASKVIEW_DTYPE)


K_MODEL = _abi.CostModel(5.0, 0.01, 0.0001)  # test_sched.cpp:44


def fb_config(token_budget=8192, policy=_abi.POLICY_FAIRBATCH, max_chunk=None):
    """test_sched.cpp:46-53."""
    return _abi.SchedulerConfig(policy, token_budget if max_chunk is None else max_chunk,
                                token_budget, _abi.CostModel(5.0, 0.01, 0.0001))


def degenerate_corpus(n: int = 5_000, seed: int = 77_001, max_tasks: int = 40):
    """Task sets outside what the engines produce, for the pure scheduler
    boundary (fb_form_batch vs form_batch, sched.cpp:129-246): zero-token
    tasks (which fair batching's `consider` admits as {id, 0} whenever
    c*ctx <= time_budget, even once the token budget is spent), negative
    contexts, tiny token budgets and c = 0.  List of (views, cfg), the
    policy cycling prefill_first / sarathi / fairbatch / fairbatch_pab."""
    rng = Rng(seed)
    out = []
    for i in range(n):
        raw, cfg, now = gen_instance(rng, max_tasks)
        for t in raw:
            if rng.next_double() < 0.25:
                t["new"] = 0
            if rng.next_double() < 0.1:
                t["ctx"] = -rng.uniform_int(1, 5000)
        budget = (1, 2, 8, 64, 256, 2048)[rng.uniform_int(0, 5)]
        cfg.token_budget = budget
        cfg.max_chunk = max(1, budget // (1 + rng.uniform_int(0, 3)))
        if rng.next_double() < 0.2:
            cfg.model.c_ms = 0.0
        cfg.policy = i % 4
        out.append((raw_to_views(raw, now), cfg))
    return out
