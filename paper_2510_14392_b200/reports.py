"""Per-request reports and scenario aggregates from device records
(metrics.h:29-102, metrics.cpp:60-205).

The device builds each RequestReport online (fb_record); this module turns
them into the reference's aggregates: nearest-rank percentiles
(metrics.cpp:118-135) and ScenarioReport (metrics.cpp:171-205).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi


@dataclass
class PercentileRow:
    p50: float = 0.0
    p95: float = 0.0
    p99: float = 0.0
    count: int = 0


def percentiles(values) -> PercentileRow:
    """Nearest-rank percentiles, metrics.cpp:118-135."""
    v = np.sort(np.asarray(values, np.float64))
    n = len(v)
    row = PercentileRow(count=n)
    if n == 0:
        return row

    def rank(p):
        r = int(math.ceil(p / 100.0 * n))
        return v[min(max(r, 1), n) - 1]

    row.p50, row.p95, row.p99 = float(rank(50.0)), float(rank(95.0)), float(rank(99.0))
    return row


@dataclass
class ScenarioReport:
    """metrics.h:74-88."""

    name: str = ""
    total_requests: int = 0
    rejected: int = 0
    finished: int = 0
    good: int = 0
    slo_violation_rate: float = 0.0
    offered_rps: float = 0.0
    effective_rps: float = 0.0
    ttft: PercentileRow = field(default_factory=PercentileRow)
    max_tpot: PercentileRow = field(default_factory=PercentileRow)
    max_tpot_alt: PercentileRow = field(default_factory=PercentileRow)
    ttft_violations: int = 0     # no first token or emits[0] > ttft (acceptance.cpp:105)
    envelope_misses: int = 0     # some token j>=1 past its envelope (acceptance.cpp:106-111)


def good_mask(rec: np.ndarray) -> np.ndarray:
    """RequestReport::good (metrics.h:48)."""
    f = rec["flags"]
    need = _abi.REC_FINISHED | _abi.REC_MET_TTFT | _abi.REC_MET_TPOT
    return ((f & need) == need) & ((f & _abi.REC_REJECTED) == 0)


def scenario_report(records: np.ndarray, arrival_us: np.ndarray, offered: float, name: str = "",
                    alt_tpot: bool = False) -> ScenarioReport:
    """scenario_report (metrics.cpp:171-205) over the requests that arrived."""
    f = records["flags"]
    arrived = (f & _abi.REC_ARRIVED) != 0
    rec = records[arrived]
    arr = np.asarray(arrival_us)[arrived]
    rep = ScenarioReport(name=name, offered_rps=offered)
    rep.total_requests = int(arrived.sum())
    ff = rec["flags"]
    rep.rejected = int(((ff & _abi.REC_REJECTED) != 0).sum())
    rep.finished = int(((ff & _abi.REC_FINISHED) != 0).sum())
    rep.good = int(good_mask(rec).sum())
    frac = 0.0 if rep.total_requests == 0 else rep.good / rep.total_requests
    rep.slo_violation_rate = 1.0 - frac
    rep.effective_rps = offered * frac
    has_ttft = rec["tokens_emitted"] >= 1
    rep.ttft = percentiles((rec["first_emit_us"][has_ttft] - arr[has_ttft]) / 1000.0)
    rep.max_tpot = percentiles(rec["max_tpot_ms"][rec["tokens_emitted"] >= 2])
    if alt_tpot:
        rep.max_tpot_alt = percentiles(rec["max_tpot_alt_ms"][rec["tokens_emitted"] >= 3])
    rep.ttft_violations = int((~has_ttft | ((ff & _abi.REC_MET_TTFT) == 0)).sum())
    rep.envelope_misses = int(((ff & _abi.REC_ENV_MISS) != 0).sum())
    return rep


def goodput(records: np.ndarray, offered: float) -> float:
    """offered * good / max(1, reports) as in acceptance.cpp:118-119."""
    arrived = (records["flags"] & _abi.REC_ARRIVED) != 0
    n = max(1, int(arrived.sum()))
    return offered * float(good_mask(records[arrived]).sum()) / n


def summary_report(row, offered: float, name: str = "", alt_tpot: bool = False) -> ScenarioReport:
    """ScenarioReport from one device summary row (fb_arena_fetch_summaries):
    the counts and percentiles come from the device, the rates are the
    host arithmetic of scenario_report (metrics.cpp:190-196)."""
    rep = ScenarioReport(name=name, offered_rps=offered)
    rep.total_requests = int(row["total_requests"])
    rep.rejected = int(row["rejected"])
    rep.finished = int(row["finished"])
    rep.good = int(row["good"])
    frac = 0.0 if rep.total_requests == 0 else rep.good / rep.total_requests
    rep.slo_violation_rate = 1.0 - frac
    rep.effective_rps = offered * frac

    def pct(r):
        return PercentileRow(float(r["p50"]), float(r["p95"]), float(r["p99"]), int(r["count"]))

    rep.ttft = pct(row["ttft_ms"])
    rep.max_tpot = pct(row["max_tpot_ms"])
    if alt_tpot:
        rep.max_tpot_alt = pct(row["max_tpot_alt_ms"])
    rep.ttft_violations = int(row["ttft_violations"])
    rep.envelope_misses = int(row["envelope_misses"])
    return rep
