"""Cluster-level simulation (run_cluster, cluster.h:107-109) on the device.

`LbConfig` mirrors cluster.h:36-47; `run_cluster` calls fb_run_cluster; `c5`
builds BASELINE config 5 (64 nodes, pab_lb over fairbatch_pab nodes,
SURVEY §8d).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi, fbgpu
from .batch import CostModel, EngineConfig, Rows, engine_config, ms_to_us


@dataclass
class LbConfig:
    """LbConfig, cluster.h:36-47 (latency in ms like the scenario JSON)."""

    policy: str = "pab_lb"
    report_interval_steps: int = 1
    report_latency_ms: float = 0.0
    w_waiting: float = 1.0
    w_running: float = 1.0
    retry_reroute: bool = False
    report_cap: int = 0

    def to_c(self) -> _abi.LbConfig:
        pol = {"pab_lb": _abi.LB_PAB, "count_lb": _abi.LB_COUNT}[self.policy]
        return _abi.LbConfig(pol, int(self.report_interval_steps), ms_to_us(self.report_latency_ms),
                             float(self.w_waiting), float(self.w_running),
                             1 if self.retry_reroute else 0, int(self.report_cap))


@dataclass
class ClusterOutput:
    node_results: np.ndarray  # RESULT_DTYPE per node
    records: np.ndarray       # RECORD_DTYPE per request (global order)
    route_node: np.ndarray    # node per request, -1 = never routed
    incomplete: int
    device_ms: float = 0.0


def node_configs_c(cfgs):
    arr = (_abi.EngineConfig * max(1, len(cfgs)))()
    for i, c in enumerate(cfgs):
        arr[i] = c.to_c() if isinstance(c, EngineConfig) else c
    return arr


def run_cluster(rows: Rows, cfgs, lb: LbConfig, horizon_us: int, device: int = 0) -> ClusterOutput:
    """fb_run_cluster: the whole cluster simulation on one GPU."""
    L = fbgpu.lib()
    n = len(cfgs)
    tr = rows.to_c()
    nc = node_configs_c(cfgs)
    lbc = lb.to_c()
    res = np.zeros(max(1, n), _abi.RESULT_DTYPE)
    rec = np.zeros(max(1, len(rows)), _abi.RECORD_DTYPE)
    route = np.zeros(max(1, len(rows)), np.int32)
    inc = C.c_int32(0)
    ms = C.c_double(0)
    fbgpu._check(L.fb_run_cluster(device, C.byref(tr), C.cast(nc, C.c_void_p), n, C.byref(lbc),
                                  int(horizon_us), _abi.vptr(res), _abi.vptr(rec),
                                  _abi.vptr(route), C.byref(inc), C.byref(ms)), "fb_run_cluster")
    return ClusterOutput(res[:n], rec[:len(rows)], route[:len(rows)], inc.value, ms.value)


MODEL_7B = CostModel(5.0, 0.05, 0.0001)


def c5_rows(seed: int = 5, rate_mult: float = 8.0, horizon_ms: float = 30_000.0) -> Rows:
    """C5 trace: cluster8.json's bursty shape at 8x the rates."""
    p = fbgpu.burst_profile(30.0 * rate_mult, 90.0 * rate_mult, 800.0, 1600.0, 892.0, 1776.0,
                            250.0, 500.0, seed)
    return fbgpu.generate_bursty(p, ms_to_us(horizon_ms))


def c5(n_nodes: int = 64, latency_ms: float = 0.0, lb_policy: str = "pab_lb"):
    """(rows, node configs, lb, horizon) of BASELINE config 5."""
    node_pol = "fairbatch_pab" if lb_policy == "pab_lb" else "fairbatch"
    cfgs = [engine_config(node_pol, 2048, MODEL_7B, 500, 50) for _ in range(n_nodes)]
    return c5_rows(), cfgs, LbConfig(lb_policy, 1, latency_ms), ms_to_us(3.6e6)
