"""Host-side containers for trace rows and simulation instances.

`Rows` is the structure-of-arrays form of `Trace::requests` (workload.h:28-43)
and `Batch` is a set of independent run_node instances (engine.h:180) that
share those rows; both map one-to-one onto `fb_trace` / `fb_instance` in
include/fbgpu.h.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi


def llround(x):
    """C llround (half away from zero) on float64 scalars or arrays; exact,
    since x - trunc(x) is representable."""
    x = np.asarray(x, dtype=np.float64)
    t = np.trunc(x)
    r = t + np.where(np.abs(x - t) >= 0.5, np.sign(x), 0.0)
    return r.astype(np.int64)


def ms_to_us(ms: float) -> int:
    """time.h:30-32 (scalar llround)."""
    x = float(ms) * 1000.0
    t = math.trunc(x)
    if abs(x - t) >= 0.5:
        t += 1 if x > 0 else -1
    return int(t)


def us_to_ms(us: int) -> float:
    """time.h:34."""
    return float(us) / 1000.0


@dataclass
class CostModel:
    """costmodel.h:29-33."""

    a_ms: float = 0.0
    b_ms: float = 0.0
    c_ms: float = 0.0

    def to_c(self) -> _abi.CostModel:
        return _abi.CostModel(self.a_ms, self.b_ms, self.c_ms)


@dataclass
class SchedulerConfig:
    """sched.h:65-74."""

    policy: str = "fairbatch"
    token_budget: int = 2048
    max_chunk: int = 2048
    model: CostModel = field(default_factory=CostModel)

    def to_c(self) -> _abi.SchedulerConfig:
        if self.policy not in _abi.POLICY_NAMES:
            raise ValueError(f"unknown policy {self.policy!r}")
        return _abi.SchedulerConfig(_abi.POLICY_NAMES[self.policy], int(self.max_chunk),
                                    int(self.token_budget), self.model.to_c())


@dataclass
class EngineConfig:
    """engine.h:76-82 (NoiseSpec and global SloTargets inlined)."""

    scheduler: SchedulerConfig = field(default_factory=SchedulerConfig)
    truth_model: CostModel = field(default_factory=CostModel)
    noise_amplitude: float = 0.0
    noise_seed: int = 0
    global_ttft_us: int = 0
    global_tpot_us: int = 0
    max_active: int = 0

    def to_c(self) -> _abi.EngineConfig:
        return _abi.EngineConfig(self.scheduler.to_c(), self.truth_model.to_c(),
                                 float(self.noise_amplitude), int(self.noise_seed) & (2**64 - 1),
                                 int(self.global_ttft_us), int(self.global_tpot_us),
                                 int(self.max_active), 0)


def engine_config(policy: str, token_budget: int, model: CostModel, ttft_ms: float,
                  tpot_ms: float, max_chunk: int | None = None, noise_amplitude: float = 0.0,
                  noise_seed: int = 0, max_active: int = 0,
                  truth: CostModel | None = None) -> EngineConfig:
    """The acceptance suite's mk_cfg (acceptance.cpp:61-71), generalised."""
    return EngineConfig(
        scheduler=SchedulerConfig(policy, int(token_budget),
                                  int(token_budget if max_chunk is None else max_chunk), model),
        truth_model=truth if truth is not None else model,
        noise_amplitude=noise_amplitude, noise_seed=noise_seed,
        global_ttft_us=ms_to_us(ttft_ms), global_tpot_us=ms_to_us(tpot_ms),
        max_active=max_active)


class Rows:
    """Trace rows as a structure of arrays (sorted by arrival per trace)."""

    def __init__(self, arrival_us, prompt_len, output_len, ttft_us, tpot_us):
        self.arrival_us = np.ascontiguousarray(arrival_us, dtype=np.int64)
        self.prompt_len = np.ascontiguousarray(prompt_len, dtype=np.int32)
        self.output_len = np.ascontiguousarray(output_len, dtype=np.int32)
        self.ttft_us = np.ascontiguousarray(ttft_us, dtype=np.int64)
        self.tpot_us = np.ascontiguousarray(tpot_us, dtype=np.int64)
        n = len(self.arrival_us)
        assert all(len(a) == n for a in (self.prompt_len, self.output_len, self.ttft_us,
                                          self.tpot_us))

    def __len__(self) -> int:
        return len(self.arrival_us)

    @staticmethod
    def empty() -> "Rows":
        z8 = np.zeros(0, np.int64)
        z4 = np.zeros(0, np.int32)
        return Rows(z8, z4, z4, z8, z8)

    @staticmethod
    def concat(parts) -> "Rows":
        parts = list(parts)
        if not parts:
            return Rows.empty()
        return Rows(*(np.concatenate([getattr(p, k) for p in parts])
                      for k in ("arrival_us", "prompt_len", "output_len", "ttft_us", "tpot_us")))

    def scaled(self, factor: float) -> "Rows":
        """scale_trace (workload.cpp:211-221): llround(arrival / factor)."""
        if not factor > 0.0:
            raise ValueError("scale factor must be > 0")
        arr = llround(self.arrival_us.astype(np.float64) / factor)
        return Rows(arr, self.prompt_len, self.output_len, self.ttft_us, self.tpot_us)

    def truncated(self, n: int) -> "Rows":
        """truncate_trace (workload.cpp:223-229); n == 0 keeps all."""
        if n == 0 or n >= len(self):
            return self
        return Rows(self.arrival_us[:n], self.prompt_len[:n], self.output_len[:n],
                    self.ttft_us[:n], self.tpot_us[:n])

    def with_slo(self, ttft_us: int, tpot_us: int) -> "Rows":
        n = len(self)
        return Rows(self.arrival_us, self.prompt_len, self.output_len,
                    np.full(n, ttft_us, np.int64), np.full(n, tpot_us, np.int64))

    def offered_rps(self) -> float:
        """offered_rps (workload.cpp:315-321)."""
        n = len(self)
        if n == 0:
            return 0.0
        span = int(self.arrival_us[-1])
        if span <= 0:
            return float(n)
        return float(n) / (us_to_ms(span) / 1000.0)

    def to_c(self) -> _abi.Trace:
        return _abi.Trace(_abi.ptr(self.arrival_us, C.c_int64), _abi.ptr(self.prompt_len, C.c_int32),
                          _abi.ptr(self.output_len, C.c_int32), _abi.ptr(self.ttft_us, C.c_int64),
                          _abi.ptr(self.tpot_us, C.c_int64), len(self))

    @property
    def nbytes(self) -> int:
        return sum(a.nbytes for a in (self.arrival_us, self.prompt_len, self.output_len,
                                      self.ttft_us, self.tpot_us))


class Batch:
    """Independent run_node instances over shared trace rows."""

    def __init__(self):
        self._parts: list[Rows] = []
        self._n_rows = 0
        self._inst: list[_abi.Instance] = []
        self._rows: Rows | None = None
        self._inst_c = None  # cached ctypes instance table (rebuilt after changes)
        self.offered: list[float] = []

    def add_rows(self, rows: Rows) -> int:
        off = self._n_rows
        self._parts.append(rows)
        self._n_rows += len(rows)
        self._rows = None
        return off

    def add_instance(self, cfg: EngineConfig, trace_off: int, n_req: int, horizon_us: int,
                     offered_rps: float = 0.0) -> int:
        self._inst.append(_abi.Instance(cfg.to_c(), int(trace_off), int(n_req), int(horizon_us)))
        self._inst_c = None
        self.offered.append(offered_rps)
        return len(self._inst) - 1

    def add(self, rows: Rows, cfg: EngineConfig, horizon_us: int) -> int:
        off = self.add_rows(rows)
        return self.add_instance(cfg, off, len(rows), horizon_us, rows.offered_rps())

    def subset(self, indices) -> "Batch":
        """A new batch with only the given instances (each with its own rows)."""
        out = Batch()
        r = self.rows
        for i in indices:
            x = self._inst[i]
            s = slice(x.trace_off, x.trace_off + x.n_req)
            off = out.add_rows(Rows(r.arrival_us[s], r.prompt_len[s], r.output_len[s],
                                    r.ttft_us[s], r.tpot_us[s]))
            out._inst.append(_abi.Instance(x.cfg, off, x.n_req, x.horizon_us))
            out.offered.append(self.offered[i])
        return out

    def extend(self, other: "Batch") -> None:
        """Appends every instance of `other` (with its rows)."""
        off = self.add_rows(other.rows)
        for i, x in enumerate(other._inst):
            self._inst.append(_abi.Instance(x.cfg, off + x.trace_off, x.n_req, x.horizon_us))
            self.offered.append(other.offered[i])
        self._inst_c = None

    @property
    def rows(self) -> Rows:
        if self._rows is None:
            self._rows = Rows.concat(self._parts)
        return self._rows

    def pin(self) -> "Batch":
        """Moves the trace rows into page-locked host memory (fb_host_alloc),
        so uploads are direct DMA."""
        from .fbgpu import pinned_copy
        r = self.rows
        self._rows = Rows(*(pinned_copy(getattr(r, k)) for k in
                            ("arrival_us", "prompt_len", "output_len", "ttft_us", "tpot_us")))
        self._parts = [self._rows]
        return self

    @property
    def n_instances(self) -> int:
        return len(self._inst)

    def instances_c(self):
        """The fb_instance table as one C array (built once per batch state)."""
        if self._inst_c is None or len(self._inst_c) != max(1, len(self._inst)):
            arr = (_abi.Instance * max(1, len(self._inst)))()
            for i, x in enumerate(self._inst):
                arr[i] = x
            self._inst_c = arr
        return self._inst_c

    def record_offsets(self) -> np.ndarray:
        off = np.zeros(len(self._inst) + 1, np.int64)
        for i, x in enumerate(self._inst):
            off[i + 1] = off[i] + x.n_req
        return off

    def instance(self, i: int) -> _abi.Instance:
        return self._inst[i]
