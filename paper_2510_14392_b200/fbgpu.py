"""ctypes bindings to libfbgpu.so -- the product path.

Mirrors the fbsim reference surfaces:
  * trace generation           generate_bursty / scale_trace  (workload.h:88-94)
  * pure scheduler             form_batch / init_time_budget / pab (sched.h:81-115)
  * batched step machine       Arena (Node, engine.h:111-176; run_node, engine.h:180)
  * per-request records        Arena.records (RequestReport, metrics.h:29-49)

There is no CPU fallback: if the CUDA library is missing or no device is
present the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _abi
from .batch import Batch, Rows

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FBGPU_LIB") or os.path.join(_HERE, "libfbgpu.so")  # FBGPU_LIB: dev A/B builds


class FbError(RuntimeError):
    """Base class; subclasses mirror the fbsim exception taxonomy (errors.h:24-53)."""


class ValidationError(FbError):
    pass


class UsageError(FbError):
    pass


class ConfigError(FbError):
    pass


class ParseError(FbError):
    pass


class CudaError(FbError):
    pass


class CapacityError(FbError):
    pass


class TimeoutError_(FbError):
    """A peer rank never reached the cluster epoch exchange."""


_ERRORS = {
    _abi.FB_ERR_VALIDATION: ValidationError,
    _abi.FB_ERR_USAGE: UsageError,
    _abi.FB_ERR_CONFIG: ConfigError,
    _abi.FB_ERR_PARSE: ParseError,
    _abi.FB_ERR_CUDA: CudaError,
    _abi.FB_ERR_CAPACITY: CapacityError,
    _abi.FB_ERR_TIMEOUT: TimeoutError_,
}

_lib = None


def lib() -> C.CDLL:
    """Loads libfbgpu.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(the product path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i64, i32, pi64 = C.c_void_p, C.c_int64, C.c_int32, C.POINTER(C.c_int64)
    sig = {
        "fb_abi_version": (C.c_int, []),
        "fb_last_error": (C.c_char_p, []),
        "fb_device_count": (C.c_int, [C.POINTER(C.c_int)]),
        "fb_generate_bursty": (C.c_int, [C.POINTER(_abi.BurstProfile), i64, i64, vp, vp, vp, vp,
                                         vp, pi64]),
        "fb_scale_trace": (C.c_int, [vp, i64, C.c_double]),
        "fb_offered_rps": (C.c_int, [vp, i64, C.POINTER(C.c_double)]),
        "fb_form_batch": (C.c_int, [C.c_int, vp, vp, vp, i64, vp, vp]),
        "fb_init_time_budget": (C.c_int, [C.c_int, vp, vp, i64, vp]),
        "fb_pab": (C.c_int, [C.c_int, vp, vp, vp, vp, vp, i64, vp]),
        "fb_arena_create": (C.c_int, [C.c_int, vp, C.POINTER(vp)]),
        "fb_arena_destroy": (C.c_int, [vp]),
        "fb_arena_load": (C.c_int, [vp, C.POINTER(_abi.Trace), vp, i64, C.POINTER(_abi.LogOpts)]),
        "fb_arena_reset": (C.c_int, [vp]),
        "fb_arena_run": (C.c_int, [vp, i64, pi64]),
        "fb_arena_synchronize": (C.c_int, [vp]),
        "fb_arena_last_run_ms": (C.c_int, [vp, C.POINTER(C.c_float)]),
        "fb_arena_last_run_split_ms": (C.c_int, [vp, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
        "fb_arena_wide_phases": (C.c_int, [vp, C.POINTER(C.c_double), pi64]),
        "fb_arena_wide_selection": (C.c_int, [vp, pi64, pi64]),
        "fb_arena_fetch_results": (C.c_int, [vp, vp]),
        "fb_arena_fetch_records": (C.c_int, [vp, vp]),
        "fb_arena_fetch_summaries": (C.c_int, [vp, vp]),
        "fb_arena_set_lead": (C.c_int, [vp, i64, i32]),
        "fb_arena_fetch_lead": (C.c_int, [vp, vp, vp]),
        "fb_arena_record_rows": (i64, [vp]),
        "fb_arena_fetch_log_counts": (C.c_int, [vp, vp]),
        "fb_arena_fetch_log": (C.c_int, [vp, i64, vp, vp, vp]),
        "fb_arena_fetch_paths": (C.c_int, [vp, vp]),
        "fb_run_batch": (C.c_int, [C.c_int, C.POINTER(_abi.Trace), vp, i64, vp, vp,
                                   C.POINTER(C.c_double)]),
        "fb_run_cluster": (C.c_int, [C.c_int, C.POINTER(_abi.Trace), vp, i32,
                                     C.POINTER(_abi.LbConfig), i64, vp, vp, vp,
                                     C.POINTER(C.c_int32), C.POINTER(C.c_double)]),
        "fb_run_cluster_logged": (C.c_int, [C.c_int, C.POINTER(_abi.Trace), vp, i32,
                                            C.POINTER(_abi.LbConfig), i64,
                                            C.POINTER(_abi.LogOpts), vp, vp, vp,
                                            C.POINTER(C.c_int32), vp, vp, vp, vp, vp, vp, i64,
                                            C.POINTER(C.c_int64)]),
        "fb_cluster_partition": (C.c_int, [i32, i32, i32, C.POINTER(C.c_int32),
                                           C.POINTER(C.c_int32)]),
        "fb_cluster_shard_create": (C.c_int, [C.c_int, C.POINTER(_abi.Trace), vp, i32,
                                              C.POINTER(_abi.LbConfig), i64, i32, i32,
                                              C.POINTER(vp)]),
        "fb_cluster_shard_exchange_handle": (C.c_int, [vp, vp]),
        "fb_cluster_shard_exchange_ptr": (C.c_int, [vp, C.POINTER(vp)]),
        "fb_cluster_shard_connect": (C.c_int, [vp, vp]),
        "fb_cluster_shard_connect_ptrs": (C.c_int, [vp, vp]),
        "fb_cluster_shard_reset": (C.c_int, [vp]),
        "fb_cluster_shard_allow_hw_cluster": (C.c_int, [vp, i32]),
        "fb_cluster_max_hw_clusters": (C.c_int, [C.c_int, i32, C.POINTER(C.c_int32)]),
        "fb_cluster_fit": (C.c_int, [C.c_int, i32, i32, C.POINTER(C.c_int32)]),
        "fb_cluster_shard_launch": (C.c_int, [vp]),
        "fb_cluster_shard_wait": (C.c_int, [vp, C.POINTER(C.c_double)]),
        "fb_cluster_shard_fetch": (C.c_int, [vp, vp, vp, vp, pi64, C.POINTER(C.c_int32)]),
        "fb_cluster_shard_destroy": (None, [vp]),
        "fb_nodes_create": (C.c_int, [C.c_int, C.POINTER(_abi.Trace), vp, i32,
                                      i64, C.POINTER(_abi.LbConfig), C.POINTER(vp)]),
        "fb_nodes_destroy": (None, [vp]),
        "fb_nodes_count": (i32, [vp]),
        "fb_nodes_advance": (C.c_int, [vp, i64, vp]),
        "fb_nodes_enqueue": (C.c_int, [vp, i64, vp, vp, i64]),
        "fb_nodes_begin": (C.c_int, [vp, i64, i32, i32]),
        "fb_nodes_drain_rejects": (C.c_int, [vp, vp, vp, i64, pi64]),
        "fb_nodes_current_pab": (C.c_int, [vp, i64, vp]),
        "fb_nodes_state": (C.c_int, [vp, vp]),
        "fb_nodes_fetch": (C.c_int, [vp, vp, vp, vp, C.POINTER(C.c_int32)]),
        "fb_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(vp)]),
        "fb_host_free": (C.c_int, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    assert L.fb_abi_version() == 1
    _lib = L
    return L


def _check(status: int, what: str) -> None:
    if status != _abi.FB_OK:
        msg = lib().fb_last_error().decode(errors="replace")
        raise _ERRORS.get(status, FbError)(f"{what}: {msg}")


def device_count() -> int:
    n = C.c_int(0)
    _check(lib().fb_device_count(C.byref(n)), "fb_device_count")
    return n.value


# ------------------------------------------------------------ pinned host memory

class _Pinned:
    """Owner of one fb_host_alloc block (freed when the last view dies)."""

    def __init__(self, nbytes: int):
        p = C.c_void_p()
        _check(lib().fb_host_alloc(max(1, nbytes), C.byref(p)), "fb_host_alloc")
        self.ptr = p.value
        self.nbytes = nbytes

    def __del__(self):
        if getattr(self, "ptr", None):
            try:
                lib().fb_host_free(C.c_void_p(self.ptr))
            except Exception:
                pass
            self.ptr = None


def pinned_empty(shape, dtype) -> np.ndarray:
    """A numpy array in page-locked host memory (direct DMA through the C ABI)."""
    dtype = np.dtype(dtype)
    n = int(np.prod(shape)) if np.ndim(shape) else int(shape)
    owner = _Pinned(n * dtype.itemsize)
    buf = (C.c_char * max(1, n * dtype.itemsize)).from_address(owner.ptr)
    buf._fb_owner = owner  # keeps the block alive as long as any view
    return np.frombuffer(buf, dtype=dtype, count=n).reshape(shape)


def pinned_copy(a: np.ndarray) -> np.ndarray:
    out = pinned_empty(a.shape, a.dtype)
    out[...] = a
    return out


# ------------------------------------------------------------ trace generation

def burst_profile(base_rate, burst_rate, burst_ms, idle_ms, prompt_mean, prompt_p90,
                  output_mean, output_p90, seed, ttft_ms=500.0, tpot_ms=50.0) -> _abi.BurstProfile:
    """BurstProfile (workload.h:55-66); durations and SLOs in ms like the scenario JSON."""
    from .batch import ms_to_us
    return _abi.BurstProfile(float(base_rate), float(burst_rate), ms_to_us(burst_ms),
                             ms_to_us(idle_ms), float(prompt_mean), float(prompt_p90),
                             float(output_mean), float(output_p90), ms_to_us(ttft_ms),
                             ms_to_us(tpot_ms), int(seed) & (2**64 - 1))


def generate_bursty(profile: _abi.BurstProfile, horizon_us: int) -> Rows:
    """generate_bursty (workload.cpp:244-298) on the host."""
    L = lib()
    n = C.c_int64(0)
    st = L.fb_generate_bursty(C.byref(profile), horizon_us, 0, None, None, None, None, None,
                              C.byref(n))
    if st not in (_abi.FB_OK, _abi.FB_ERR_CAPACITY):
        _check(st, "fb_generate_bursty")
    k = n.value
    arr = np.zeros(k, np.int64)
    pr = np.zeros(k, np.int32)
    ou = np.zeros(k, np.int32)
    tt = np.zeros(k, np.int64)
    tp = np.zeros(k, np.int64)
    _check(L.fb_generate_bursty(C.byref(profile), horizon_us, k, _abi.vptr(arr), _abi.vptr(pr),
                                _abi.vptr(ou), _abi.vptr(tt), _abi.vptr(tp), C.byref(n)),
           "fb_generate_bursty")
    return Rows(arr, pr, ou, tt, tp)


def scale_trace(rows: Rows, factor: float) -> Rows:
    """scale_trace (workload.cpp:211-221)."""
    a = rows.arrival_us.copy()
    _check(lib().fb_scale_trace(_abi.vptr(a), len(a), float(factor)), "fb_scale_trace")
    return Rows(a, rows.prompt_len, rows.output_len, rows.ttft_us, rows.tpot_us)


# ------------------------------------------------------------ pure scheduler

def _task_sets(sets):
    off = np.zeros(len(sets) + 1, np.int64)
    for i, s in enumerate(sets):
        off[i + 1] = off[i] + len(s)
    tasks = (np.concatenate(sets) if len(sets) and off[-1] > 0
             else np.zeros(0, _abi.TASKVIEW_DTYPE)).astype(_abi.TASKVIEW_DTYPE)
    return np.ascontiguousarray(tasks), off


def form_batch(sets, cfgs, device: int = 0):
    """form_batch (sched.cpp:234-246) for a list of TaskView arrays on the GPU.

    Returns (plans, entries) with plans[s] a BATCHPLAN_DTYPE row and
    entries[s] the PLANENTRYID_DTYPE rows of set s in admission order."""
    tasks, off = _task_sets(sets)
    n = len(sets)
    c = (_abi.SchedulerConfig * max(1, n))(*cfgs)
    entries = np.zeros(max(1, int(off[-1])), _abi.PLANENTRYID_DTYPE)
    plans = np.zeros(max(1, n), _abi.BATCHPLAN_DTYPE)
    _check(lib().fb_form_batch(device, _abi.vptr(tasks), _abi.vptr(off), C.cast(c, C.c_void_p), n,
                               _abi.vptr(entries), _abi.vptr(plans)), "fb_form_batch")
    out = []
    for s in range(n):
        e0 = int(plans[s]["entry_off"])
        out.append(entries[e0:e0 + int(plans[s]["n_entries"])].copy())
    return plans[:n], out


def init_time_budget(sets, device: int = 0) -> np.ndarray:
    """init_time_budget (sched.cpp:90-106) per set."""
    tasks, off = _task_sets(sets)
    out = np.zeros(max(1, len(sets)), np.int64)
    _check(lib().fb_init_time_budget(device, _abi.vptr(tasks), _abi.vptr(off), len(sets),
                                     _abi.vptr(out)), "fb_init_time_budget")
    return out[:len(sets)]


def pab(sets, models, ttft_us, tpot_us, device: int = 0) -> np.ndarray:
    """pab (sched.cpp:248-278) per set."""
    tasks, off = _task_sets(sets)
    n = len(sets)
    m = (_abi.CostModel * max(1, n))(*models)
    tt = np.ascontiguousarray(np.broadcast_to(np.asarray(ttft_us, np.int64), (n,)))
    tp = np.ascontiguousarray(np.broadcast_to(np.asarray(tpot_us, np.int64), (n,)))
    out = np.zeros(max(1, n), np.int64)
    _check(lib().fb_pab(device, _abi.vptr(tasks), _abi.vptr(off), C.cast(m, C.c_void_p),
                        _abi.vptr(tt), _abi.vptr(tp), n, _abi.vptr(out)), "fb_pab")
    return out[:n]


# ------------------------------------------------------------ arena

@dataclass
class Logs:
    counts: np.ndarray
    steps: list
    entries: list
    rejects: list


class Arena:
    """Thousands of Node instances resident in HBM (one warp each)."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self._lib = lib()
        h = C.c_void_p()
        _check(self._lib.fb_arena_create(device, C.c_void_p(stream) if stream else None,
                                         C.byref(h)), "fb_arena_create")
        self._h = h
        self.device = device
        self._keep = None
        self.log_opts = None
        self.n_instances = 0

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.fb_arena_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load(self, batch: Batch, log: _abi.LogOpts | None = None) -> None:
        rows = batch.rows
        tr = rows.to_c()
        inst = batch.instances_c()
        self._keep = (rows, tr, inst)
        self.log_opts = log
        self.n_instances = batch.n_instances
        _check(self._lib.fb_arena_load(self._h, C.byref(tr), C.cast(inst, C.c_void_p),
                                       batch.n_instances, C.byref(log) if log else None),
               "fb_arena_load")

    def reset(self) -> None:
        _check(self._lib.fb_arena_reset(self._h), "fb_arena_reset")

    def run(self, max_events: int = 0, sync: bool = False) -> int | None:
        """Advances every instance by <= max_events loop iterations (0 = to quiescence).
        With sync=True returns the number of instances still running."""
        if sync:
            n = C.c_int64(0)
            _check(self._lib.fb_arena_run(self._h, max_events, C.byref(n)), "fb_arena_run")
            return n.value
        _check(self._lib.fb_arena_run(self._h, max_events, None), "fb_arena_run")
        return None

    def synchronize(self) -> None:
        _check(self._lib.fb_arena_synchronize(self._h), "fb_arena_synchronize")

    def last_run_ms(self) -> float:
        ms = C.c_float(0)
        _check(self._lib.fb_arena_last_run_ms(self._h, C.byref(ms)), "fb_arena_last_run_ms")
        return ms.value

    def last_run_split_ms(self) -> tuple[float, float]:
        """(warp engine ms, grid-wide wide engine ms) of the last run."""
        a, b = C.c_float(0), C.c_float(0)
        _check(self._lib.fb_arena_last_run_split_ms(self._h, C.byref(a), C.byref(b)),
               "fb_arena_last_run_split_ms")
        return a.value, b.value

    def wide_phases(self) -> tuple[dict, int]:
        """Phase clock of the last run's grid-wide wide engine: ({phase: ms}, iterations)."""
        ms = (C.c_double * 5)()
        it = C.c_int64(0)
        _check(self._lib.fb_arena_wide_phases(self._h, ms, C.byref(it)), "fb_arena_wide_phases")
        names = ("owner_advance", "k1_views", "k2_hist", "k2_gather", "owner_finish_cta0")
        return dict(zip(names, list(ms))), it.value

    def wide_selection(self) -> dict:
        """Node steps of the last run whose window K1 gathered itself (fused)
        and node steps that took the K2a / K2b passes."""
        f, k = C.c_int64(0), C.c_int64(0)
        _check(self._lib.fb_arena_wide_selection(self._h, C.byref(f), C.byref(k)),
               "fb_arena_wide_selection")
        return {"fused": f.value, "k2": k.value}

    def results(self) -> np.ndarray:
        out = np.zeros(max(1, self.n_instances), _abi.RESULT_DTYPE)
        _check(self._lib.fb_arena_fetch_results(self._h, _abi.vptr(out)), "fb_arena_fetch_results")
        return out[:self.n_instances]

    def records(self, out: np.ndarray | None = None) -> np.ndarray:
        """Per-request records; `out` (e.g. from pinned_empty) is filled in place."""
        n = self._lib.fb_arena_record_rows(self._h)
        if out is None:
            out = np.empty(max(1, n), _abi.RECORD_DTYPE)
        elif out.dtype != _abi.RECORD_DTYPE or len(out) < n or not out.flags.c_contiguous:
            raise ValueError("records out: need a contiguous RECORD_DTYPE array of n_rec rows")
        _check(self._lib.fb_arena_fetch_records(self._h, _abi.vptr(out)), "fb_arena_fetch_records")
        return out[:n]

    def summaries(self) -> np.ndarray:
        """Per-instance ScenarioReport aggregates computed on the device
        (SUMMARY_DTYPE rows; see reports.summary_report)."""
        out = np.zeros(max(1, self.n_instances), _abi.SUMMARY_DTYPE)
        _check(self._lib.fb_arena_fetch_summaries(self._h, _abi.vptr(out)),
               "fb_arena_fetch_summaries")
        return out[:self.n_instances]

    def set_lead(self, bucket_us: int, cap: int) -> None:
        """Enable envelope-lead accounting (applies from the next load/reset)."""
        _check(self._lib.fb_arena_set_lead(self._h, int(bucket_us), int(cap)), "fb_arena_set_lead")
        self._lead_cap = int(cap)

    def lead(self) -> list:
        """envelope_lead_series per instance (lead tokens at t = k * bucket);
        None where the point capacity was too small."""
        cap = self._lead_cap
        out = np.zeros((max(1, self.n_instances), cap), np.int64)
        n = np.zeros(max(1, self.n_instances), np.int32)
        _check(self._lib.fb_arena_fetch_lead(self._h, _abi.vptr(out), _abi.vptr(n)),
               "fb_arena_fetch_lead")
        return [None if n[i] < 0 else out[i, :n[i]].copy() for i in range(self.n_instances)]

    def record_rows(self) -> int:
        return int(self._lib.fb_arena_record_rows(self._h))

    def paths(self) -> np.ndarray:
        """Per instance FB_PATH_* bits: 1 register-resident, 2 warp memory, 4 CTA-wide,
        8 / 16 repeated-plan steps on the register / memory path."""
        out = np.zeros(max(1, self.n_instances), np.uint32)
        _check(self._lib.fb_arena_fetch_paths(self._h, _abi.vptr(out)), "fb_arena_fetch_paths")
        return out[:self.n_instances]

    def logs(self):
        """(counts, steps[n_inst, cap], entries[n_inst, cap], rejects[n_inst, cap])."""
        lo = self.log_opts
        n = self.n_instances
        counts = np.zeros(max(1, n), _abi.LOGCOUNT_DTYPE)
        _check(self._lib.fb_arena_fetch_log_counts(self._h, _abi.vptr(counts)), "log counts")
        steps = np.zeros((n, max(1, lo.step_cap)), _abi.STEPLOG_DTYPE)
        entries = np.zeros((n, max(1, lo.entry_cap)), _abi.ENTRY_DTYPE)
        rejects = np.zeros((n, max(1, lo.reject_cap)), _abi.REJECT_DTYPE)
        for i in range(n):
            _check(self._lib.fb_arena_fetch_log(self._h, i, _abi.vptr(steps[i]),
                                                _abi.vptr(entries[i]), _abi.vptr(rejects[i])),
                   "fb_arena_fetch_log")
        return counts[:n], steps, entries, rejects


def run_batch(batch: Batch, device: int = 0):
    """One-shot host-to-host run (fb_run_batch): returns (results, records, wall_ms)."""
    rows = batch.rows
    tr = rows.to_c()
    inst = batch.instances_c()
    results = np.zeros(max(1, batch.n_instances), _abi.RESULT_DTYPE)
    records = np.zeros(max(1, int(batch.record_offsets()[-1])), _abi.RECORD_DTYPE)
    ms = C.c_double(0)
    _check(lib().fb_run_batch(device, C.byref(tr), C.cast(inst, C.c_void_p), batch.n_instances,
                              _abi.vptr(results), _abi.vptr(records), C.byref(ms)), "fb_run_batch")
    return results[:batch.n_instances], records[:int(batch.record_offsets()[-1])], ms.value
