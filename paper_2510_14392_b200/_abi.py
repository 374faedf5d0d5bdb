"""ctypes mirror of include/fbgpu.h (the C ABI).

Pure data definitions: struct layouts, enums and argument signatures.  The
same layouts are used to drive the product library (libfbgpu.so), the C
oracle (oracle/liboracle.so, tests only) and the reference shim
(oracle/_ref/libfbsim_ref.so, tests and the bench reference arm only).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

FB_OK = 0
FB_ERR_VALIDATION = 1
FB_ERR_USAGE = 2
FB_ERR_CONFIG = 3
FB_ERR_PARSE = 4
FB_ERR_CUDA = 5
FB_ERR_CAPACITY = 6
FB_ERR_TIMEOUT = 7
FB_IPC_HANDLE_BYTES = 64

POLICY_PREFILL_FIRST = 0
POLICY_SARATHI = 1
POLICY_FAIRBATCH = 2
POLICY_FAIRBATCH_PAB = 3
POLICY_NAMES = {
    "prefill_first": POLICY_PREFILL_FIRST,
    "sarathi": POLICY_SARATHI,
    "fairbatch": POLICY_FAIRBATCH,
    "fairbatch_pab": POLICY_FAIRBATCH_PAB,
}

PHASE_PREFILL = 0
PHASE_DECODE = 1

LB_COUNT = 0
LB_PAB = 1

REC_ARRIVED = 1
REC_REJECTED = 2
REC_FINISHED = 4
REC_MET_TTFT = 8
REC_MET_TPOT = 16
REC_ENV_MISS = 32


class CostModel(C.Structure):
    _fields_ = [("a_ms", C.c_double), ("b_ms", C.c_double), ("c_ms", C.c_double)]


class SchedulerConfig(C.Structure):
    _fields_ = [
        ("policy", C.c_int32),
        ("max_chunk", C.c_int32),
        ("token_budget", C.c_int64),
        ("model", CostModel),
    ]


class EngineConfig(C.Structure):
    _fields_ = [
        ("scheduler", SchedulerConfig),
        ("truth_model", CostModel),
        ("noise_amplitude", C.c_double),
        ("noise_seed", C.c_uint64),
        ("global_ttft_us", C.c_int64),
        ("global_tpot_us", C.c_int64),
        ("max_active", C.c_int32),
        ("reserved", C.c_int32),
    ]


class Trace(C.Structure):
    _fields_ = [
        ("arrival_us", C.POINTER(C.c_int64)),
        ("prompt_len", C.POINTER(C.c_int32)),
        ("output_len", C.POINTER(C.c_int32)),
        ("ttft_us", C.POINTER(C.c_int64)),
        ("tpot_us", C.POINTER(C.c_int64)),
        ("n_rows", C.c_int64),
    ]


class Instance(C.Structure):
    _fields_ = [
        ("cfg", EngineConfig),
        ("trace_off", C.c_int64),
        ("n_req", C.c_int64),
        ("horizon_us", C.c_int64),
    ]


class Record(C.Structure):
    _fields_ = [
        ("first_emit_us", C.c_int64),
        ("max_tpot_ms", C.c_double),
        ("max_tpot_alt_ms", C.c_double),
        ("tokens_emitted", C.c_int32),
        ("flags", C.c_uint32),
    ]


class InstanceResult(C.Structure):
    _fields_ = [
        ("steps", C.c_uint64),
        ("plan_digest", C.c_uint64),
        ("end_time_us", C.c_int64),
        ("n_arrived", C.c_int64),
        ("n_rejected", C.c_int64),
        ("sum_visible", C.c_int64),
        ("sum_entries", C.c_int64),
        ("sum_new_tokens", C.c_int64),
        ("incomplete", C.c_int32),
        ("status", C.c_int32),
    ]


class StepLog(C.Structure):
    _fields_ = [
        ("t_us", C.c_int64),
        ("duration_us", C.c_int64),
        ("predicted_ms", C.c_double),
        ("actual_ms", C.c_double),
        ("total_new", C.c_int64),
        ("total_ctx", C.c_int64),
        ("init_budget_ms", C.c_double),
        ("entry_off", C.c_int32),
        ("n_entries", C.c_int32),
    ]


class PlanEntry(C.Structure):
    _fields_ = [("req", C.c_int32), ("new_tokens", C.c_int32)]


class RejectLog(C.Structure):
    _fields_ = [
        ("t_us", C.c_int64),
        ("pab_tokens", C.c_int64),
        ("req", C.c_int32),
        ("step", C.c_int32),
    ]


class LogOpts(C.Structure):
    _fields_ = [
        ("step_cap", C.c_int32),
        ("entry_cap", C.c_int32),
        ("reject_cap", C.c_int32),
        ("reserved", C.c_int32),
    ]


class LogCounts(C.Structure):
    _fields_ = [
        ("steps", C.c_int32),
        ("entries", C.c_int32),
        ("rejects", C.c_int32),
        ("truncated", C.c_int32),
    ]


class BurstProfile(C.Structure):
    _fields_ = [
        ("base_rate", C.c_double),
        ("burst_rate", C.c_double),
        ("burst_duration_us", C.c_int64),
        ("idle_duration_us", C.c_int64),
        ("prompt_mean", C.c_double),
        ("prompt_p90", C.c_double),
        ("output_mean", C.c_double),
        ("output_p90", C.c_double),
        ("ttft_us", C.c_int64),
        ("tpot_us", C.c_int64),
        ("seed", C.c_uint64),
    ]


class LbConfig(C.Structure):
    _fields_ = [
        ("policy", C.c_int32),
        ("report_interval_steps", C.c_int32),
        ("report_latency_us", C.c_int64),
        ("w_waiting", C.c_double),
        ("w_running", C.c_double),
        ("retry_reroute", C.c_int32),
        ("report_cap", C.c_int32),
    ]


class TaskView(C.Structure):
    _fields_ = [
        ("request_id", C.c_int64),
        ("slack_us", C.c_int64),
        ("context", C.c_int64),
        ("arrival_seq", C.c_int64),
        ("tpot_us", C.c_int64),
        ("new_tokens", C.c_int32),
        ("phase", C.c_int32),
    ]


class BatchPlan(C.Structure):
    _fields_ = [
        ("predicted_ms", C.c_double),
        ("time_budget_used_ms", C.c_double),
        ("token_budget_used", C.c_int64),
        ("init_time_budget_ms", C.c_double),
        ("entry_off", C.c_int64),
        ("n_entries", C.c_int64),
    ]


class PlanEntryId(C.Structure):
    _fields_ = [("request_id", C.c_int64), ("new_tokens", C.c_int32), ("reserved", C.c_int32)]


# numpy dtypes with the same layouts (aligned, matches the C structs)
def _np_dtype(struct):
    return np.dtype(np.ctypeslib.as_ctypes_type(np.dtype(struct)))


NODE_REPORT_DTYPE = np.dtype([("emitted_at", "<i8"), ("pab_tokens", "<i8"), ("waiting", "<i4"),
                              ("running", "<i4"), ("fresh", "<i4"), ("busy", "<i4")])  # fb_node_report
NODE_STATE_DTYPE = np.dtype([("step_end", "<i8"), ("waiting", "<i8"), ("running", "<i8"),
                             ("steps_completed", "<i8"), ("busy", "<i4"),
                             ("has_live", "<i4")])  # fb_node_state
RECORD_DTYPE = np.dtype(
    [("first_emit_us", "<i8"), ("max_tpot_ms", "<f8"), ("max_tpot_alt_ms", "<f8"),
     ("tokens_emitted", "<i4"), ("flags", "<u4")], align=True)
RESULT_DTYPE = np.dtype(
    [("steps", "<u8"), ("plan_digest", "<u8"), ("end_time_us", "<i8"), ("n_arrived", "<i8"),
     ("n_rejected", "<i8"), ("sum_visible", "<i8"), ("sum_entries", "<i8"),
     ("sum_new_tokens", "<i8"), ("incomplete", "<i4"), ("status", "<i4")], align=True)
STEPLOG_DTYPE = np.dtype(
    [("t_us", "<i8"), ("duration_us", "<i8"), ("predicted_ms", "<f8"), ("actual_ms", "<f8"),
     ("total_new", "<i8"), ("total_ctx", "<i8"), ("init_budget_ms", "<f8"),
     ("entry_off", "<i4"), ("n_entries", "<i4")], align=True)
ENTRY_DTYPE = np.dtype([("req", "<i4"), ("new_tokens", "<i4")], align=True)
REJECT_DTYPE = np.dtype([("t_us", "<i8"), ("pab_tokens", "<i8"), ("req", "<i4"),
                         ("step", "<i4")], align=True)
LOGCOUNT_DTYPE = np.dtype([("steps", "<i4"), ("entries", "<i4"), ("rejects", "<i4"),
                           ("truncated", "<i4")], align=True)
ROUTELOG_DTYPE = np.dtype([("t_us", "<i8"), ("req", "<i4"), ("node", "<i4"),
                           ("rej_before", "<i4"), ("steps_before", "<i4")], align=True)
TASKVIEW_DTYPE = np.dtype(
    [("request_id", "<i8"), ("slack_us", "<i8"), ("context", "<i8"), ("arrival_seq", "<i8"),
     ("tpot_us", "<i8"), ("new_tokens", "<i4"), ("phase", "<i4")], align=True)
PLANENTRYID_DTYPE = np.dtype([("request_id", "<i8"), ("new_tokens", "<i4"),
                              ("reserved", "<i4")], align=True)
BATCHPLAN_DTYPE = np.dtype(
    [("predicted_ms", "<f8"), ("time_budget_used_ms", "<f8"), ("token_budget_used", "<i8"),
     ("init_time_budget_ms", "<f8"), ("entry_off", "<i8"), ("n_entries", "<i8")], align=True)

class Percentiles(C.Structure):
    _fields_ = [("p50", C.c_double), ("p95", C.c_double), ("p99", C.c_double),
                ("count", C.c_int64)]


class Summary(C.Structure):
    """fb_summary: per-instance ScenarioReport aggregates (metrics.cpp:171-205)."""
    _fields_ = [("total_requests", C.c_int64), ("rejected", C.c_int64), ("finished", C.c_int64),
                ("good", C.c_int64), ("ttft_violations", C.c_int64),
                ("envelope_misses", C.c_int64), ("ttft_ms", Percentiles),
                ("max_tpot_ms", Percentiles), ("max_tpot_alt_ms", Percentiles)]


_PCT = [("p50", "<f8"), ("p95", "<f8"), ("p99", "<f8"), ("count", "<i8")]
SUMMARY_DTYPE = np.dtype(
    [("total_requests", "<i8"), ("rejected", "<i8"), ("finished", "<i8"), ("good", "<i8"),
     ("ttft_violations", "<i8"), ("envelope_misses", "<i8"), ("ttft_ms", _PCT),
     ("max_tpot_ms", _PCT), ("max_tpot_alt_ms", _PCT)], align=True)

for _st, _dt in ((Summary, SUMMARY_DTYPE), (Record, RECORD_DTYPE), (InstanceResult, RESULT_DTYPE), (StepLog, STEPLOG_DTYPE),
                 (PlanEntry, ENTRY_DTYPE), (RejectLog, REJECT_DTYPE), (LogCounts, LOGCOUNT_DTYPE),
                 (TaskView, TASKVIEW_DTYPE), (PlanEntryId, PLANENTRYID_DTYPE),
                 (BatchPlan, BATCHPLAN_DTYPE)):
    assert C.sizeof(_st) == _dt.itemsize, (_st.__name__, C.sizeof(_st), _dt.itemsize)


def ptr(arr, ctype):
    """Raw pointer to a contiguous numpy array (None for None)."""
    if arr is None:
        return None
    assert arr.flags["C_CONTIGUOUS"]
    return arr.ctypes.data_as(C.POINTER(ctype))


def vptr(arr):
    if arr is None:
        return None
    assert arr.flags["C_CONTIGUOUS"]
    return C.c_void_p(arr.ctypes.data)
