"""Test-side loaders for the CPU checkers (TEST INFRASTRUCTURE ONLY).

  * OracleLib -- oracle/liboracle.so, the C restatement of the reference path
  * RefLib    -- oracle/_ref/libfbsim_ref.so, the unmodified reference library
                compiled from /root/reference plus a C-ABI shim

Both expose the same calls as the product's C ABI (include/fbgpu.h) with an
orc_ / ref_ prefix, so a parity test runs one Batch through every backend and
compares outputs field by field.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

from paper_2510_14392_b200 import _abi
from paper_2510_14392_b200.batch import Batch, Rows

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libfbsim_ref.so")


def ensure_oracle_built() -> None:
    """The C restatement is rebuilt on demand (gcc is on every box)."""
    src = os.path.join(ROOT, "oracle", "fbsim_oracle.c")
    if not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)


@dataclass
class RunOutput:
    results: np.ndarray  # RESULT_DTYPE per instance
    records: np.ndarray  # RECORD_DTYPE per row (instance order)
    counts: np.ndarray | None = None  # LOGCOUNT_DTYPE per instance
    steps: np.ndarray | None = None  # STEPLOG_DTYPE [n_inst, step_cap]
    entries: np.ndarray | None = None  # ENTRY_DTYPE [n_inst, entry_cap]
    rejects: np.ndarray | None = None  # REJECT_DTYPE [n_inst, reject_cap]


def alloc_logs(n_inst: int, log: _abi.LogOpts | None):
    if log is None:
        return None, None, None, None
    counts = np.zeros(n_inst, _abi.LOGCOUNT_DTYPE)
    steps = np.zeros((n_inst, max(1, log.step_cap)), _abi.STEPLOG_DTYPE)
    entries = np.zeros((n_inst, max(1, log.entry_cap)), _abi.ENTRY_DTYPE)
    rejects = np.zeros((n_inst, max(1, log.reject_cap)), _abi.REJECT_DTYPE)
    return counts, steps, entries, rejects


class _CpuLib:
    prefix = ""

    def __init__(self, path: str):
        self.lib = C.CDLL(path)
        p = self.prefix
        self._gen = getattr(self.lib, p + "generate_bursty")
        self._gen.restype = C.c_int
        self._gen.argtypes = [C.POINTER(_abi.BurstProfile), C.c_int64, C.c_int64,
                              C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                              C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        self._scale = getattr(self.lib, p + "scale_trace")
        self._scale.restype = C.c_int
        self._scale.argtypes = [C.POINTER(C.c_int64), C.c_int64, C.c_double]
        self._ku = getattr(self.lib, p + "keyed_uniform")
        self._ku.restype = C.c_double
        self._ku.argtypes = [C.c_uint64, C.c_uint64]
        self._itb = getattr(self.lib, p + "init_time_budget")
        self._itb.restype = C.c_int
        self._itb.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
        self._fb = getattr(self.lib, p + "form_batch")
        self._fb.restype = C.c_int
        self._fb.argtypes = [C.c_void_p, C.c_int64, C.POINTER(_abi.SchedulerConfig), C.c_void_p,
                             C.c_void_p]
        self._pab = getattr(self.lib, p + "pab")
        self._pab.restype = C.c_int
        self._pab.argtypes = [C.c_void_p, C.c_int64, C.POINTER(_abi.CostModel), C.c_int64,
                              C.c_int64, C.POINTER(C.c_int64)]

    # -- trace generation -------------------------------------------------
    def generate_bursty(self, prof: _abi.BurstProfile, horizon_us: int) -> Rows:
        n = C.c_int64(0)
        st = self._gen(C.byref(prof), horizon_us, 0, None, None, None, None, None, C.byref(n))
        if st not in (_abi.FB_OK, _abi.FB_ERR_CAPACITY):
            raise RuntimeError(f"{self.prefix}generate_bursty failed: {st}")
        k = n.value
        arr = np.zeros(k, np.int64)
        pr = np.zeros(k, np.int32)
        ou = np.zeros(k, np.int32)
        tt = np.zeros(k, np.int64)
        tp = np.zeros(k, np.int64)
        st = self._gen(C.byref(prof), horizon_us, k, _abi.ptr(arr, C.c_int64),
                       _abi.ptr(pr, C.c_int32), _abi.ptr(ou, C.c_int32), _abi.ptr(tt, C.c_int64),
                       _abi.ptr(tp, C.c_int64), C.byref(n))
        assert st == _abi.FB_OK and n.value == k
        return Rows(arr, pr, ou, tt, tp)

    def scale_trace(self, arrival: np.ndarray, factor: float) -> np.ndarray:
        a = np.ascontiguousarray(arrival, np.int64).copy()
        st = self._scale(_abi.ptr(a, C.c_int64), len(a), factor)
        if st:
            raise ValueError("scale_trace rejected the factor")
        return a

    def keyed_uniform(self, seed: int, ordinal: int) -> float:
        return self._ku(seed, ordinal)

    # -- pure scheduler ----------------------------------------------------
    def init_time_budget(self, tasks: np.ndarray) -> int:
        out = C.c_int64(0)
        st = self._itb(_abi.vptr(tasks), len(tasks), C.byref(out))
        if st:
            raise RuntimeError(f"init_time_budget status {st}")
        return out.value

    def form_batch(self, tasks: np.ndarray, cfg: _abi.SchedulerConfig):
        entries = np.zeros(max(1, len(tasks)), _abi.PLANENTRYID_DTYPE)
        plan = np.zeros(1, _abi.BATCHPLAN_DTYPE)
        st = self._fb(_abi.vptr(tasks), len(tasks), C.byref(cfg), _abi.vptr(entries),
                      _abi.vptr(plan))
        if st:
            raise RuntimeError(f"form_batch status {st}")
        return plan[0], entries[: int(plan[0]["n_entries"])]

    def pab(self, tasks: np.ndarray, model: _abi.CostModel, ttft_us: int, tpot_us: int) -> int:
        out = C.c_int64(0)
        st = self._pab(_abi.vptr(tasks), len(tasks), C.byref(model), ttft_us, tpot_us,
                       C.byref(out))
        if st:
            raise RuntimeError(f"pab status {st}")
        return out.value


class OracleLib(_CpuLib):
    prefix = "orc_"

    def __init__(self):
        ensure_oracle_built()
        super().__init__(ORACLE_SO)
        self._run = self.lib.orc_run_instances
        self._run.restype = C.c_int
        self._run.argtypes = [C.POINTER(_abi.Trace), C.c_void_p, C.c_int64,
                              C.POINTER(_abi.LogOpts), C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]

    def run_cluster(self, rows: Rows, cfgs, lb, horizon_us: int):
        fn = self.lib.orc_run_cluster
        fn.restype = C.c_int
        st, out = _cluster_call(fn, rows, cfgs, lb, horizon_us)
        if st:
            raise RuntimeError(f"orc_run_cluster status {st}")
        return out

    def run_cluster_dist(self, rows: Rows, cfgs, lb, horizon_us: int, dist):
        """The multi-rank cluster protocol on the CPU: this rank's nodes through
        orc_cluster_shard_*, the per-epoch fb_node_report allgather over
        `dist` (gloo), and the product's merge_shards."""
        import torch
        from paper_2510_14392_b200.cluster import ShardOutput, merge_shards, node_configs_c
        L = self.lib
        vp = C.c_void_p
        sig = {
            "orc_cluster_shard_create": [C.POINTER(_abi.Trace), vp, C.c_int32,
                                         C.POINTER(_abi.LbConfig), C.c_int64, C.c_int32,
                                         C.c_int32, C.POINTER(vp)],
            "orc_cluster_shard_epochs": [vp],
            "orc_cluster_shard_advance": [vp, C.c_int64, vp],
            "orc_cluster_shard_route_begin": [vp, C.c_int64, vp, C.POINTER(C.c_int32)],
            "orc_cluster_shard_fetch": [vp, vp, vp, vp, C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int32)],
            "orc_cluster_shard_destroy": [vp],
            "orc_cluster_partition": [C.c_int32] * 3 + [C.POINTER(C.c_int32)] * 2,
        }
        for name, args in sig.items():
            getattr(L, name).argtypes = args
            getattr(L, name).restype = C.c_int
        L.orc_cluster_shard_epochs.restype = C.c_int64
        L.orc_cluster_shard_destroy.restype = None
        rank, world = dist.get_rank(), dist.get_world_size()
        n = len(cfgs)
        lo, nl = C.c_int32(0), C.c_int32(0)
        assert L.orc_cluster_partition(n, world, rank, C.byref(lo), C.byref(nl)) == 0
        cap = max((n * (r + 1) // world) - (n * r // world) for r in range(world))
        tr = rows.to_c()
        nc = node_configs_c(cfgs)
        lbc = lb.to_c()
        h = vp()
        st = L.orc_cluster_shard_create(C.byref(tr), C.cast(nc, vp), n, C.byref(lbc),
                                        int(horizon_us), rank, world, C.byref(h))
        if st:
            raise RuntimeError(f"orc_cluster_shard_create status {st}")
        try:
            local = np.zeros(cap, _abi.NODE_REPORT_DTYPE)
            stopped = C.c_int32(0)
            for e in range(L.orc_cluster_shard_epochs(h)):
                st = L.orc_cluster_shard_advance(h, e, _abi.vptr(local))
                if st:
                    raise RuntimeError(f"orc_cluster_shard_advance status {st}")
                t = torch.from_numpy(local.view(np.int64).copy())
                parts = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(parts, t)
                all_rep = np.concatenate([
                    p.numpy().view(_abi.NODE_REPORT_DTYPE)[:(n * (r + 1) // world) - (n * r // world)]
                    for r, p in enumerate(parts)])
                st = L.orc_cluster_shard_route_begin(h, e, _abi.vptr(all_rep), C.byref(stopped))
                if st:
                    raise RuntimeError(f"orc_cluster_shard_route_begin status {st}")
                if stopped.value:
                    break
            res = np.zeros(max(1, nl.value), _abi.RESULT_DTYPE)
            rec = np.zeros(max(1, len(rows)), _abi.RECORD_DTYPE)
            route = np.zeros(max(1, len(rows)), np.int32)
            nrt, inc = C.c_int64(0), C.c_int32(0)
            st = L.orc_cluster_shard_fetch(h, _abi.vptr(res), _abi.vptr(rec), _abi.vptr(route),
                                           C.byref(nrt), C.byref(inc))
            if st:
                raise RuntimeError(f"orc_cluster_shard_fetch status {st}")
        finally:
            L.orc_cluster_shard_destroy(h)
        out = ShardOutput(lo.value, res[:nl.value], rec[:len(rows)], route[:len(rows)],
                          nrt.value, inc.value)
        gathered = [None] * world
        dist.all_gather_object(gathered, out)
        return merge_shards(gathered, n)

    def run(self, batch: Batch, log: _abi.LogOpts | None = None, nthreads: int = 1) -> RunOutput:
        n = batch.n_instances
        rows = batch.rows
        tr = rows.to_c()
        inst = batch.instances_c()
        results = np.zeros(n, _abi.RESULT_DTYPE)
        records = np.zeros(int(batch.record_offsets()[-1]), _abi.RECORD_DTYPE)
        counts, steps, entries, rejects = alloc_logs(n, log)
        st = self._run(C.byref(tr), C.cast(inst, C.c_void_p), n,
                       C.byref(log) if log is not None else None, _abi.vptr(results),
                       _abi.vptr(records), _abi.vptr(counts), _abi.vptr(steps),
                       _abi.vptr(entries), _abi.vptr(rejects), nthreads)
        if st:
            raise RuntimeError(f"orc_run_instances status {st}")
        return RunOutput(results, records, counts, steps, entries, rejects)


def _cluster_call(fn, rows, cfgs, lb, horizon_us, *extra):
    from paper_2510_14392_b200.cluster import ClusterOutput, node_configs_c
    n = len(cfgs)
    tr = rows.to_c()
    nc = node_configs_c(cfgs)
    lbc = lb.to_c()
    res = np.zeros(max(1, n), _abi.RESULT_DTYPE)
    rec = np.zeros(max(1, len(rows)), _abi.RECORD_DTYPE)
    route = np.zeros(max(1, len(rows)), np.int32)
    inc = C.c_int32(0)
    st = fn(C.byref(tr), C.cast(nc, C.c_void_p), C.c_int32(n), C.byref(lbc), C.c_int64(horizon_us),
            _abi.vptr(res), _abi.vptr(rec), _abi.vptr(route), C.byref(inc), *extra)
    return st, ClusterOutput(res[:n], rec[:len(rows)], route[:len(rows)], inc.value)


CLUSTER_KEYS = ("steps", "plan_digest", "n_arrived", "n_rejected", "sum_entries",
                "sum_new_tokens", "incomplete")


def cluster_summary(out) -> dict:
    """Exact, comparable part of a cluster run."""
    import hashlib
    return {
        "nodes": [{k: int(r[k]) for k in CLUSTER_KEYS} for r in out.node_results],
        "records_sha256": hashlib.sha256(out.records.tobytes()).hexdigest(),
        "route_sha256": hashlib.sha256(out.route_node.astype(np.int32).tobytes()).hexdigest(),
        "incomplete": int(out.incomplete),
    }


class RefLib(_CpuLib):
    prefix = "ref_"

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self):
        super().__init__(REF_SO)
        self.lib.ref_last_error.restype = C.c_char_p
        self._run = self.lib.ref_run_instances
        self._run.restype = C.c_int
        self._run.argtypes = [C.POINTER(_abi.Trace), C.c_void_p, C.c_int64,
                              C.POINTER(_abi.LogOpts), C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        self._batch = self.lib.ref_run_node_batch
        self._batch.restype = C.c_int
        self._batch.argtypes = [C.POINTER(_abi.Trace), C.c_void_p, C.c_int64, C.c_void_p,
                                C.c_void_p, C.c_int]

    def run(self, batch: Batch, log: _abi.LogOpts | None = None, nthreads: int = 1,
            check: bool = False) -> RunOutput:
        n = batch.n_instances
        tr = batch.rows.to_c()
        inst = batch.instances_c()
        results = np.zeros(n, _abi.RESULT_DTYPE)
        records = np.zeros(int(batch.record_offsets()[-1]), _abi.RECORD_DTYPE)
        counts, steps, entries, rejects = alloc_logs(n, log)
        st = self._run(C.byref(tr), C.cast(inst, C.c_void_p), n,
                       C.byref(log) if log is not None else None, _abi.vptr(results),
                       _abi.vptr(records), _abi.vptr(counts), _abi.vptr(steps),
                       _abi.vptr(entries), _abi.vptr(rejects), nthreads, 1 if check else 0)
        if st:
            raise RuntimeError(f"ref_run_instances status {st}: {self.lib.ref_last_error()}")
        return RunOutput(results, records, counts, steps, entries, rejects)

    def run_cluster(self, rows: Rows, cfgs, lb, horizon_us: int, check: bool = False):
        """The reference's run_cluster (mirrored through Node/route/apply_report)."""
        from paper_2510_14392_b200.cluster import ClusterOutput, node_configs_c
        fn = self.lib.ref_run_cluster
        fn.restype = C.c_int
        n = len(cfgs)
        tr = rows.to_c()
        nc = node_configs_c(cfgs)
        lbc = lb.to_c()
        res = np.zeros(max(1, n), _abi.RESULT_DTYPE)
        rec = np.zeros(max(1, len(rows)), _abi.RECORD_DTYPE)
        route = np.zeros(max(1, len(rows)), np.int32)
        inc = C.c_int32(0)
        st = fn(C.byref(tr), C.cast(nc, C.c_void_p), C.c_int32(n), C.byref(lbc),
                C.c_int64(horizon_us), _abi.vptr(res), _abi.vptr(rec), _abi.vptr(route),
                C.byref(inc), C.c_int(1 if check else 0))
        if st:
            raise RuntimeError(f"ref_run_cluster status {st}: {self.lib.ref_last_error()}")
        return ClusterOutput(res[:n], rec[:len(rows)], route[:len(rows)], inc.value)

    def run_cluster_stock(self, rows: Rows, cfgs, lb, horizon_us: int, n_rep: int = 1,
                          nthreads: int = 1, records: bool = False):
        """The reference's own run_cluster, unmirrored (timing baseline):
        n_rep copies on a thread pool.  Per-node results [n_rep, n_nodes]
        (steps / n_arrived / n_rejected / incomplete) and copy 0's records."""
        from paper_2510_14392_b200.cluster import node_configs_c
        fn = self.lib.ref_run_cluster_stock
        fn.restype = C.c_int
        n = len(cfgs)
        tr = rows.to_c()
        nc = node_configs_c(cfgs)
        lbc = lb.to_c()
        res = np.zeros((n_rep, n), _abi.RESULT_DTYPE)
        rec = np.zeros(max(1, len(rows)), _abi.RECORD_DTYPE) if records else None
        st = fn(C.byref(tr), C.cast(nc, C.c_void_p), C.c_int32(n), C.byref(lbc),
                C.c_int64(horizon_us), C.c_int32(n_rep), _abi.vptr(res), _abi.vptr(rec),
                C.c_int(nthreads))
        if st:
            raise RuntimeError(f"ref_run_cluster_stock status {st}: {self.lib.ref_last_error()}")
        return res, (rec[:len(rows)] if records else None)

    def event_log(self, batch: Batch, i: int, tmp_path: str) -> str:
        """The reference's save_event_log JSONL of instance i."""
        fn = self.lib.ref_event_log
        fn.restype = C.c_int
        tr = batch.rows.to_c()
        inst = batch.instance(i)
        n = C.c_int64(0)
        cap = 1 << 20
        while True:
            buf = C.create_string_buffer(cap)
            st = fn(C.byref(tr), C.byref(inst), tmp_path.encode(), buf, C.c_int64(cap), C.byref(n))
            if st == _abi.FB_ERR_CAPACITY:
                cap = n.value + 1
                continue
            if st:
                raise RuntimeError(f"ref_event_log status {st}")
            return buf.raw[: n.value].decode()

    def cluster_logs(self, rows: Rows, cfgs, lb, horizon_us: int, tmp_path: str):
        """The real run_cluster's node event logs and routing log, as written by
        the reference's save_event_log / save_routing_log."""
        from paper_2510_14392_b200.cluster import node_configs_c
        fn = self.lib.ref_cluster_logs
        fn.restype = C.c_int
        n = len(cfgs)
        tr = rows.to_c()
        nc = node_configs_c(cfgs)
        lbc = lb.to_c()
        offs = np.zeros(n + 2, np.int64)
        ln = C.c_int64(0)
        cap = 1 << 22
        while True:
            buf = C.create_string_buffer(cap)
            st = fn(C.byref(tr), C.cast(nc, C.c_void_p), C.c_int32(n), C.byref(lbc),
                    C.c_int64(horizon_us), tmp_path.encode(), buf, C.c_int64(cap),
                    _abi.vptr(offs), C.byref(ln))
            if st == _abi.FB_ERR_CAPACITY:
                cap = ln.value + 1
                continue
            if st:
                raise RuntimeError(f"ref_cluster_logs status {st}: {self.lib.ref_last_error()}")
            text = buf.raw[: ln.value].decode()
            parts = [text[offs[i]:offs[i + 1]] for i in range(n + 1)]
            return parts[:n], parts[n]

    def replay_check(self, jsonl: str, tmp_path: str) -> list[str]:
        """The reference's load_event_log + replay_check of a JSONL text."""
        fn = self.lib.ref_replay_check
        fn.restype = C.c_int
        with open(tmp_path, "w") as f:
            f.write(jsonl)
        n, nv = C.c_int64(0), C.c_int64(0)
        cap = 1 << 16
        while True:
            buf = C.create_string_buffer(cap)
            st = fn(tmp_path.encode(), buf, C.c_int64(cap), C.byref(n), C.byref(nv))
            if st == _abi.FB_ERR_CAPACITY:
                cap = n.value + 1
                continue
            if st:
                raise RuntimeError(f"ref_replay_check status {st}: {self.lib.ref_last_error()}")
            text = buf.raw[: n.value].decode()
            return text.split("\n")[:-1] if text else []

    def lead_series(self, batch: Batch, i: int, bucket_us: int) -> np.ndarray:
        """The reference's envelope_lead_series (metrics.cpp:137-169) of instance i."""
        fn = self.lib.ref_lead_series
        fn.restype = C.c_int
        tr = batch.rows.to_c()
        inst = batch.instance(i)
        n = C.c_int64(0)
        cap = 4096
        while True:
            out = np.zeros(cap, np.int64)
            st = fn(C.byref(tr), C.byref(inst), C.c_int64(bucket_us), _abi.vptr(out),
                    C.c_int64(cap), C.byref(n))
            if st == _abi.FB_ERR_CAPACITY:
                cap = n.value
                continue
            if st:
                raise RuntimeError(f"ref_lead_series status {st}")
            return out[: n.value]

    def run_node_batch(self, batch: Batch, nthreads: int = 1, records: bool = True) -> RunOutput:
        n = batch.n_instances
        tr = batch.rows.to_c()
        inst = batch.instances_c()
        results = np.zeros(n, _abi.RESULT_DTYPE)
        rec = np.zeros(int(batch.record_offsets()[-1]), _abi.RECORD_DTYPE) if records else None
        st = self._batch(C.byref(tr), C.cast(inst, C.c_void_p), n, _abi.vptr(results),
                         _abi.vptr(rec), nthreads)
        if st:
            raise RuntimeError(f"ref_run_node_batch status {st}")
        return RunOutput(results, rec)
