"""Cluster-level simulation (run_cluster, cluster.h:107-109) on the device.

`LbConfig` mirrors cluster.h:36-47; `run_cluster` calls fb_run_cluster (one
GPU); `run_cluster_dist` partitions the nodes over the ranks of a
torch.distributed group (one GPU per rank) and runs the fb_cluster_shard_*
protocol -- per dispatch epoch every node's report goes into every rank's
exchange buffer over NVLink peer memory, then a replicated router routes the
epoch's arrivals; `merge_shards` reassembles the single-GPU
outputs.  `c5` builds BASELINE config 5 (64 nodes, pab_lb over fairbatch_pab
nodes).
"""
from __future__ import annotations

import ctypes as C
import time
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


def partition(n_nodes: int, world: int, rank: int) -> tuple[int, int]:
    """(node_lo, n_local) of `rank` -- fb_cluster_partition's contiguous ranges."""
    if n_nodes < 1 or world < 1 or not 0 <= rank < world or world > n_nodes:
        raise ValueError("bad cluster partition")
    lo = n_nodes * rank // world
    return lo, n_nodes * (rank + 1) // world - lo


@dataclass
class ShardOutput:
    """One rank's share of a cluster run (fb_cluster_shard_fetch)."""

    node_lo: int
    node_results: np.ndarray  # RESULT_DTYPE of nodes [node_lo, node_lo + n_local)
    records: np.ndarray       # per request; filled for requests routed to local nodes
    route_node: np.ndarray    # identical on every rank
    n_routed: int
    incomplete: int
    device_ms: float = 0.0


def merge_shards(parts: list[ShardOutput], n_nodes: int) -> ClusterOutput:
    """The single-GPU ClusterOutput from every rank's ShardOutput."""
    parts = sorted(parts, key=lambda p: p.node_lo)
    route = parts[0].route_node
    for p in parts[1:]:
        if not np.array_equal(p.route_node, route) or p.n_routed != parts[0].n_routed:
            raise RuntimeError("ranks disagree on the routing decisions")
    res = np.concatenate([p.node_results for p in parts])
    if len(res) != n_nodes:
        raise RuntimeError("shard outputs do not cover the cluster")
    inc = int(any(p.incomplete for p in parts))
    res["incomplete"] = inc
    rec = parts[0].records.copy()
    for p in parts[1:]:
        own = (route >= p.node_lo) & (route < p.node_lo + len(p.node_results))
        rec[own] = p.records[own]
    return ClusterOutput(res, rec, route.copy(), inc, max(p.device_ms for p in parts))


class ClusterShard:
    """fb_cluster_shard_*: this rank's nodes of one cluster simulation."""

    def __init__(self, rows: Rows, cfgs, lb: LbConfig, horizon_us: int, rank: int, world: int,
                 device: int = 0):
        L = fbgpu.lib()
        self._L = L
        self.n_nodes = len(cfgs)
        self.n_rows = len(rows)
        self.node_lo, self.n_local = partition(self.n_nodes, world, rank)
        self._tr = rows.to_c()  # keep the host rows alive while the shard exists
        nc = node_configs_c(cfgs)
        lbc = lb.to_c()
        h = C.c_void_p()
        fbgpu._check(L.fb_cluster_shard_create(device, C.byref(self._tr), C.cast(nc, C.c_void_p),
                                               self.n_nodes, C.byref(lbc), int(horizon_us),
                                               rank, world, C.byref(h)),
                     "fb_cluster_shard_create")
        self._h = h

    def exchange_handle(self) -> bytes:
        buf = (C.c_ubyte * _abi.FB_IPC_HANDLE_BYTES)()
        fbgpu._check(self._L.fb_cluster_shard_exchange_handle(self._h, buf),
                     "fb_cluster_shard_exchange_handle")
        return bytes(buf)

    def exchange_ptr(self) -> int:
        p = C.c_void_p()
        fbgpu._check(self._L.fb_cluster_shard_exchange_ptr(self._h, C.byref(p)),
                     "fb_cluster_shard_exchange_ptr")
        return int(p.value)

    def connect(self, handles: list[bytes]) -> None:
        raw = b"".join(handles)
        fbgpu._check(self._L.fb_cluster_shard_connect(self._h, raw), "fb_cluster_shard_connect")

    def connect_ptrs(self, ptrs: list[int]) -> None:
        arr = (C.c_void_p * len(ptrs))(*ptrs)
        fbgpu._check(self._L.fb_cluster_shard_connect_ptrs(self._h, arr),
                     "fb_cluster_shard_connect_ptrs")

    def reset(self) -> None:
        fbgpu._check(self._L.fb_cluster_shard_reset(self._h), "fb_cluster_shard_reset")

    def launch(self) -> None:
        fbgpu._check(self._L.fb_cluster_shard_launch(self._h), "fb_cluster_shard_launch")

    def wait(self) -> float:
        ms = C.c_double(0)
        fbgpu._check(self._L.fb_cluster_shard_wait(self._h, C.byref(ms)), "fb_cluster_shard_wait")
        return ms.value

    def fetch(self, device_ms: float = 0.0) -> ShardOutput:
        res = np.zeros(max(1, self.n_local), _abi.RESULT_DTYPE)
        rec = np.zeros(max(1, self.n_rows), _abi.RECORD_DTYPE)
        route = np.zeros(max(1, self.n_rows), np.int32)
        nrt = C.c_int64(0)
        inc = C.c_int32(0)
        fbgpu._check(self._L.fb_cluster_shard_fetch(self._h, _abi.vptr(res), _abi.vptr(rec),
                                                    _abi.vptr(route), C.byref(nrt), C.byref(inc)),
                     "fb_cluster_shard_fetch")
        return ShardOutput(self.node_lo, res[:self.n_local], rec[:self.n_rows],
                           route[:self.n_rows], nrt.value, inc.value, device_ms)

    def close(self) -> None:
        if self._h:
            self._L.fb_cluster_shard_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_cluster_dist(rows: Rows, cfgs, lb: LbConfig, horizon_us: int, dist,
                     device: int | None = None) -> ClusterOutput:
    """run_cluster with the nodes partitioned over the ranks of `dist` (one
    GPU per rank, NVLink peer memory between them); every rank returns the
    merged single-GPU output."""
    rank, world = dist.get_rank(), dist.get_world_size()
    if device is None:
        import torch
        device = torch.cuda.current_device()
    sh = ClusterShard(rows, cfgs, lb, horizon_us, rank, world, device)
    try:
        if world > 1:
            handles = [None] * world
            dist.all_gather_object(handles, sh.exchange_handle())
            sh.connect(handles)
        sh.reset()
        dist.barrier()  # every exchange counter is zero before any rank launches
        sh.launch()
        out = sh.fetch(sh.wait())
    finally:
        sh.close()
    parts = [None] * world
    dist.all_gather_object(parts, out)
    return merge_shards(parts, len(cfgs))


@dataclass
class ClusterLogs:
    """run_cluster's logs (ClusterResult, cluster.h:93-98): per node the plan
    log its EventLog is rebuilt from, and the routing log with the view
    snapshot of every decision (events.cluster_event_logs writes both in the
    reference's JSONL formats)."""
    out: ClusterOutput
    counts: np.ndarray     # LOGCOUNT_DTYPE per node
    steps: np.ndarray      # [node, step_cap] STEPLOG_DTYPE
    entries: np.ndarray    # [node, entry_cap] ENTRY_DTYPE
    rejects: np.ndarray    # [node, reject_cap] REJECT_DTYPE
    routes: np.ndarray     # ROUTELOG_DTYPE, decision order
    snapshots: np.ndarray  # [decision, node] float64


def run_cluster_logged(rows: Rows, cfgs, lb: LbConfig, horizon_us: int,
                       device: int = 0) -> ClusterLogs:
    """fb_run_cluster_logged; the plan-log capacities come from a first
    (unlogged) run of the same cluster, so nothing is truncated."""
    L = fbgpu.lib()
    first = run_cluster(rows, cfgs, lb, horizon_us, device)
    nr = first.node_results
    lo = _abi.LogOpts(max(1, int(nr["steps"].max())), max(1, int(nr["sum_entries"].max())),
                      max(1, int(nr["n_rejected"].max())), 0)
    n, m = len(cfgs), len(rows)
    tr = rows.to_c()
    nc = node_configs_c(cfgs)
    lbc = lb.to_c()
    res = np.zeros(max(1, n), _abi.RESULT_DTYPE)
    rec = np.zeros(max(1, m), _abi.RECORD_DTYPE)
    route = np.zeros(max(1, m), np.int32)
    inc = C.c_int32(0)
    counts = np.zeros(max(1, n), _abi.LOGCOUNT_DTYPE)
    steps = np.zeros((n, lo.step_cap), _abi.STEPLOG_DTYPE)
    entries = np.zeros((n, lo.entry_cap), _abi.ENTRY_DTYPE)
    rejects = np.zeros((n, lo.reject_cap), _abi.REJECT_DTYPE)
    cap = 2 * m + 1 if lb.retry_reroute else m + 1
    routes = np.zeros(cap, _abi.ROUTELOG_DTYPE)
    snaps = np.zeros((cap, n), np.float64)
    nrt = C.c_int64(0)
    fbgpu._check(L.fb_run_cluster_logged(
        device, C.byref(tr), C.cast(nc, C.c_void_p), n, C.byref(lbc), int(horizon_us),
        C.byref(lo), _abi.vptr(res), _abi.vptr(rec), _abi.vptr(route), C.byref(inc),
        _abi.vptr(counts), _abi.vptr(steps), _abi.vptr(entries), _abi.vptr(rejects),
        _abi.vptr(routes), _abi.vptr(snaps), cap, C.byref(nrt)), "fb_run_cluster_logged")
    out = ClusterOutput(res[:n], rec[:m], route[:m], inc.value, 0.0)
    k = nrt.value
    return ClusterLogs(out, counts[:n], steps, entries, rejects, routes[:k], snaps[:k])


def cluster_fit(n_nodes: int, ctas_per_sm: int = 1, device: int = 0) -> int:
    """How many one-cluster grids of n_nodes fit the device at once."""
    fit = C.c_int32(0)
    fbgpu._check(fbgpu.lib().fb_cluster_fit(device, n_nodes, ctas_per_sm, C.byref(fit)),
                 "fb_cluster_fit")
    return fit.value


def cluster_density(n_copies: int, n_nodes: int, device: int = 0) -> int:
    """fb_cluster_shard_allow_hw_cluster mode for n_copies side by side: 1
    (one CTA per SM) while they fit so, 2 (two per SM) while they fit so,
    else 0 (cooperative grids)."""
    if n_copies <= cluster_fit(n_nodes, 1, device):
        return 1
    if n_copies <= cluster_fit(n_nodes, 2, device):
        return 2
    return 0


def run_clusters(cases, device: int = 0, span: dict | None = None) -> list[ClusterOutput]:
    """Independent cluster simulations at once -- one one-rank shard per case,
    each on its own stream, so their persistent cluster kernels (a few CTAs
    each, bound by the per-epoch exchange latency) run side by side and a
    sweep over seeds x rates x policies fills the GPU (replicas
    amortise the epoch latency).  `cases` holds (rows, cfgs, lb, horizon_us);
    the outputs equal run_cluster's case by case."""
    cases = list(cases)
    if not cases:
        return []
    shards = []
    L = fbgpu.lib()
    try:
        for rows, cfgs, lb, hz in cases:
            shards.append(ClusterShard(rows, cfgs, lb, hz, 0, 1, device))
        # one-cluster grids only while they all fit the device at once (more
        # would run in waves): one CTA per SM while they fit so, else two per
        # SM (each copy slower, twice as many at once), else every shard takes
        # the cooperative grid
        mode = cluster_density(len(cases), max(len(c[1]) for c in cases), device)
        if mode != 1:
            for sh in shards:
                fbgpu._check(L.fb_cluster_shard_allow_hw_cluster(sh._h, mode),
                             "fb_cluster_shard_allow_hw_cluster")
        for sh in shards:
            sh.reset()
        t0 = time.perf_counter()
        for sh in shards:
            sh.launch()
        done = [sh.wait() for sh in shards]
        if span is not None:  # host clock from the first launch to the last completion
            span["ms"] = (time.perf_counter() - t0) * 1000.0
        return [merge_shards([sh.fetch(d)], len(c[1])) for sh, d, c in zip(shards, done, cases)]
    finally:
        for sh in shards:
            sh.close()


class NodeSet:
    """fb_nodes_*: n Node objects (engine.h:111-176) on the device, driven one
    call at a time by a host dispatcher.  Requests are rows of `rows`
    (request_id = row).  `reports`: None, or the LbConfig whose report hook
    (initial report, make_report every report_interval_steps completions,
    delivered report_latency_ms later) the nodes run."""

    def __init__(self, rows: Rows, cfgs, horizon_us: int, reports: LbConfig | None = None,
                 device: int = 0):
        L = fbgpu.lib()
        self._L = L
        self.n = len(cfgs)
        self.n_rows = len(rows)
        self._tr = rows.to_c()
        nc = node_configs_c(cfgs)
        lbc = reports.to_c() if reports is not None else None
        h = C.c_void_p()
        fbgpu._check(L.fb_nodes_create(device, C.byref(self._tr), C.cast(nc, C.c_void_p), self.n,
                                       int(horizon_us), C.byref(lbc) if lbc is not None else None,
                                       C.byref(h)), "fb_nodes_create")
        self._h = h
        self._rep = np.zeros(self.n, _abi.NODE_REPORT_DTYPE)
        self._pab = np.zeros(self.n, np.int64)
        self._st = np.zeros(self.n, _abi.NODE_STATE_DTYPE)

    def close(self) -> None:
        if self._h:
            self._L.fb_nodes_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def advance(self, t: int) -> np.ndarray:
        """Step to time t; per node the newest report delivered by t."""
        fbgpu._check(self._L.fb_nodes_advance(self._h, int(t), _abi.vptr(self._rep)),
                     "fb_nodes_advance")
        return self._rep

    def enqueue(self, t: int, nodes, rows) -> None:
        nd = np.ascontiguousarray(nodes, np.int32)
        rw = np.ascontiguousarray(rows, np.int64)
        fbgpu._check(self._L.fb_nodes_enqueue(self._h, int(t), _abi.vptr(nd), _abi.vptr(rw),
                                              len(nd)), "fb_nodes_enqueue")

    def begin(self, t: int, lo: int = 0, hi: int | None = None) -> None:
        fbgpu._check(self._L.fb_nodes_begin(self._h, int(t), lo, self.n if hi is None else hi),
                     "fb_nodes_begin")

    def drain_rejects(self):
        """[(node, row)] rejected since the last drain, in node order."""
        n = C.c_int64(0)
        st = self._L.fb_nodes_drain_rejects(self._h, None, None, 0, C.byref(n))
        if st == _abi.FB_OK and n.value == 0:
            return []
        nodes = np.zeros(n.value, np.int32)
        rows = np.zeros(n.value, np.int64)
        fbgpu._check(self._L.fb_nodes_drain_rejects(self._h, _abi.vptr(nodes), _abi.vptr(rows),
                                                    n.value, C.byref(n)),
                     "fb_nodes_drain_rejects")
        return list(zip(nodes.tolist(), rows.tolist()))

    def current_pab(self, now: int) -> np.ndarray:
        fbgpu._check(self._L.fb_nodes_current_pab(self._h, int(now), _abi.vptr(self._pab)),
                     "fb_nodes_current_pab")
        return self._pab.copy()

    def state(self) -> np.ndarray:
        fbgpu._check(self._L.fb_nodes_state(self._h, _abi.vptr(self._st)), "fb_nodes_state")
        return self._st.copy()

    def fetch(self) -> ClusterOutput:
        res = np.zeros(self.n, _abi.RESULT_DTYPE)
        rec = np.zeros(max(1, self.n_rows), _abi.RECORD_DTYPE)
        route = np.zeros(max(1, self.n_rows), np.int32)
        inc = C.c_int32(0)
        fbgpu._check(self._L.fb_nodes_fetch(self._h, _abi.vptr(res), _abi.vptr(rec),
                                            _abi.vptr(route), C.byref(inc)), "fb_nodes_fetch")
        return ClusterOutput(res, rec[:self.n_rows], route[:self.n_rows], inc.value)


class HostRouter:
    """The dispatcher's ClusterView (cluster.h:55-73) with apply_report and
    route (cluster.cpp:60-112), on the host."""

    def __init__(self, n: int, lb: LbConfig):
        self.lb = lb
        self.has = [False] * n
        self.t = [-1] * n
        self.pab = [0] * n
        self.wait = [0] * n
        self.run = [0] * n
        self.dec = [0] * n
        self.inc = [0] * n

    def apply(self, i: int, emitted_at: int, pab: int, waiting: int, running: int) -> None:
        if self.has[i] and emitted_at < self.t[i]:
            return
        self.has[i] = True
        self.t[i] = emitted_at
        self.pab[i] = pab
        self.wait[i] = waiting
        self.run[i] = running
        self.dec[i] = 0
        self.inc[i] = 0

    def route(self, prompt: int) -> int:
        n = len(self.pab)
        chosen = -1
        if self.lb.policy == "pab_lb":
            eff = [self.pab[i] - self.dec[i] for i in range(n)]
            for i in range(n):
                if eff[i] >= prompt and (chosen < 0 or eff[i] > eff[chosen]):
                    chosen = i
            if chosen < 0:
                for i in range(n):
                    if chosen < 0 or eff[i] > eff[chosen]:
                        chosen = i
            self.dec[chosen] += prompt
        else:
            best = 0.0
            for i in range(n):
                score = (self.lb.w_waiting * float(self.wait[i] + self.inc[i])
                         + self.lb.w_running * float(self.run[i]))
                if chosen < 0 or score < best:
                    chosen, best = i, score
            self.inc[chosen] += 1
        return chosen


def run_cluster_host(rows: Rows, cfgs, lb: LbConfig, horizon_us: int, device: int = 0,
                     dist=None) -> ClusterOutput:
    """run_cluster (cluster.cpp:134-251) driven from the host over the
    interactive node set: the dispatcher (HostRouter) sees only delivered
    reports, routes with Node::enqueue and reroutes drained rejects -- the
    batched Node surface an external upper-level dispatcher uses.

    Without retry_reroute the loop visits the dispatch epochs (distinct
    arrival times; the nodes advance on their own in between);
    with it, every global event time, and begin_step runs node by node so a
    rerouted request can wake a later node at the same instant.

    `dist` (a torch.distributed group): the nodes are partitioned over the
    ranks (`partition`, one GPU each).  Per dispatch epoch the ranks
    all-gather their nodes' 32-byte load reports (the north star's per-epoch
    allgather of load estimates); routing is replicated on every rank, each
    rank enqueues the requests routed to its own nodes.  With retry_reroute
    the owner of node i broadcasts node i's rejects after its begin_step, so
    every rank reroutes them identically.  Every rank returns the whole
    cluster's output."""
    rank, world = (dist.get_rank(), dist.get_world_size()) if dist is not None else (0, 1)
    n = len(cfgs)
    lo, nl = partition(n, world, rank)
    owner = np.zeros(n, np.int64)
    for r in range(world):
        a, k = partition(n, world, r)
        owner[a:a + k] = r
    nodes = NodeSet(rows, cfgs[lo:lo + nl], horizon_us, lb, device)
    if dist is not None:
        import torch
        cap = max(partition(n, world, r)[1] for r in range(world))
        # NCCL moves device tensors only: the per-epoch report all-gather
        # and the clock all-reduce then run on this rank's GPU (over NVLink
        # between GPUs); gloo (the CPU tests) takes host tensors
        cdev = (torch.device("cuda", device) if dist.get_backend() == "nccl"
                else torch.device("cpu"))
    try:
        view = HostRouter(n, lb)
        arrival = rows.arrival_us
        prompt = rows.prompt_len
        n_rows = len(rows)
        kinf = np.iinfo(np.int64).max
        arr = 0
        retried = set()
        route = np.full(n_rows, -1, np.int32)

        def all_reports(local):
            if dist is None:
                return local
            buf = np.zeros(cap, _abi.NODE_REPORT_DTYPE)
            buf[:nl] = local
            t = torch.from_numpy(buf.view(np.int64).copy()).to(cdev)
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t)
            return np.concatenate([p.cpu().numpy().view(_abi.NODE_REPORT_DTYPE)
                                   [:partition(n, world, r)[1]] for r, p in enumerate(parts)])

        def enqueue(t, targets, qrows):
            targets = np.asarray(targets, np.int64)
            qrows = np.asarray(qrows, np.int64)
            route[qrows] = targets
            mine = (targets >= lo) & (targets < lo + nl)
            nodes.enqueue(t, targets[mine] - lo, qrows[mine])

        def global_min_step_end():
            st = nodes.state()
            busy = st["busy"] != 0
            m = int(st["step_end"][busy].min()) if busy.any() else kinf
            if dist is not None:
                v = torch.tensor([m], dtype=torch.int64, device=cdev)
                dist.all_reduce(v, op=dist.ReduceOp.MIN)
                m = int(v.item())
            return m

        while True:
            t = global_min_step_end() if lb.retry_reroute else kinf
            if arr < n_rows:
                t = min(t, int(arrival[arr]))
            if t == kinf:
                break
            rep = all_reports(nodes.advance(t))
            if not rep["busy"].any() and t >= horizon_us:
                break
            for i in np.nonzero(rep["fresh"])[0]:
                r = rep[i]
                view.apply(int(i), int(r["emitted_at"]), int(r["pab_tokens"]), int(r["waiting"]),
                           int(r["running"]))
            q0 = arr
            targets = []
            while arr < n_rows and arrival[arr] == t:
                targets.append(view.route(int(prompt[arr])))
                arr += 1
            enqueue(t, targets, np.arange(q0, arr))
            if t >= horizon_us:
                continue
            if not lb.retry_reroute:
                nodes.begin(t)
                continue
            progress = True
            while progress:
                progress = False
                for i in range(n):
                    rej = []
                    if owner[i] == rank:
                        nodes.begin(t, i - lo, i - lo + 1)
                        rej = [row for _, row in nodes.drain_rejects()]
                    if dist is not None:
                        box = [rej]
                        dist.broadcast_object_list(box, src=int(owner[i]))
                        rej = box[0]
                    for row in rej:
                        if row not in retried:
                            retried.add(row)
                            enqueue(t, [view.route(int(prompt[row]))], [row])
                            progress = True
        nodes.advance(kinf)  # in-flight steps finish; no step begins past the horizon
        local = nodes.fetch()
        if dist is None:
            parts = [(lo, local)]
        else:
            parts = [None] * world
            dist.all_gather_object(parts, (lo, local))
        res = np.concatenate([o.node_results for _, o in sorted(parts, key=lambda x: x[0])])
        rec = np.zeros(n_rows, _abi.RECORD_DTYPE)
        rec["first_emit_us"] = -1
        for plo, o in parts:
            pn = len(o.node_results)
            own = (route >= plo) & (route < plo + pn)
            rec[own] = o.records[own]
        inc = int(arr < n_rows or any(o.incomplete for _, o in parts))
        res["incomplete"] = inc
        return ClusterOutput(res, rec, route, inc)
    finally:
        nodes.close()


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
