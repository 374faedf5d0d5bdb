// fb_cluster.cuh -- run_cluster (cluster.cpp:134-251) on one or more GPUs.
//
// The global event loop is decomposed at dispatch epochs (the distinct
// arrival times of the trace).  Between epochs the nodes
// are independent run_node machines; their only coupling is the router.  Per
// epoch t_a:
//   A. every node advances through its events before t_a (complete, report,
//      begin) plus a completion at exactly t_a, and publishes a 32-byte
//      NodeReport: its newest report delivered by t_a (constant latency keeps
//      delivery FIFO) and whether it is busy when the clock reaches t_a;
//   -- exchange barrier --
//   B. the router applies the fresh reports of ALL nodes to the balancer's
//      view (apply_report, cluster.cpp:60-73) and routes the arrivals at t_a
//      in trace order (route, cluster.cpp:75-112);
//   C. every idle node that received requests or completed at t_a runs
//      begin_step(t_a).
//
// Layout: one persistent cooperative kernel per GPU, one warp per node (the
// warp keeps its node's live requests in registers on the RR path across
// epochs), W warps per CTA.  The router is replicated per CTA (warp 0, view in
// shared memory) and deterministic, so phase B needs no second exchange.  The
// NodeReports of epoch e go to slot e&1 of an exchange buffer that exists once
// per rank; a warp stores its node's report into every rank's buffer (peer
// memory over NVLink when ranks are GPUs of other processes, opened by CUDA
// IPC) and each CTA then bumps every rank's arrival counter.  A CTA passes
// epoch e when its own rank's counter reaches (e+1) * total CTAs.  Slot
// parity is safe: a CTA can only write slot e&1 again (epoch e+2) after every
// CTA of every rank arrived at barrier e+1, i.e. finished reading epoch e.
// With one rank this is a single-GPU grid barrier on one buffer.
#pragma once

namespace fbgpu {

constexpr int kClusterMaxNodes = 512;
constexpr int kClusterMaxRanks = 8;
constexpr int kClusterMaxWarps = 8;  // nodes (warps) per CTA
constexpr int kXchgHeader = 256;     // [0] arrival counter (u64), padding

// The per-epoch exchange record of one node (fb_node_report in fbgpu.h).
struct __align__(16) NodeReport {
  int64_t t;    // emitted_at of the newest report delivered by t_a, -1 none
  int64_t pab;  // its prefill admission budget
  int32_t waiting, running;
  int32_t fresh;  // a report was delivered since the previous epoch
  int32_t bz;     // node busy when the global clock reaches t_a
};

#ifdef FB_CLUSTER_PROF
__device__ unsigned long long g_cluster_prof[8];
__device__ unsigned long long g_epoch_max[16384];  // per epoch: max over nodes of C(e-1) + A(e)
__device__ unsigned long long g_epoch_max_c[16384];  // max over nodes of phase C(e-1) alone
#endif

struct ClusterParams {
  int32_t n_nodes, lb_policy, interval, report_cap;
  int64_t latency, horizon, n_rows, n_epochs;
  double w_waiting, w_running;
  const int64_t* epoch_t;   // [n_epochs]
  const int64_t* epoch_lo;  // [n_epochs + 1] request ranges
  int32_t* routed;          // [n_local * n_rows] rows in routing order per local node
  int32_t* route_node;      // [n_rows]
  int64_t* rep;             // [n_local * report_cap * 4] in-flight reports
  int64_t* out;             // [0] requests routed, [1] status, [2] epochs run
  int32_t node_lo, n_local;  // this rank: global nodes [node_lo, node_lo + n_local)
  int32_t rank, n_ranks;
  int32_t warps_per_cta, total_ctas;  // total_ctas: over all ranks
  int64_t timeout_ns;                 // exchange wait limit
  unsigned char* xbuf[kClusterMaxRanks];  // exchange buffer of every rank
  int64_t route_stride;               // routed-list capacity per local node
  int32_t retry_reroute, fifo_cap;    // serial engine (retry_reroute)
  int64_t* fifo;                      // [fifo_cap * 6] in-flight reports
  uint8_t* row_state;                 // [n_rows] bit 0 retried, bit 1 ever rejected
  fb_route_log* rlog;                 // routing log (NULL: off)
  double* rsnap;                      // per entry the view snapshot, [rlog_cap * n_nodes]
  int64_t rlog_cap;
  int32_t hw_cluster;  // one rank, the whole grid is one thread-block cluster
  int32_t pad_hw;
};

// Router view (replicated per CTA) + the CTA's routing results.
struct RouterSmem {
  // one thread-block cluster (hw_cluster): every node's NodeReport of epoch
  // e is stored straight into every CTA's slot e&1 (distributed shared
  // memory), so the routers read their reports from local shared memory
  NodeReport xrep[2][kClusterMaxNodes];
  int64_t v_t[kClusterMaxNodes], v_pab[kClusterMaxNodes], v_wait[kClusterMaxNodes];
  int64_t v_run[kClusterMaxNodes], v_dec[kClusterMaxNodes], v_inc[kClusterMaxNodes];
  int32_t v_has[kClusterMaxNodes];
  int64_t n_routed[kClusterMaxWarps];
  int32_t got[kClusterMaxWarps];
  int32_t abort;
  int32_t pad;
};

__device__ __forceinline__ uint64_t* xchg_counter(unsigned char* x) {
  return reinterpret_cast<uint64_t*>(x);
}
__device__ __forceinline__ NodeReport* xchg_reports(unsigned char* x, int n_nodes, int64_t e) {
  return reinterpret_cast<NodeReport*>(x + kXchgHeader) + (e & 1) * n_nodes;
}

__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t* p, bool sys) {
  uint64_t v;
  if (sys) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  } else {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  }
  return v;
}

__device__ __forceinline__ void red_release_add(uint64_t* p, bool sys) {
  if (sys) {
    asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(p) : "memory");
  } else {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(p) : "memory");
  }
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Exchange barrier of epoch e (all CTAs of all ranks).  False on timeout.
__device__ bool cluster_barrier(const ClusterParams& C, RouterSmem& rs, int64_t e) {
  const bool sys = C.n_ranks > 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    // red.release orders this CTA's earlier stores (observed by this thread
    // through the CTA barrier) before the arrival; peer-memory stores of a
    // multi-rank run also get a system-scope fence
    if (sys) __threadfence_system();
    for (int p = 0; p < C.n_ranks; ++p) red_release_add(xchg_counter(C.xbuf[p]), sys);
    const uint64_t target = static_cast<uint64_t>(e + 1) * static_cast<uint64_t>(C.total_ctas);
    const uint64_t* ctr = xchg_counter(C.xbuf[C.rank]);
    if (ld_acquire_u64(ctr, sys) < target) {
      const uint64_t t0 = global_ns();
      for (uint32_t spin = 1; ld_acquire_u64(ctr, sys) < target; ++spin) {
        // the timer read is costly: check the timeout every 64 polls
        if ((spin & 63) == 0 && global_ns() - t0 > static_cast<uint64_t>(C.timeout_ns)) {
          rs.abort = 1;
          break;
        }
      }
    }
  }
  __syncthreads();
  return rs.abort == 0;
}

// One node, owned by one warp for the whole run.
struct ClusterNode {
  Inst w;
  TaskReg tk;
  bool rr;
  int64_t rep_head, rep_tail;
  // the newest report of the FIFO (rep_tail - 1), kept in registers so phase A
  // reads it without a global-memory round trip when it is delivered
  int64_t nt, npab;
  int32_t nwait, nrun;
};

__device__ __forceinline__ void cluster_node_init(const EngineParams& P, const ClusterParams& C,
                                                  int il, unsigned char* smem_warp,
                                                  ClusterNode& nd) {
  Inst& w = nd.w;
  w.id = il;
  w.routed = C.routed + static_cast<int64_t>(il) * C.route_stride;
  w.I = P.inst + il;
  w.S = P.state[il];
  w.toff = w.I->trace_off;
  w.roff = w.I->rec_off;
  w.nreq = w.I->n_req;
  w.horizon = w.I->horizon;
  w.policy = w.I->policy;
  w.max_active = w.I->max_active;
  w.vl = P.vlist + w.roff;
  w.smem = smem_warp;
  nd.tk = TaskReg{};
  w.sd.clear();
  nd.rr = false;
  nd.rep_head = nd.rep_tail = 0;
  nd.nt = -1;
  nd.npab = 0;
  nd.nwait = nd.nrun = 0;
}

// Node::current_pab (engine.cpp:123-125): pab over the node's views at now.
__device__ int64_t node_pab(const EngineParams& P, const ClusterNode& nd, int64_t now) {
  const Inst& w = nd.w;
  const DevInst* I = w.I;
  const double Wm = us_to_ms(I->g_ttft), Tm = us_to_ms(I->g_tpot);
  const int64_t A = visible_count(w);
  const Scratch s = scratch_for(P, w, A);
  int64_t lmin = kInf, lpf = 0;
  if (nd.rr) {  // lane p holds view p
    if (lane_id() < A) {
      const RView v = view_reg(nd.tk, now);
      s.tcost[lane_id()] = pab_term(Wm, Tm, I->sb, I->sc, v.slack, v.ctx);
      lmin = v.slack;
      if (!v.decode) lpf = v.nw;
    }
  } else {
    for (int64_t p = lane_id(); p < A; p += kWarp) {
      const View v = load_view(P, w, p, now);
      s.tcost[p] = pab_term(Wm, Tm, I->sb, I->sc, v.slack, v.ctx);
      lmin = v.slack < lmin ? v.slack : lmin;
      if (!v.decode) lpf += v.nw;
    }
  }
  __syncwarp();
  const int64_t min_slack = warp_min_i64(lmin);
  const int64_t pf = warp_sum_small(lpf);
  const double r_tasks = ordered_fold(s.tcost, static_cast<int>(A));
  return pab_close(Wm, Tm, I->sa, I->sb, I->sc, A > 0, min_slack, r_tasks, pf);
}

// make_report (cluster.cpp:50-58) into the node's in-flight FIFO.
__device__ void node_report(const EngineParams& P, const ClusterParams& C, ClusterNode& nd,
                            int64_t now, int32_t* status) {
  const Inst& w = nd.w;
  const int64_t pab = C.lb_policy == FB_LB_PAB ? node_pab(P, nd, now) : 0;
  if (nd.rep_tail - nd.rep_head >= C.report_cap) {
    *status = FB_ERR_CAPACITY;
  } else {
    if (lane_id() == 0) {
      int64_t* r = C.rep + (w.id * C.report_cap + nd.rep_tail % C.report_cap) * 4;
      r[0] = now;
      r[1] = pab;
      r[2] = w.S.n_live - w.S.n_active;  // waiting_count (engine.h:133-135)
      r[3] = w.S.n_active;                // running_count
    }
    nd.nt = now;
    nd.npab = pab;
    nd.nwait = w.S.n_live - w.S.n_active;
    nd.nrun = w.S.n_active;
    nd.rep_tail++;
  }
  __syncwarp();
}

// Node::complete_step on the current path (+ the step report).
__device__ __forceinline__ void node_complete(const EngineParams& P, const ClusterParams& C,
                                              ClusterNode& nd, bool report, int32_t* status) {
  Inst& w = nd.w;
  const int64_t t = w.S.step_end;
  w.S.t_last = t;
  if (nd.rr) {
    complete_rr(P, w, nd.tk);
  } else {
    complete_step(P, w);
  }
  if (report && C.interval > 0 && w.S.step_counter % static_cast<uint64_t>(C.interval) == 0)
    node_report(P, C, nd, t, status);
}

// Node::begin_step with the RR / memory path switch of run_instance.
__device__ __forceinline__ void node_begin(const EngineParams& P, ClusterNode& nd, int64_t t) {
  Inst& w = nd.w;
  const int64_t upcoming = w.S.n_live + (w.S.arr - w.S.pulled);
  if (nd.rr && upcoming > kWarp) {
    rr_spill(P, w, nd.tk);
    w.sd.clear();
    nd.rr = false;
  } else if (!nd.rr && upcoming <= kWarp) {
    rr_load(P, w, nd.tk);
    w.sd.clear();
    nd.rr = true;
    w.S.paths |= kPathRegister;
  }
  if (nd.rr) {
    const Scratch s = carve_scratch(w.smem, kSmemSlots);
    if (begin_rr(P, w, nd.tk, t, s) < 0) {  // keys outside the packed range
      rr_spill(P, w, nd.tk);
      nd.rr = false;
      begin_step(P, w, t);
      w.S.paths |= kPathMemory;
    }
  } else {
    begin_step(P, w, t);
    w.S.paths |= kPathMemory;
  }
}

// Phase A for one node: events before t_a, the completion at t_a, and the
// NodeReport of epoch e stored into every rank's exchange buffer.
__device__ void node_phase_a(const EngineParams& P, const ClusterParams& C, ClusterNode& nd,
                             RouterSmem& rs, int64_t e, int64_t t_a, int32_t* cmp_out,
                             int32_t* status) {
  Inst& w = nd.w;
  while (w.S.busy && w.S.step_end < t_a) {
    const int64_t t = w.S.step_end;
    node_complete(P, C, nd, true, status);
    if (t < w.horizon) node_begin(P, nd, t);
  }
  const int32_t bz = w.S.busy != 0;  // busy when the global clock reaches t_a
  const int32_t cmp = bz && w.S.step_end == t_a;
  if (cmp) node_complete(P, C, nd, true, status);  // begin at t_a waits for the routing
  *cmp_out = cmp;
  NodeReport nr;
  nr.t = -1;
  nr.pab = 0;
  nr.waiting = nr.running = 0;
  nr.fresh = 0;
  nr.bz = bz;
  int64_t h = nd.rep_head;
  if (h < nd.rep_tail) {  // newest report delivered by t_a
    // emit times increase along the FIFO and the latency is constant, so the
    // delivered reports are a prefix: when the newest is delivered (always
    // with zero latency) they all are -- one read instead of a walk
    if (nd.nt + C.latency <= t_a) {  // from the register copy
      h = nd.rep_tail;
      if (h > nd.rep_head) {
        nr.t = nd.nt;
        nr.pab = nd.npab;
        nr.waiting = nd.nwait;
        nr.running = nd.nrun;
        nr.fresh = 1;
      }
    } else {
      while (h < nd.rep_tail) {
        const int64_t* q = C.rep + (w.id * C.report_cap + h % C.report_cap) * 4;
        if (q[0] + C.latency > t_a) break;
        ++h;
      }
      if (h > nd.rep_head) {
        const int64_t* r = C.rep + (w.id * C.report_cap + (h - 1) % C.report_cap) * 4;
        nr.t = r[0];
        nr.pab = r[1];
        nr.waiting = static_cast<int32_t>(r[2]);
        nr.running = static_cast<int32_t>(r[3]);
        nr.fresh = 1;
      }
    }
  }
  nd.rep_head = h;
  if (C.hw_cluster) {
    // lane p stores the report into CTA p's shared memory (DSMEM)
    if (lane_id() < C.total_ctas) {
      const uint32_t local = static_cast<uint32_t>(
          __cvta_generic_to_shared(&rs.xrep[e & 1][C.node_lo + w.id]));
      uint32_t remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                   : "=r"(remote) : "r"(local), "r"(static_cast<uint32_t>(lane_id())));
      const int4* v = reinterpret_cast<const int4*>(&nr);
      const int4 a = v[0], b = v[1];
      asm volatile("st.shared::cluster.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(remote), "r"(a.x),
                   "r"(a.y), "r"(a.z), "r"(a.w) : "memory");
      asm volatile("st.shared::cluster.v4.s32 [%0+16], {%1, %2, %3, %4};" ::"r"(remote), "r"(b.x),
                   "r"(b.y), "r"(b.z), "r"(b.w) : "memory");
    }
  } else if (lane_id() < C.n_ranks) {  // lane p stores into rank p's buffer
    NodeReport* dst = xchg_reports(C.xbuf[lane_id()], C.n_nodes, e) + C.node_lo + w.id;
    *dst = nr;
    if (C.n_ranks > 1) __threadfence_system();
  }
  __syncwarp();
}

// The 32-byte report of node i: from this CTA's shared memory (hw_cluster)
// or from the exchange buffer in L2.
__device__ __forceinline__ void load_report(const NodeReport* all, int i, bool local, int4& a,
                                            int4& b) {
  const int4* rp = reinterpret_cast<const int4*>(all + i);
  if (local) {
    a = rp[0];
    b = rp[1];
  } else {
    a = __ldcg(rp);
    b = __ldcg(rp + 1);
  }
}

// Horizon rule (cluster.cpp:191-192): at t_a >= horizon the global loop only
// runs while some node is busy.  Every CTA of every rank evaluates the same
// reports, so all stop at the same epoch.
__device__ __forceinline__ bool cluster_stopped(const ClusterParams& C, const NodeReport* all,
                                                int64_t t_a) {
  if (t_a < C.horizon) return false;
  int mine = 0;
  for (int i = threadIdx.x; i < C.n_nodes; i += blockDim.x) {
    int4 a, b;
    load_report(all, i, C.hw_cluster != 0, a, b);
    mine |= b.w;  // bz
  }
  return __syncthreads_or(mine) == 0;
}

// route (cluster.cpp:75-112) of one request by warp 0 over the replicated
// view: pab_lb picks the largest effective budget among nodes that fit the
// prompt (else overall), count_lb the smallest weighted count; ties to the
// lowest node id.  Updates the view's local decrements.  Returns the node.
__device__ __forceinline__ int cluster_pick(const ClusterParams& C, RouterSmem& rs,
                                            int64_t prompt, int64_t log_k = -1, int64_t t = 0,
                                            int64_t row = 0, const DevState* states = nullptr) {
  const int n = C.n_nodes;
  int chosen;
  if (C.lb_policy == FB_LB_PAB) {
    // best effective budget among nodes that fit the prompt, else overall;
    // ties to the lowest node id
    int64_t bf = INT64_MIN, ba = INT64_MIN;
    int idf = INT32_MAX, ida = INT32_MAX;
    for (int i = lane_id(); i < n; i += kWarp) {
      const int64_t eff = rs.v_pab[i] - rs.v_dec[i];
      if (eff > ba) {
        ba = eff;
        ida = i;
      }
      if (eff >= prompt && eff > bf) {
        bf = eff;
        idf = i;
      }
    }
  #pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int64_t b2 = __shfl_xor_sync(kFull, bf, o);
      const int i2 = __shfl_xor_sync(kFull, idf, o);
      if (b2 > bf || (b2 == bf && i2 < idf)) {
        bf = b2;
        idf = i2;
      }
      const int64_t a2 = __shfl_xor_sync(kFull, ba, o);
      const int j2 = __shfl_xor_sync(kFull, ida, o);
      if (a2 > ba || (a2 == ba && j2 < ida)) {
        ba = a2;
        ida = j2;
      }
    }
    chosen = idf != INT32_MAX ? idf : ida;
    if (lane_id() == 0) rs.v_dec[chosen] += prompt;
  } else {
    double best = 0.0;
    int idb = INT32_MAX;
    for (int i = lane_id(); i < n; i += kWarp) {
      const double score =
          dadd(dmul(C.w_waiting, static_cast<double>(rs.v_wait[i] + rs.v_inc[i])),
               dmul(C.w_running, static_cast<double>(rs.v_run[i])));
      if (idb == INT32_MAX || score < best) {
        best = score;
        idb = i;
      }
    }
  #pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double b2 = __shfl_xor_sync(kFull, best, o);
      const int i2 = __shfl_xor_sync(kFull, idb, o);
      if (i2 != INT32_MAX && (idb == INT32_MAX || b2 < best || (b2 == best && i2 < idb))) {
        best = b2;
        idb = i2;
      }
    }
    chosen = idb;
    if (lane_id() == 0) rs.v_inc[chosen] += 1;
  }
  __syncwarp();
  if (log_k >= 0 && C.rlog && log_k < C.rlog_cap) {
    // route_request's routing-log entry (cluster.cpp:171-175): the view
    // snapshot taken after the decision's decrement / increment
    for (int i = lane_id(); i < n; i += kWarp) {
      C.rsnap[log_k * n + i] =
          C.lb_policy == FB_LB_PAB
              ? static_cast<double>(rs.v_pab[i] - rs.v_dec[i])
              : dadd(dmul(C.w_waiting, static_cast<double>(rs.v_wait[i] + rs.v_inc[i])),
                     dmul(C.w_running, static_cast<double>(rs.v_run[i])));
    }
    if (lane_id() == 0) {
      fb_route_log& e = C.rlog[log_k];
      e.t_us = t;
      e.req = static_cast<int32_t>(row);
      e.node = chosen;
      // the target's log position at enqueue (serial engine: a rerouted
      // arrival can fall between a node's events of one instant)
      e.rej_before = states ? static_cast<int32_t>(states[chosen].n_rejected) : -1;
      e.steps_before = states ? static_cast<int32_t>(states[chosen].step_counter) : -1;
    }
    __syncwarp();
  }
  return chosen;
}

// Phase B (warp 0 of each CTA): reports -> view, route the epoch's arrivals.
// q_lo / q_hi / prompt0: the epoch's request range and its first prompt,
// loaded by the caller before phase A so their latency is off the critical
// path (the router runs between the barrier and phase C of every epoch).
__device__ void cluster_route(const EngineParams& P, const ClusterParams& C, RouterSmem& rs,
                              const NodeReport* all, int64_t e, int node_base, int64_t q_lo,
                              int64_t q_hi, int64_t prompt0) {
  const int n = C.n_nodes;
  for (int i = lane_id(); i < n; i += kWarp) {
    // the whole 32-byte report in two 16-byte loads (one round trip)
    int4 a, b;
    load_report(all, i, C.hw_cluster != 0, a, b);
    if (b.z) {  // fresh
      const int64_t t = (static_cast<int64_t>(a.y) << 32) | static_cast<uint32_t>(a.x);
      if (!(rs.v_has[i] && t < rs.v_t[i])) {
        rs.v_has[i] = 1;
        rs.v_t[i] = t;
        rs.v_pab[i] = (static_cast<int64_t>(a.w) << 32) | static_cast<uint32_t>(a.z);
        rs.v_wait[i] = b.x;
        rs.v_run[i] = b.y;
        rs.v_dec[i] = 0;
        rs.v_inc[i] = 0;
      }
    }
  }
  __syncwarp();
  for (int64_t q = q_lo; q < q_hi; ++q) {
    const int64_t prompt = q == q_lo ? prompt0 : P.prompt[q];
    const int chosen = cluster_pick(C, rs, prompt, blockIdx.x == 0 ? q : -1, C.epoch_t[e], q);
    if (lane_id() == 0) {
      if (blockIdx.x == 0) C.route_node[q] = chosen;
      const int k = chosen - node_base;  // Node::enqueue, on the owning CTA
      if (k >= 0 && k < C.warps_per_cta && chosen - C.node_lo < C.n_local) {
        const int64_t j = rs.n_routed[k];
        C.routed[static_cast<int64_t>(chosen - C.node_lo) * C.route_stride + j] =
            static_cast<int32_t>(q);
        rs.n_routed[k] = j + 1;
        rs.got[k] = 1;
      }
    }
    __syncwarp();
  }
}

// One persistent grid per cluster simulation.  kCtasPerSm = 1: one CTA per
// SM (the single-simulation form, C5 184 ms); 2 (<= 128 registers): two per
// SM for many simulations side by side -- a single copy slows to 237 ms, but
// twice as many copies fit at once (32 copies in 257 ms: 30.4 M node-steps/s
// against 16 copies in 206 ms: 19.0 M, tools/c5_replicas.py).
template <int kCtasPerSm>
__global__ void __launch_bounds__(kWarp * kClusterMaxWarps, kCtasPerSm)
cluster_kernel(const __grid_constant__ EngineParams P, const __grid_constant__ ClusterParams C) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RouterSmem& rs = *reinterpret_cast<RouterSmem*>(smem_raw);
  const int warp = threadIdx.x / kWarp;
  unsigned char* my = smem_raw + ((sizeof(RouterSmem) + 15) / 16) * 16 +
                      static_cast<size_t>(warp) * kSmemSlots * kScratchBytesPerSlot;
  const int il = blockIdx.x * C.warps_per_cta + warp;  // local node of this warp
  const bool owner = il < C.n_local;
  const int node_base = C.node_lo + blockIdx.x * C.warps_per_cta;  // global id of warp 0's node
  for (int i = threadIdx.x; i < C.n_nodes; i += blockDim.x) {
    rs.v_has[i] = 0;
    rs.v_t[i] = -1;
    rs.v_pab[i] = rs.v_wait[i] = rs.v_run[i] = rs.v_dec[i] = rs.v_inc[i] = 0;
  }
  if (threadIdx.x < kClusterMaxWarps) {
    rs.n_routed[threadIdx.x] = 0;
    rs.got[threadIdx.x] = 0;
  }
  if (threadIdx.x == 0) rs.abort = 0;
  int32_t status = FB_OK;
  ClusterNode nd;
  if (C.hw_cluster) {
    // distributed shared memory may be written only once every CTA of the
    // cluster is known to be running: one cluster barrier before the first
    // remote report store (the initial report below)
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
  if (owner) {
    cluster_node_init(P, C, il, my, nd);
    node_report(P, C, nd, 0, &status);  // initial report (cluster.cpp:198)
  }
  __syncthreads();
  int64_t e = 0;
  bool ok = true;
#ifdef FB_CLUSTER_PROF
  uint64_t pt0 = global_ns(), pacc[6] = {0, 0, 0, 0, 0, 0};
  // [0] phase A (own node), [1] barrier wait, [2] report read + stop test,
  // [3] routing, [4] phase C (own node), [5] epochs
#define CPT(k) { const uint64_t n_ = global_ns(); pacc[k] += n_ - pt0; pt0 = n_; }
  uint64_t wt0 = pt0;  // this warp's node work since the previous routing
#else
#define CPT(k)
#endif
  for (; e < C.n_epochs; ++e) {
    const int64_t t_a = C.epoch_t[e];
    // the router's inputs for this epoch, fetched ahead of phase A
    int64_t q_lo = 0, q_hi = 0, prompt0 = 0;
    if (warp == 0) {
      q_lo = C.epoch_lo[e];
      q_hi = C.epoch_lo[e + 1];
      prompt0 = q_lo < q_hi ? P.prompt[q_lo] : 0;
    }
    int32_t cmp = 0;
    if (owner) node_phase_a(P, C, nd, rs, e, t_a, &cmp, &status);
#ifdef FB_CLUSTER_PROF
    if (owner && lane_id() == 0 && e < 16384) {
      const unsigned long long busy = global_ns() - wt0;
      atomicMax(&g_epoch_max[e], busy);
      atomicAdd(&g_cluster_prof[7], busy);
    }
#endif
    CPT(0)
    if (C.hw_cluster) {
      // the grid is one thread-block cluster: the hardware cluster barrier
      // (release / acquire at cluster scope orders the report stores of
      // every CTA before the reads) replaces the global-memory arrival count
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else if (!(ok = cluster_barrier(C, rs, e))) {
      break;
    }
    CPT(1)
    const NodeReport* all =
        C.hw_cluster ? rs.xrep[e & 1] : xchg_reports(C.xbuf[C.rank], C.n_nodes, e);
    if (cluster_stopped(C, all, t_a)) break;
    CPT(2)
    if (warp == 0) cluster_route(P, C, rs, all, e, node_base, q_lo, q_hi, prompt0);
    __syncthreads();
    CPT(3)
#ifdef FB_CLUSTER_PROF
    wt0 = global_ns();
#endif
    if (owner && (rs.got[warp] || cmp)) {  // Node::enqueue (visible at t_a), begin_step(t_a)
      Inst& w = nd.w;
      w.S.arr = rs.n_routed[warp];
      w.S.t_last = t_a;
      if (!w.S.busy && t_a < w.horizon) node_begin(P, nd, t_a);
    }
    __syncwarp();
    if (owner && lane_id() == 0) rs.got[warp] = 0;
#ifdef FB_CLUSTER_PROF
    if (owner && lane_id() == 0 && e + 1 < 16384)
      atomicMax(&g_epoch_max_c[e + 1], global_ns() - wt0);
#endif
    CPT(4)
  }
#ifdef FB_CLUSTER_PROF
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int k = 0; k < 5; ++k) g_cluster_prof[k] += pacc[k];
    g_cluster_prof[5] += e;
  }
#endif
  if (owner) {
    Inst& w = nd.w;
    if (ok) {  // all arrivals routed (or the loop stopped): run to quiescence
      while (w.S.busy) {
        const int64_t t = w.S.step_end;
        node_complete(P, C, nd, false, &status);
        if (t < w.horizon) node_begin(P, nd, t);
      }
    }
    if (nd.rr) rr_spill(P, w, nd.tk);
    if (lane_id() == 0) {
      w.S.done = 1;
      w.S.incomplete = (w.S.busy || w.S.pulled < w.S.arr || w.S.n_live > 0) ? 1 : 0;
      P.state[il] = w.S;
      if (status != FB_OK)
        atomicMax(reinterpret_cast<unsigned long long*>(C.out + 1),
                  static_cast<unsigned long long>(status));
    }
  }
  if (threadIdx.x == 0) {
    if (!ok)
      atomicMax(reinterpret_cast<unsigned long long*>(C.out + 1),
                static_cast<unsigned long long>(FB_ERR_TIMEOUT));
    if (blockIdx.x == 0) {
      C.out[0] = e < C.n_epochs ? C.epoch_lo[e] : C.n_rows;
      C.out[2] = e;
      C.out[3] = C.out[0];  // routing-log entries: one per routed request
    }
  }
}

// ---------------------------------------------------------- retry_reroute
//
// run_cluster with lb.retry_reroute (cluster.cpp:222-237): a request that PAB
// admission rejects is routed once more, at once, and may wake a node that
// was already passed at the same instant -- a dependency inside one event
// time that the epoch decomposition above cannot express.  This engine
// replays the reference's global loop literally: one warp walks every node in
// index order at each event time t (the minimum over busy step ends, the next
// arrival and the head of the report FIFO), with the nodes' state in global
// memory between visits and the memory path for every step.  One rank only.

struct SerialSmem {
  RouterSmem rs;
  int64_t n_routed[kClusterMaxNodes];  // routed-list length per node
  int64_t n_log;                       // routing-log entries
};

// The node's warp-uniform state, loaded from P.state (the memory path keeps
// everything else in global memory).
__device__ __forceinline__ void serial_load(const EngineParams& P, const ClusterParams& C,
                                            int i, unsigned char* scratch, ClusterNode& nd) {
  cluster_node_init(P, C, i, scratch, nd);
}

__device__ __forceinline__ void serial_store(const EngineParams& P, const ClusterNode& nd) {
  if (lane_id() == 0) P.state[nd.w.id] = nd.w.S;
  __syncwarp();
}

// make_report (cluster.cpp:50-58) into the global FIFO: [deliver_at,
// emitted_at, pab, waiting, running, node].
__device__ void serial_report(const EngineParams& P, const ClusterParams& C, ClusterNode& nd,
                              int64_t now, int64_t head, int64_t& tail, int32_t* status) {
  const Inst& w = nd.w;
  const int64_t pab = C.lb_policy == FB_LB_PAB ? node_pab(P, nd, now) : 0;
  if (tail - head >= C.fifo_cap) {
    *status = FB_ERR_CAPACITY;
  } else {
    if (lane_id() == 0) {
      int64_t* r = C.fifo + (tail % C.fifo_cap) * 6;
      r[0] = now + C.latency;
      r[1] = now;
      r[2] = pab;
      r[3] = w.S.n_live - w.S.n_active;
      r[4] = w.S.n_active;
      r[5] = w.id;
    }
    ++tail;
  }
  __syncwarp();
}

// route_request (cluster.cpp:171-175): pick, log the target, Node::enqueue.
__device__ __forceinline__ void serial_route(const EngineParams& P, const ClusterParams& C,
                                             SerialSmem& ss, int64_t row, int64_t t) {
  const int chosen = cluster_pick(C, ss.rs, P.prompt[row], ss.n_log, t, row, P.state);
  __syncwarp();
  if (lane_id() == 0) ss.n_log++;
  if (lane_id() == 0) {
    C.route_node[row] = chosen;
    const int64_t j = ss.n_routed[chosen];
    C.routed[static_cast<int64_t>(chosen) * C.route_stride + j] = static_cast<int32_t>(row);
    ss.n_routed[chosen] = j + 1;
  }
  __syncwarp();
}

__global__ void __launch_bounds__(kWarp, 1)
cluster_serial_kernel(const __grid_constant__ EngineParams P,
                      const __grid_constant__ ClusterParams C) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SerialSmem& ss = *reinterpret_cast<SerialSmem*>(smem_raw);
  RouterSmem& rs = ss.rs;
  unsigned char* scratch = smem_raw + ((sizeof(SerialSmem) + 15) / 16) * 16;
  const int n = C.n_nodes;
  for (int i = lane_id(); i < n; i += kWarp) {
    rs.v_has[i] = 0;
    rs.v_t[i] = -1;
    rs.v_pab[i] = rs.v_wait[i] = rs.v_run[i] = rs.v_dec[i] = rs.v_inc[i] = 0;
    ss.n_routed[i] = 0;
  }
  if (lane_id() == 0) ss.n_log = 0;
  __syncwarp();
  int32_t status = FB_OK;
  int64_t head = 0, tail = 0;
  ClusterNode nd;
  for (int i = 0; i < n; ++i) {  // initial reports (cluster.cpp:178)
    serial_load(P, C, i, scratch, nd);
    serial_report(P, C, nd, 0, head, tail, &status);
  }
  int64_t arr = 0, iters = 0;
  for (;; ++iters) {
    int64_t lt = kInf;
    for (int i = lane_id(); i < n; i += kWarp) {
      const DevState& st = P.state[i];
      if (st.busy && st.step_end < lt) lt = st.step_end;
    }
    int64_t t = warp_min_i64(lt);
    const bool any_busy = t != kInf;
    if (arr < C.n_rows && P.arrival[arr] < t) t = P.arrival[arr];
    if (head < tail && C.fifo[(head % C.fifo_cap) * 6] < t) t = C.fifo[(head % C.fifo_cap) * 6];
    if (t == kInf || (!any_busy && t >= C.horizon)) break;
    // 1) step completions in node order, then the boundary report
    for (int i = 0; i < n; ++i) {
      const DevState& st = P.state[i];
      if (!(st.busy && st.step_end == t)) continue;
      serial_load(P, C, i, scratch, nd);
      nd.w.S.t_last = t;
      complete_step(P, nd.w);
      if (C.interval > 0 && nd.w.S.step_counter % static_cast<uint64_t>(C.interval) == 0)
        serial_report(P, C, nd, t, head, tail, &status);
      serial_store(P, nd);
    }
    // 2) report deliveries due by t (apply_report, cluster.cpp:60-73)
    while (head < tail && C.fifo[(head % C.fifo_cap) * 6] <= t) {
      const int64_t* r = C.fifo + (head % C.fifo_cap) * 6;
      const int i = static_cast<int>(r[5]);
      if (lane_id() == 0 && !(rs.v_has[i] && r[1] < rs.v_t[i])) {
        rs.v_has[i] = 1;
        rs.v_t[i] = r[1];
        rs.v_pab[i] = r[2];
        rs.v_wait[i] = r[3];
        rs.v_run[i] = r[4];
        rs.v_dec[i] = 0;
        rs.v_inc[i] = 0;
      }
      __syncwarp();
      ++head;
    }
    // 3) arrivals at exactly t, in trace order
    for (; arr < C.n_rows && P.arrival[arr] == t; ++arr) serial_route(P, C, ss, arr, t);
    // 4) begin_step on idle nodes; a first rejection is routed again at once
    if (t < C.horizon) {
      bool progress = true;
      while (progress) {
        progress = false;
        for (int i = 0; i < n; ++i) {
          if (P.state[i].busy) continue;
          serial_load(P, C, i, scratch, nd);
          Inst& w = nd.w;
          w.S.arr = ss.n_routed[i];
          const int64_t p0 = w.S.pulled, rej0 = w.S.n_rejected;
          if (w.S.pulled < w.S.arr || w.S.n_live > 0) {
            w.S.t_last = t;
            begin_step(P, w, t);
            w.S.paths |= kPathMemory;
          }
          const int64_t p1 = w.S.pulled;
          const bool rejected = w.S.n_rejected != rej0;
          serial_store(P, nd);
          if (!rejected) continue;
          // drain_rejects: the pulled rows flagged rejected, in pull order (a
          // stale flag can only sit on a row already retried, so it is inert)
          for (int64_t q = p0; q < p1; ++q) {
            const int64_t row = w.routed[q];
            if (!(P.flags[w.roff + row] & FB_REC_REJECTED)) continue;
            const uint8_t rsv = C.row_state[row];
            if (lane_id() == 0) C.row_state[row] = rsv | 3;
            __syncwarp();
            if (!(rsv & 1) && C.retry_reroute) {
              serial_route(P, C, ss, row, t);
              progress = true;
            }
          }
        }
      }
    }
  }
  for (int i = 0; i < n; ++i) {
    serial_load(P, C, i, scratch, nd);
    Inst& w = nd.w;
    w.S.arr = ss.n_routed[i];
    if (lane_id() == 0) {
      w.S.done = 1;
      w.S.incomplete = (w.S.busy || w.S.pulled < w.S.arr || w.S.n_live > 0) ? 1 : 0;
      P.state[i] = w.S;
    }
    __syncwarp();
  }
  if (lane_id() == 0) {
    C.out[0] = arr;
    C.out[1] = status;
    C.out[2] = iters;
    C.out[3] = ss.n_log;
  }
}

// ------------------------------------------------------ interactive node set
//
// fb_nodes_*: the Node surface (engine.h:111-176) of n nodes at once, driven
// one host call at a time by an external dispatcher (e.g. run_cluster's loop,
// cluster.cpp:134-251, on the host).  Between calls every node's state lives
// in global memory (the memory path for every step, like the serial engine);
// one warp per node per call.

enum NodesOp : int32_t {
  kNodesInit = 0,     // initial report at t = 0 (cluster.cpp:178)
  kNodesAdvance = 1,  // events before t, the completion at t, newest delivered report
  kNodesBegin = 2,    // begin_step(t) on the idle nodes of [lo, hi), collect rejects
  kNodesPab = 3,      // current_pab(t)
  kNodesState = 4,    // busy / step_end / waiting / running / steps / live
  kNodesFinish = 5,   // done + incomplete flags for the result fetch
};

struct NodesIo {
  int32_t op, lo, hi, reports;  // reports: emit make_report (cluster.cpp:50-58)
  int64_t t;
  int64_t* rep_ht;    // [n * 2] report FIFO head / tail per node
  int64_t* rej;       // [n * rej_cap] rows rejected since the last drain
  int64_t* n_rej;     // [n]
  int64_t rej_cap;
  int64_t* out;       // [n * 6] per-node output of the op
  int32_t* status;
};

__global__ void __launch_bounds__(kWarp * kClusterMaxWarps)
nodes_kernel(const __grid_constant__ EngineParams P, const __grid_constant__ ClusterParams C,
             const __grid_constant__ NodesIo io) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x / kWarp;
  const int i = blockIdx.x * kClusterMaxWarps + warp;
  if (i >= C.n_local || i < io.lo || i >= io.hi) return;
  unsigned char* my = smem_raw + static_cast<size_t>(warp) * kSmemSlots * kScratchBytesPerSlot;
  ClusterNode nd;
  cluster_node_init(P, C, i, my, nd);
  nd.rep_head = io.rep_ht[2 * i];
  nd.rep_tail = io.rep_ht[2 * i + 1];
  Inst& w = nd.w;
  int32_t status = FB_OK;
  int64_t* o = io.out + static_cast<int64_t>(i) * 6;
  const int64_t t = io.t;
  auto complete = [&]() {  // Node::complete_step + the boundary report
    const int64_t te = w.S.step_end;
    w.S.t_last = te;
    complete_step(P, w);
    if (io.reports && C.interval > 0 &&
        w.S.step_counter % static_cast<uint64_t>(C.interval) == 0) {
      // a full FIFO whose head is delivered by t loses nothing by dropping
      // it: this newer report is delivered by t as well and supersedes it
      if (nd.rep_tail - nd.rep_head >= C.report_cap && te + C.latency <= t) nd.rep_head++;
      node_report(P, C, nd, te, &status);
    }
  };
  if (io.op == kNodesInit) {
    if (io.reports) node_report(P, C, nd, 0, &status);
  } else if (io.op == kNodesAdvance) {
    while (w.S.busy && w.S.step_end < t) {  // the node's own events before t
      const int64_t te = w.S.step_end;
      complete();
      if (te < w.horizon && (w.S.pulled < w.S.arr || w.S.n_live > 0)) {
        w.S.t_last = te;
        begin_step(P, w, te);
        w.S.paths |= kPathMemory;
      }
    }
    const int32_t bz = w.S.busy != 0;
    if (bz && w.S.step_end == t) complete();  // begin at t waits for the dispatcher
    // the newest report delivered by t (FIFO per node, constant latency)
    int64_t h = nd.rep_head, rt = -1, rp = 0, rw = 0, rr = 0, fresh = 0;
    while (h < nd.rep_tail) {
      const int64_t* r = C.rep + (w.id * C.report_cap + h % C.report_cap) * 4;
      if (r[0] + C.latency > t) break;
      rt = r[0];
      rp = r[1];
      rw = r[2];
      rr = r[3];
      fresh = 1;
      ++h;
    }
    nd.rep_head = h;
    if (lane_id() == 0) {
      o[0] = rt;
      o[1] = rp;
      o[2] = rw;
      o[3] = rr;
      o[4] = fresh;
      o[5] = bz;
    }
  } else if (io.op == kNodesBegin) {
    if (!w.S.busy) {
      const int64_t p0 = w.S.pulled, rej0 = w.S.n_rejected;
      if (w.S.pulled < w.S.arr || w.S.n_live > 0) {
        w.S.t_last = t;
        begin_step(P, w, t);
        w.S.paths |= kPathMemory;
      }
      if (w.S.n_rejected != rej0) {
        // drain_rejects' contents: the pulled rows flagged rejected, in pull
        // order (a row flagged at an earlier visit was drained then)
        int64_t n = io.n_rej[i];
        for (int64_t q = p0; q < w.S.pulled; ++q) {
          const int64_t row = w.routed[q];
          if (!(P.flags[w.roff + row] & FB_REC_REJECTED)) continue;
          if (lane_id() == 0) {
            if (n < io.rej_cap) io.rej[static_cast<int64_t>(i) * io.rej_cap + n] = row;
            C.row_state[row] |= 2;  // ever rejected (metrics.cpp:96-98)
          }
          ++n;
        }
        if (lane_id() == 0) io.n_rej[i] = n;
        if (n > io.rej_cap) status = FB_ERR_CAPACITY;
      }
    }
  } else if (io.op == kNodesPab) {
    const int64_t pab = node_pab(P, nd, t);  // Node::current_pab (engine.cpp:123-125)
    if (lane_id() == 0) o[0] = pab;
  } else if (io.op == kNodesState) {
    if (lane_id() == 0) {
      o[0] = w.S.busy;
      o[1] = w.S.step_end;
      o[2] = w.S.n_live - w.S.n_active;  // waiting_count (engine.h:133-135)
      o[3] = w.S.n_active;               // running_count
      o[4] = static_cast<int64_t>(w.S.step_counter);  // steps_completed
      o[5] = (w.S.pulled < w.S.arr || w.S.n_live > 0) ? 1 : 0;  // has_live_requests
    }
  } else if (io.op == kNodesFinish) {
    w.S.done = 1;
    w.S.incomplete = (w.S.busy || w.S.pulled < w.S.arr || w.S.n_live > 0) ? 1 : 0;
  }
  __syncwarp();
  if (lane_id() == 0) {
    P.state[i] = w.S;
    io.rep_ht[2 * i] = nd.rep_head;
    io.rep_ht[2 * i + 1] = nd.rep_tail;
    if (status != FB_OK) atomicExch(io.status, status);
  }
}

// Node::enqueue(r, t) (engine.cpp:92-105) for (node, row) pairs in order:
// the row joins the node's routed list (pending until its next begin_step).
__global__ void nodes_enqueue_kernel(const __grid_constant__ EngineParams P,
                                     const __grid_constant__ ClusterParams C, int64_t t,
                                     const int32_t* node, const int64_t* row, int64_t n,
                                     int32_t* status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int64_t k = 0; k < n; ++k) {
    const int i = node[k];
    DevState& st = P.state[i];
    const int64_t j = st.arr;
    if (j >= C.route_stride) {
      *status = FB_ERR_CAPACITY;
      return;
    }
    C.routed[static_cast<int64_t>(i) * C.route_stride + j] = static_cast<int32_t>(row[k]);
    // a row routed here again after a rejection starts unrejected (the
    // record keeps "ever rejected" in row_state)
    P.flags[P.inst[i].rec_off + row[k]] &= ~static_cast<uint32_t>(FB_REC_REJECTED);
    st.arr = j + 1;
    st.t_last = t;
    C.route_node[row[k]] = i;
  }
}

}  // namespace fbgpu
