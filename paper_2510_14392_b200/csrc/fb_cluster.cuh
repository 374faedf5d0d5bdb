// fb_cluster.cuh -- run_cluster (cluster.cpp:134-251) in one persistent CTA.
//
// The global event loop is decomposed at dispatch epochs (the distinct
// arrival times of the trace): between epochs the nodes are
// independent run_node machines (their only coupling is the router), so per
// epoch t_a
//   A. every warp advances its nodes through all events before t_a (complete,
//      report, begin) plus a completion at exactly t_a, then pops the node's
//      newest report due by t_a (constant latency keeps delivery FIFO);
//   B. warp 0 applies the fresh reports to the balancer's view (decrements
//      reset, apply_report cluster.cpp:60-73) and routes the arrivals at t_a
//      in trace order (route, cluster.cpp:75-112) with warp arg-max/arg-min;
//   C. every idle node that received requests runs begin_step(t_a).
// Nodes use the warp engine's memory path; the load estimate is K5 (pab over
// the node's views, ordered fold).
#pragma once

namespace fbgpu {

constexpr int kClusterWarps = 32;
constexpr int kClusterMaxNodes = 512;

struct ClusterParams {
  int32_t n_nodes, lb_policy, interval, report_cap;
  int64_t latency, horizon, n_rows, n_epochs;
  double w_waiting, w_running;
  const int64_t* epoch_t;   // [n_epochs]
  const int64_t* epoch_lo;  // [n_epochs + 1] request ranges
  int32_t* routed;          // [n_nodes * n_rows] rows in routing order per node
  int32_t* route_node;      // [n_rows]
  int64_t* rep;             // [n_nodes * report_cap * 4] in-flight reports
  int64_t* out;             // [0] requests routed, [1] status
};

struct ClusterSmem {
  // balancer view (NodeView, cluster.h:55-69)
  int64_t v_t[kClusterMaxNodes], v_pab[kClusterMaxNodes], v_wait[kClusterMaxNodes];
  int64_t v_run[kClusterMaxNodes], v_dec[kClusterMaxNodes], v_inc[kClusterMaxNodes];
  int32_t v_has[kClusterMaxNodes];
  // per-node bookkeeping mirrored from DevState
  int64_t step_end[kClusterMaxNodes];
  int64_t n_routed[kClusterMaxNodes];
  int64_t rep_head[kClusterMaxNodes], rep_tail[kClusterMaxNodes];
  int32_t busy[kClusterMaxNodes];
  int32_t got[kClusterMaxNodes];  // routed something this epoch
  // fresh report of this epoch
  int64_t f_t[kClusterMaxNodes], f_pab[kClusterMaxNodes], f_wait[kClusterMaxNodes],
      f_run[kClusterMaxNodes];
  int32_t fresh[kClusterMaxNodes];
  int32_t bz[kClusterMaxNodes];   // busy when the global clock reaches t_a
  int32_t cmp[kClusterMaxNodes];  // completed exactly at t_a
  int32_t status;
};

__device__ __forceinline__ Inst cluster_node(const EngineParams& P, const ClusterParams& C,
                                             int i, unsigned char* smem_warp) {
  Inst w;
  w.id = i;
  w.routed = C.routed + static_cast<int64_t>(i) * C.n_rows;
  w.I = P.inst + i;
  w.S = P.state[i];
  w.toff = w.I->trace_off;
  w.roff = w.I->rec_off;
  w.nreq = w.I->n_req;
  w.horizon = w.I->horizon;
  w.policy = w.I->policy;
  w.max_active = w.I->max_active;
  w.vl = P.vlist + w.roff;
  w.smem = smem_warp;
  return w;
}

// Node::current_pab (engine.cpp:123-125): pab over the node's views at now.
__device__ int64_t node_pab(const EngineParams& P, const Inst& w, int64_t now) {
  const DevInst* I = w.I;
  const double Wm = us_to_ms(I->g_ttft), Tm = us_to_ms(I->g_tpot);
  const int64_t A = visible_count(w);
  const Scratch s = scratch_for(P, w, A);
  int64_t lmin = kInf, lpf = 0;
  for (int64_t p = lane_id(); p < A; p += kWarp) {
    const View v = load_view(P, w, p, now);
    s.tcost[p] = pab_term(Wm, Tm, I->sb, I->sc, v.slack, v.ctx);
    lmin = v.slack < lmin ? v.slack : lmin;
    if (!v.decode) lpf += v.nw;
  }
  __syncwarp();
  const int64_t min_slack = warp_min_i64(lmin);
  const int64_t pf = warp_sum_small(lpf);
  const double r_tasks = ordered_fold(s.tcost, static_cast<int>(A));
  return pab_close(Wm, Tm, I->sa, I->sb, I->sc, A > 0, min_slack, r_tasks, pf);
}

// make_report (cluster.cpp:50-58) into the node's in-flight FIFO.
__device__ void node_report(const EngineParams& P, const ClusterParams& C, ClusterSmem& cs,
                            const Inst& w, int64_t now) {
  const int i = static_cast<int>(w.id);
  const int64_t pab = C.lb_policy == FB_LB_PAB ? node_pab(P, w, now) : 0;
  if (lane_id() == 0) {
    const int64_t tail = cs.rep_tail[i];
    if (tail - cs.rep_head[i] >= C.report_cap) {
      cs.status = FB_ERR_CAPACITY;
    } else {
      int64_t* r = C.rep + (static_cast<int64_t>(i) * C.report_cap + tail % C.report_cap) * 4;
      r[0] = now;
      r[1] = pab;
      r[2] = w.S.n_live - w.S.n_active;  // waiting_count (engine.h:133-135)
      r[3] = w.S.n_active;                // running_count
      cs.rep_tail[i] = tail + 1;
    }
  }
  __syncwarp();
}

// Runs node events before t_a (and the completion at t_a when `at_too`).
__device__ void advance_node(const EngineParams& P, const ClusterParams& C, ClusterSmem& cs,
                             Inst& w, int64_t t_a, bool at_too) {
  while (w.S.busy && (w.S.step_end < t_a || (at_too && w.S.step_end == t_a))) {
    const int64_t t = w.S.step_end;
    w.S.t_last = t;
    complete_step(P, w);
    if (C.interval > 0 && w.S.step_counter % static_cast<uint64_t>(C.interval) == 0)
      node_report(P, C, cs, w, t);
    if (t == t_a) break;  // begin at t_a waits for the routing
    if (t < w.horizon) begin_step(P, w, t);
  }
}

__global__ void __launch_bounds__(kWarp * kClusterWarps, 1)
cluster_kernel(const __grid_constant__ EngineParams P, const __grid_constant__ ClusterParams C) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ClusterSmem& cs = *reinterpret_cast<ClusterSmem*>(smem_raw);
  unsigned char* scratch_base = smem_raw + ((sizeof(ClusterSmem) + 15) / 16) * 16;
  const int warp = threadIdx.x / kWarp;
  unsigned char* my = scratch_base + static_cast<size_t>(warp) * kSmemSlots * kScratchBytesPerSlot;
  const int n = C.n_nodes;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    cs.v_has[i] = 0;
    cs.v_t[i] = -1;
    cs.v_pab[i] = cs.v_wait[i] = cs.v_run[i] = cs.v_dec[i] = cs.v_inc[i] = 0;
    cs.busy[i] = 0;
    cs.step_end[i] = 0;
    cs.n_routed[i] = 0;
    cs.rep_head[i] = cs.rep_tail[i] = 0;
    cs.fresh[i] = 0;
  }
  if (threadIdx.x == 0) cs.status = FB_OK;
  __syncthreads();
  // initial reports at t = 0 (cluster.cpp:198)
  for (int i = warp; i < n; i += kClusterWarps) {
    const Inst w = cluster_node(P, C, i, my);
    node_report(P, C, cs, w, 0);
  }
  __syncthreads();
  int64_t e = 0;
  for (; e < C.n_epochs; ++e) {
    const int64_t t_a = C.epoch_t[e];
    // A: advance, deliver
    for (int i = warp; i < n; i += kClusterWarps) {
      if (cs.busy[i] && cs.step_end[i] <= t_a) {
        Inst w = cluster_node(P, C, i, my);
        advance_node(P, C, cs, w, t_a, false);
        const bool busy_at = w.S.busy != 0;  // busy when the clock reaches t_a
        const bool ends_at = busy_at && w.S.step_end == t_a;
        advance_node(P, C, cs, w, t_a, true);
        if (lane_id() == 0) {
          P.state[i] = w.S;
          cs.busy[i] = w.S.busy;
          cs.step_end[i] = w.S.step_end;
          cs.bz[i] = busy_at;
          cs.cmp[i] = ends_at;  // owes a begin_step(t_a) after the routing
        }
      } else if (lane_id() == 0) {
        cs.bz[i] = cs.busy[i];
        cs.cmp[i] = 0;
      }
      if (lane_id() == 0) {
        int64_t h = cs.rep_head[i];
        bool got = false;
        while (h < cs.rep_tail[i]) {
          const int64_t* r = C.rep + (static_cast<int64_t>(i) * C.report_cap + h % C.report_cap) * 4;
          if (r[0] + C.latency > t_a) break;
          cs.f_t[i] = r[0];
          cs.f_pab[i] = r[1];
          cs.f_wait[i] = r[2];
          cs.f_run[i] = r[3];
          got = true;
          ++h;
        }
        cs.rep_head[i] = h;
        cs.fresh[i] = got;
        cs.got[i] = 0;
      }
      __syncwarp();
    }
    __syncthreads();
    // horizon: at t_a >= horizon the global loop only runs while a node is
    // busy (cluster.cpp:191-192); nodes never begin at or after the horizon
    bool any_busy = false;
    for (int i = 0; i < n; ++i) any_busy |= cs.bz[i] != 0;
    if (t_a >= C.horizon && !any_busy) break;
    // B: reports -> view, route in trace order (warp 0)
    if (warp == 0) {
      for (int i = lane_id(); i < n; i += kWarp) {
        if (cs.fresh[i] && !(cs.v_has[i] && cs.f_t[i] < cs.v_t[i])) {
          cs.v_has[i] = 1;
          cs.v_t[i] = cs.f_t[i];
          cs.v_pab[i] = cs.f_pab[i];
          cs.v_wait[i] = cs.f_wait[i];
          cs.v_run[i] = cs.f_run[i];
          cs.v_dec[i] = 0;
          cs.v_inc[i] = 0;
        }
      }
      __syncwarp();
      for (int64_t q = C.epoch_lo[e]; q < C.epoch_lo[e + 1]; ++q) {
        const int64_t prompt = P.prompt[q];
        int chosen;
        if (C.lb_policy == FB_LB_PAB) {
          // best effective budget among nodes that fit the prompt, else overall;
          // ties to the lowest node id
          int64_t bf = INT64_MIN, ba = INT64_MIN;
          int idf = INT32_MAX, ida = INT32_MAX;
          for (int i = lane_id(); i < n; i += kWarp) {
            const int64_t eff = cs.v_pab[i] - cs.v_dec[i];
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
          if (lane_id() == 0) cs.v_dec[chosen] += prompt;
        } else {
          double best = 0.0;
          int idb = INT32_MAX;
          for (int i = lane_id(); i < n; i += kWarp) {
            const double score =
                dadd(dmul(C.w_waiting, static_cast<double>(cs.v_wait[i] + cs.v_inc[i])),
                     dmul(C.w_running, static_cast<double>(cs.v_run[i])));
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
          if (lane_id() == 0) cs.v_inc[chosen] += 1;
        }
        if (lane_id() == 0) {
          const int64_t k = cs.n_routed[chosen];
          C.routed[static_cast<int64_t>(chosen) * C.n_rows + k] = static_cast<int32_t>(q);
          cs.n_routed[chosen] = k + 1;
          cs.got[chosen] = 1;
          C.route_node[q] = chosen;
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // C: enqueue (visible at t_a) and begin_step(t_a) on idle nodes
    for (int i = warp; i < n; i += kClusterWarps) {
      if (cs.got[i] || cs.cmp[i]) {
        Inst w = cluster_node(P, C, i, my);
        w.S.arr = cs.n_routed[i];  // Node::enqueue
        w.S.t_last = t_a;
        if (!w.S.busy && t_a < w.horizon) begin_step(P, w, t_a);
        if (lane_id() == 0) {
          P.state[i] = w.S;
          cs.busy[i] = w.S.busy;
          cs.step_end[i] = w.S.step_end;
        }
        __syncwarp();
      }
    }
    __syncthreads();
  }
  // all arrivals routed (or the loop stopped): run every node to quiescence
  for (int i = warp; i < n; i += kClusterWarps) {
    Inst w = cluster_node(P, C, i, my);
    advance_node(P, C, cs, w, kInf, false);
    if (lane_id() == 0) {
      w.S.done = 1;
      w.S.incomplete = (w.S.busy || w.S.pulled < w.S.arr || w.S.n_live > 0) ? 1 : 0;
      P.state[i] = w.S;
    }
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    C.out[0] = e < C.n_epochs ? C.epoch_lo[e] : C.n_rows;
    C.out[1] = cs.status;
  }
}

}  // namespace fbgpu
