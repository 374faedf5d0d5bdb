// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// C-ABI shim over the UNMODIFIED reference library (/root/reference/proj/src,
// compiled in place by oracle/Makefile into oracle/_ref/libfbsim_ref.so).  It
// lets the Python tests and bench.py's reference arm drive the real fbsim code
// with the same POD structs as include/fbgpu.h (prefix ref_ instead of fb_).
//
// run_node is driven through the public Node API exactly like run_node's own
// loop (engine.cpp:266-288) so that every BatchPlan can be captured from
// complete_step() (engine.h:102-106); with check != 0 the captured event log is
// compared field-by-field against the real run_node's log.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <deque>
#include <memory>
#include <set>
#include <exception>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "fbsim/cluster.h"
#include "fbsim/engine.h"
#include "fbsim/metrics.h"
#include "fbsim/rng.h"
#include "fbsim/sched.h"
#include "fbsim/workload.h"

extern "C" {
#include "../include/fbgpu.h"
#include "../include/fbgpu_digest.h"
}

using namespace fbsim;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& what) {
  g_err = what;
  return code;
}

int map_exception(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ValidationError*>(&e)) return FB_ERR_VALIDATION;
  if (dynamic_cast<const UsageError*>(&e)) return FB_ERR_USAGE;
  if (dynamic_cast<const ConfigError*>(&e)) return FB_ERR_CONFIG;
  if (dynamic_cast<const ParseError*>(&e)) return FB_ERR_PARSE;
  return FB_ERR_USAGE;
}

CostModel to_model(const fb_cost_model& m) { return CostModel{m.a_ms, m.b_ms, m.c_ms}; }

SchedulerConfig to_sched(const fb_scheduler_config& c) {
  SchedulerConfig s;
  s.policy = static_cast<Policy>(c.policy);
  s.token_budget = c.token_budget;
  s.max_chunk = c.max_chunk;
  s.model = to_model(c.model);
  return s;
}

EngineConfig to_engine(const fb_engine_config& c) {
  EngineConfig e;
  e.scheduler = to_sched(c.scheduler);
  e.truth_model = to_model(c.truth_model);
  e.noise.amplitude = c.noise_amplitude;
  e.noise.seed = c.noise_seed;
  e.global_slo = {c.global_ttft_us, c.global_tpot_us};
  e.max_active = c.max_active;
  return e;
}

std::vector<TaskView> to_views(const fb_task_view* t, int64_t n) {
  std::vector<TaskView> v(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    v[i].request_id = t[i].request_id;
    v[i].phase = t[i].phase == FB_PHASE_DECODE ? Phase::kDecode : Phase::kPrefill;
    v[i].slack = t[i].slack_us;
    v[i].new_tokens_available = t[i].new_tokens;
    v[i].context = t[i].context;
    v[i].arrival_seq = t[i].arrival_seq;
    v[i].tpot_slo = t[i].tpot_us;
  }
  return v;
}

Trace instance_trace(const fb_trace* rows, const fb_instance& inst) {
  Trace tr;
  tr.requests.resize(static_cast<size_t>(inst.n_req));
  for (int64_t i = 0; i < inst.n_req; ++i) {
    const int64_t k = inst.trace_off + i;
    Request& r = tr.requests[i];
    r.id = i;
    r.arrival = rows->arrival_us[k];
    r.prompt_len = rows->prompt_len[k];
    r.output_len = rows->output_len[k];
    r.ttft_slo = rows->ttft_us[k];
    r.tpot_slo = rows->tpot_us[k];
  }
  return tr;
}

bool same_event(const Event& a, const Event& b) {
  return a.t == b.t && a.kind == b.kind && a.req_id == b.req_id &&
         a.arrival == b.arrival && a.prompt_len == b.prompt_len &&
         a.output_len == b.output_len && a.pab_tokens == b.pab_tokens &&
         a.step == b.step && a.new_tokens == b.new_tokens &&
         a.context_tokens == b.context_tokens &&
         std::memcmp(&a.predicted_ms, &b.predicted_ms, sizeof(double)) == 0 &&
         std::memcmp(&a.actual_ms, &b.actual_ms, sizeof(double)) == 0 &&
         a.token_idx == b.token_idx;
}

// Fills records from the reference's own request_reports (metrics.cpp:60-116).
void fill_records(const std::vector<EventLog>& logs, const Trace& tr,
                  fb_record* rec) {
  for (size_t i = 0; i < tr.requests.size(); ++i) {
    rec[i] = fb_record{-1, 0.0, 0.0, 0, 0u};
  }
  for (const auto& r : request_reports(logs)) {
    fb_record& o = rec[r.req_id];
    uint32_t f = FB_REC_ARRIVED;
    if (r.rejected) f |= FB_REC_REJECTED;
    if (r.finished) f |= FB_REC_FINISHED;
    if (r.met_ttft) f |= FB_REC_MET_TTFT;
    if (r.met_tpot) f |= FB_REC_MET_TPOT;
    for (size_t j = 1; j < r.emits.size(); ++j) {  // acceptance.cpp:106-111
      if (r.emits[j] > r.ttft_slo + r.tpot_slo * static_cast<TimeUs>(j)) {
        f |= FB_REC_ENV_MISS;
        break;
      }
    }
    o.first_emit_us = r.has_ttft() ? r.arrival + r.emits[0] : -1;
    o.max_tpot_ms = r.max_tpot_ms();
    o.max_tpot_alt_ms = r.max_tpot_alt_ms();
    o.tokens_emitted = r.tokens_emitted;
    o.flags = f;
  }
}

// run_node mirrored through the Node API (engine.cpp:266-288).
int run_mirror(const fb_trace* rows, const fb_instance& inst,
               const fb_log_opts* lo, fb_instance_result* res, fb_record* rec,
               fb_log_counts* counts, fb_step_log* steps, fb_plan_entry* entries,
               fb_reject_log* rejects, int check) {
  constexpr TimeUs kInf = std::numeric_limits<TimeUs>::max();
  const Trace tr = instance_trace(rows, inst);
  const EngineConfig cfg = to_engine(inst.cfg);
  Node node(0, cfg);
  std::vector<BatchPlan> plans;
  std::vector<double> actuals;
  size_t arr = 0;
  const auto& reqs = tr.requests;
  TimeUs t_last = 0;
  for (;;) {
    const TimeUs t_step = node.busy() ? node.step_end() : kInf;
    const TimeUs t_arr = arr < reqs.size() ? reqs[arr].arrival : kInf;
    const TimeUs t = std::min(t_step, t_arr);
    if (t == kInf) break;
    if (!node.busy() && t >= inst.horizon_us) break;
    t_last = t;
    if (node.busy() && t_step == t) {
      StepOutcome out = node.complete_step();
      plans.push_back(std::move(out.plan));
      actuals.push_back(out.actual_ms);
    }
    while (arr < reqs.size() && reqs[arr].arrival == t) {
      node.enqueue(reqs[arr], reqs[arr].arrival);
      ++arr;
    }
    if (!node.busy() && t < inst.horizon_us) node.begin_step(t);
  }
  EventLog log = std::move(node.log());
  log.incomplete = node.has_live_requests() || arr < reqs.size();

  if (check) {
    const EventLog real = run_node(tr, cfg, inst.horizon_us);
    if (real.events.size() != log.events.size() || real.incomplete != log.incomplete)
      return fail(FB_ERR_VALIDATION, "mirror diverged from run_node (size)");
    for (size_t i = 0; i < real.events.size(); ++i)
      if (!same_event(real.events[i], log.events[i]))
        return fail(FB_ERR_VALIDATION, "mirror diverged from run_node at event " +
                                           std::to_string(i));
  }

  std::memset(res, 0, sizeof(*res));
  if (counts) std::memset(counts, 0, sizeof(*counts));
  uint64_t h = FB_DIGEST_INIT;
  size_t step = 0;
  for (const auto& e : log.events) {
    if (e.kind == EventKind::kArrival) {
      res->n_arrived++;
    } else if (e.kind == EventKind::kAdmissionReject) {
      res->n_rejected++;
      h = fb_digest_reject(h, e.t, static_cast<uint32_t>(e.req_id), e.pab_tokens);
      if (rejects && counts) {
        if (counts->rejects < lo->reject_cap) {
          fb_reject_log& rl = rejects[counts->rejects++];
          rl.t_us = e.t;
          rl.pab_tokens = e.pab_tokens;
          rl.req = static_cast<int32_t>(e.req_id);
          rl.step = static_cast<int32_t>(step);  // batch_starts logged before it
        } else {
          counts->truncated = 1;
        }
      }
    } else if (e.kind == EventKind::kBatchStart) {
      const BatchPlan& p = plans.at(step);
      uint64_t esum = 0;
      for (size_t k = 0; k < p.entries.size(); ++k)
        esum ^= fb_digest_entry(static_cast<uint32_t>(k),
                                static_cast<uint32_t>(p.entries[k].request_id),
                                static_cast<uint32_t>(p.entries[k].new_tokens));
      const double actual = actuals.at(step);
      h = fb_digest_step(h, e.t, static_cast<uint32_t>(p.entries.size()), esum,
                         e.predicted_ms, actual);
      res->sum_entries += static_cast<int64_t>(p.entries.size());
      res->sum_new_tokens += e.new_tokens;
      if (steps && counts) {
        if (counts->steps < lo->step_cap &&
            counts->entries + static_cast<int64_t>(p.entries.size()) <= lo->entry_cap) {
          fb_step_log& sl = steps[counts->steps++];
          sl.t_us = e.t;
          sl.duration_us = std::max<TimeUs>(1, ms_to_us(actual));
          sl.predicted_ms = e.predicted_ms;
          sl.actual_ms = actual;
          sl.total_new = e.new_tokens;
          sl.total_ctx = e.context_tokens;
          sl.init_budget_ms = p.init_time_budget_ms;
          sl.entry_off = counts->entries;
          sl.n_entries = static_cast<int32_t>(p.entries.size());
          for (const auto& pe : p.entries) {
            entries[counts->entries].req = static_cast<int32_t>(pe.request_id);
            entries[counts->entries].new_tokens = pe.new_tokens;
            counts->entries++;
          }
        } else {
          counts->truncated = 1;
        }
      }
      ++step;
    }
  }
  res->steps = node.steps_completed();
  res->plan_digest = h;
  res->end_time_us = t_last;
  res->incomplete = log.incomplete ? 1 : 0;
  res->status = FB_OK;
  res->sum_visible = -1;  // not observable through the reference API
  if (rec) fill_records({log}, tr, rec);
  return FB_OK;
}

// Plan digest + counters of one node log (same definition as run_mirror).
void digest_node_log(const EventLog& log, const std::vector<BatchPlan>& plans,
                     const std::vector<double>& actuals, uint64_t steps_completed,
                     fb_instance_result* res) {
  std::memset(res, 0, sizeof(*res));
  uint64_t h = FB_DIGEST_INIT;
  size_t step = 0;
  for (const auto& e : log.events) {
    if (e.kind == EventKind::kArrival) {
      res->n_arrived++;
    } else if (e.kind == EventKind::kAdmissionReject) {
      res->n_rejected++;
      h = fb_digest_reject(h, e.t, static_cast<uint32_t>(e.req_id), e.pab_tokens);
    } else if (e.kind == EventKind::kBatchStart) {
      const BatchPlan& p = plans.at(step);
      uint64_t esum = 0;
      for (size_t k = 0; k < p.entries.size(); ++k)
        esum ^= fb_digest_entry(static_cast<uint32_t>(k),
                                static_cast<uint32_t>(p.entries[k].request_id),
                                static_cast<uint32_t>(p.entries[k].new_tokens));
      h = fb_digest_step(h, e.t, static_cast<uint32_t>(p.entries.size()), esum,
                         e.predicted_ms, actuals.at(step));
      res->sum_entries += static_cast<int64_t>(p.entries.size());
      res->sum_new_tokens += e.new_tokens;
      ++step;
    }
  }
  res->steps = steps_completed;
  res->plan_digest = h;
  res->incomplete = log.incomplete ? 1 : 0;
  res->sum_visible = -1;
  res->end_time_us = -1;
}

}  // namespace

extern "C" {

// run_cluster (cluster.cpp:134-251) mirrored through Node / route /
// apply_report / make_report so that every node's plans can be captured;
// with check != 0 the node logs and routing decisions are compared with the
// real run_cluster.  route_node[i] = node of request i (-1: never routed).
int ref_run_cluster(const fb_trace* rows, const fb_engine_config* cfgs, int32_t n_nodes,
                    const fb_lb_config* lbc, int64_t horizon, fb_instance_result* node_results,
                    fb_record* records, int32_t* route_node, int32_t* incomplete_out,
                    int check) {
  try {
    constexpr TimeUs kInf = std::numeric_limits<TimeUs>::max();
    fb_instance whole{};
    whole.trace_off = 0;
    whole.n_req = rows->n_rows;
    const Trace tr = instance_trace(rows, whole);
    LbConfig lb;
    lb.policy = lbc->policy == FB_LB_PAB ? LbPolicy::kPabLb : LbPolicy::kCountLb;
    lb.report_interval_steps = lbc->report_interval_steps;
    lb.report_latency = lbc->report_latency_us;
    lb.w_waiting = lbc->w_waiting;
    lb.w_running = lbc->w_running;
    lb.retry_reroute = lbc->retry_reroute != 0;
    std::vector<EngineConfig> ecfg;
    for (int i = 0; i < n_nodes; ++i) ecfg.push_back(to_engine(cfgs[i]));
    const int n = n_nodes;
    std::vector<std::unique_ptr<Node>> nodes;
    for (int i = 0; i < n; ++i) nodes.push_back(std::make_unique<Node>(i, ecfg[i]));
    std::vector<std::vector<BatchPlan>> plans(n);
    std::vector<std::vector<double>> actuals(n);
    std::vector<int> route(tr.requests.size(), -1);
    ClusterView view;
    view.nodes.resize(n);
    struct InFlight {
      TimeUs deliver_at;
      MetricReport report;
    };
    std::deque<InFlight> deliveries;
    std::set<std::int64_t> retried;
    auto emit_report = [&](const Node& node, TimeUs now) {
      deliveries.push_back({now + lb.report_latency, make_report(node, now, lb.policy)});
    };
    std::vector<int> routed_nodes;  // in routing order
    auto route_request = [&](const Request& r, TimeUs now) {
      const int target = fbsim::route(view, r, lb);
      route[static_cast<size_t>(r.id)] = target;
      routed_nodes.push_back(target);
      nodes[static_cast<size_t>(target)]->enqueue(r, now);
    };
    for (const auto& node : nodes) emit_report(*node, 0);
    size_t arr = 0;
    const auto& reqs = tr.requests;
    for (;;) {
      TimeUs t = kInf;
      for (const auto& node : nodes)
        if (node->busy()) t = std::min(t, node->step_end());
      const bool any_busy = t != kInf;
      if (arr < reqs.size()) t = std::min(t, reqs[arr].arrival);
      if (!deliveries.empty()) t = std::min(t, deliveries.front().deliver_at);
      if (t == kInf) break;
      if (!any_busy && t >= horizon) break;
      for (int i = 0; i < n; ++i) {
        auto& node = nodes[static_cast<size_t>(i)];
        if (node->busy() && node->step_end() == t) {
          StepOutcome out = node->complete_step();
          plans[i].push_back(std::move(out.plan));
          actuals[i].push_back(out.actual_ms);
          if (lb.report_interval_steps > 0 &&
              node->steps_completed() % static_cast<std::uint64_t>(lb.report_interval_steps) == 0)
            emit_report(*node, t);
        }
      }
      while (!deliveries.empty() && deliveries.front().deliver_at <= t) {
        apply_report(view, deliveries.front().report);
        deliveries.pop_front();
      }
      while (arr < reqs.size() && reqs[arr].arrival == t) {
        route_request(reqs[arr], t);
        ++arr;
      }
      if (t < horizon) {
        bool progress = true;
        while (progress) {
          progress = false;
          for (auto& node : nodes) {
            if (!node->busy()) node->begin_step(t);
            for (const auto& r : node->drain_rejects()) {
              if (lb.retry_reroute && retried.insert(r.id).second) {
                route_request(r, t);
                progress = true;
              }
            }
          }
        }
      }
    }
    bool live = arr < reqs.size();
    for (auto& node : nodes) live = live || node->has_live_requests();
    std::vector<EventLog> logs;
    for (auto& node : nodes) {
      EventLog lg = std::move(node->log());
      lg.incomplete = live;
      logs.push_back(std::move(lg));
    }
    if (check) {
      const ClusterResult real = run_cluster(tr, ecfg, lb, horizon);
      if (real.incomplete != live) return fail(FB_ERR_VALIDATION, "cluster mirror: incomplete");
      if (real.routing.size() != routed_nodes.size())
        return fail(FB_ERR_VALIDATION, "cluster mirror: routing size");
      for (size_t k = 0; k < routed_nodes.size(); ++k)
        if (real.routing[k].node != routed_nodes[k])
          return fail(FB_ERR_VALIDATION, "cluster mirror: routing differs");
      for (int i = 0; i < n; ++i) {
        const auto& a = real.node_logs[static_cast<size_t>(i)].events;
        const auto& b = logs[static_cast<size_t>(i)].events;
        if (a.size() != b.size()) return fail(FB_ERR_VALIDATION, "cluster mirror: log size");
        for (size_t k = 0; k < a.size(); ++k)
          if (!same_event(a[k], b[k])) return fail(FB_ERR_VALIDATION, "cluster mirror: event");
      }
    }
    for (int i = 0; i < n; ++i)
      if (node_results)
        digest_node_log(logs[static_cast<size_t>(i)], plans[i], actuals[i],
                        nodes[static_cast<size_t>(i)]->steps_completed(), &node_results[i]);
    if (records) fill_records(logs, tr, records);
    if (route_node)
      for (size_t k = 0; k < route.size(); ++k) route_node[k] = route[k];
    if (incomplete_out) *incomplete_out = live ? 1 : 0;
    return FB_OK;
  } catch (const std::exception& e) {
    return map_exception(e);
  }
}

const char* ref_last_error(void) { return g_err.c_str(); }

// The reference's own JSONL event log (run_node + save_event_log,
// engine.cpp:395-451) of one instance, copied into buf (len_out = bytes;
// FB_ERR_CAPACITY when cap is too small).
int ref_event_log(const fb_trace* rows, const fb_instance* inst, const char* tmp_path, char* buf,
                  int64_t cap, int64_t* len_out) {
  try {
    const Trace tr = instance_trace(rows, *inst);
    const EventLog log = run_node(tr, to_engine(inst->cfg), inst->horizon_us);
    save_event_log(log, tmp_path);
    FILE* f = std::fopen(tmp_path, "rb");
    if (!f) return fail(FB_ERR_PARSE, "cannot reopen event log");
    std::string s;
    char tmp[65536];
    size_t k;
    while ((k = std::fread(tmp, 1, sizeof(tmp), f)) > 0) s.append(tmp, k);
    std::fclose(f);
    *len_out = static_cast<int64_t>(s.size());
    if (static_cast<int64_t>(s.size()) > cap) return fail(FB_ERR_CAPACITY, "buffer too small");
    std::memcpy(buf, s.data(), s.size());
    return FB_OK;
  } catch (const std::exception& e) {
    return map_exception(e);
  }
}

// The real run_cluster's outputs in the reference's own file formats: every
// node's save_event_log JSONL, then save_routing_log's JSONL (with the view
// snapshots), concatenated into buf; offsets[0..n_nodes+1] delimit them.
int ref_cluster_logs(const fb_trace* rows, const fb_engine_config* cfgs, int32_t n_nodes,
                     const fb_lb_config* lbc, int64_t horizon, const char* tmp_path, char* buf,
                     int64_t cap, int64_t* offsets, int64_t* len_out) {
  try {
    fb_instance whole{};
    whole.trace_off = 0;
    whole.n_req = rows->n_rows;
    const Trace tr = instance_trace(rows, whole);
    LbConfig lb;
    lb.policy = lbc->policy == FB_LB_PAB ? LbPolicy::kPabLb : LbPolicy::kCountLb;
    lb.report_interval_steps = lbc->report_interval_steps;
    lb.report_latency = lbc->report_latency_us;
    lb.w_waiting = lbc->w_waiting;
    lb.w_running = lbc->w_running;
    lb.retry_reroute = lbc->retry_reroute != 0;
    std::vector<EngineConfig> ecfg;
    for (int i = 0; i < n_nodes; ++i) ecfg.push_back(to_engine(cfgs[i]));
    const ClusterResult res = run_cluster(tr, ecfg, lb, horizon);
    auto slurp = [&](std::string& out) {
      FILE* f = std::fopen(tmp_path, "rb");
      if (!f) throw ParseError("cannot reopen log");
      char tmp[65536];
      size_t k;
      while ((k = std::fread(tmp, 1, sizeof(tmp), f)) > 0) out.append(tmp, k);
      std::fclose(f);
    };
    std::string all;
    offsets[0] = 0;
    for (int i = 0; i < n_nodes; ++i) {
      save_event_log(res.node_logs[static_cast<size_t>(i)], tmp_path);
      slurp(all);
      offsets[i + 1] = static_cast<int64_t>(all.size());
    }
    save_routing_log(res.routing, lb.policy, tmp_path);
    slurp(all);
    offsets[n_nodes + 1] = static_cast<int64_t>(all.size());
    *len_out = static_cast<int64_t>(all.size());
    if (*len_out > cap) return fail(FB_ERR_CAPACITY, "buffer too small");
    std::memcpy(buf, all.data(), all.size());
    return FB_OK;
  } catch (const std::exception& e) {
    return map_exception(e);
  }
}

// The reference's own load_event_log + replay_check (engine.cpp:290-393,
// 453-520) of a JSONL file: the violations joined by '\n' into buf.
int ref_replay_check(const char* path, char* buf, int64_t cap, int64_t* len_out,
                     int64_t* n_violations) {
  try {
    const ReplayReport rep = replay_check(load_event_log(path));
    std::string s;
    for (const auto& v : rep.violations) {
      s += v;
      s += '\n';
    }
    *n_violations = static_cast<int64_t>(rep.violations.size());
    *len_out = static_cast<int64_t>(s.size());
    if (static_cast<int64_t>(s.size()) > cap) return fail(FB_ERR_CAPACITY, "buffer too small");
    std::memcpy(buf, s.data(), s.size());
    return FB_OK;
  } catch (const std::exception& e) {
    return map_exception(e);
  }
}

// The reference's envelope-lead series (metrics.cpp:137-169) of one
// instance: run_node, request_reports, envelope_lead_series(bucket).
int ref_lead_series(const fb_trace* rows, const fb_instance* inst, int64_t bucket_us,
                    int64_t* lead_out, int64_t cap, int64_t* n_out) {
  try {
    const Trace tr = instance_trace(rows, *inst);
    const EventLog log = run_node(tr, to_engine(inst->cfg), inst->horizon_us);
    const std::vector<EventLog> logs{log};
    const auto series = envelope_lead_series(request_reports(logs), bucket_us);
    *n_out = static_cast<int64_t>(series.size());
    if (*n_out > cap) return fail(FB_ERR_CAPACITY, "buffer too small");
    for (size_t k = 0; k < series.size(); ++k) lead_out[k] = series[k].lead_tokens;
    return FB_OK;
  } catch (const std::exception& e) {
    return map_exception(e);
  }
}

int ref_generate_bursty(const fb_burst_profile* p, int64_t horizon_us, int64_t cap,
                        int64_t* arrival_us, int32_t* prompt_len,
                        int32_t* output_len, int64_t* ttft_us, int64_t* tpot_us,
                        int64_t* n_out) {
  try {
    BurstProfile bp;
    bp.base_rate = p->base_rate;
    bp.burst_rate = p->burst_rate;
    bp.burst_duration = p->burst_duration_us;
    bp.idle_duration = p->idle_duration_us;
    bp.prompt_len = {p->prompt_mean, p->prompt_p90};
    bp.output_len = {p->output_mean, p->output_p90};
    bp.ttft_slo = p->ttft_us;
    bp.tpot_slo = p->tpot_us;
    bp.seed = p->seed;
    const Trace tr = generate_bursty(bp, horizon_us);
    const int64_t n = static_cast<int64_t>(tr.requests.size());
    *n_out = n;
    if (n > cap) return fail(FB_ERR_CAPACITY, "capacity");
    for (int64_t i = 0; i < n; ++i) {
      arrival_us[i] = tr.requests[i].arrival;
      prompt_len[i] = tr.requests[i].prompt_len;
      output_len[i] = tr.requests[i].output_len;
      ttft_us[i] = tr.requests[i].ttft_slo;
      tpot_us[i] = tr.requests[i].tpot_slo;
    }
    return FB_OK;
  } catch (const std::exception& e) {
    return map_exception(e);
  }
}

int ref_scale_trace(int64_t* arrival_us, int64_t n, double factor) {
  try {
    Trace tr;
    tr.requests.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) tr.requests[i].arrival = arrival_us[i];
    const Trace out = scale_trace(tr, factor);
    for (int64_t i = 0; i < n; ++i) arrival_us[i] = out.requests[i].arrival;
    return FB_OK;
  } catch (const std::exception& e) {
    return map_exception(e);
  }
}

double ref_keyed_uniform(uint64_t seed, uint64_t ordinal) {
  return keyed_uniform(seed, ordinal);
}

int ref_init_time_budget(const fb_task_view* tasks, int64_t n, int64_t* out) {
  try {
    *out = init_time_budget(to_views(tasks, n));
    return FB_OK;
  } catch (const std::exception& e) {
    return map_exception(e);
  }
}

int ref_form_batch(const fb_task_view* tasks, int64_t n,
                   const fb_scheduler_config* cfg, fb_plan_entry_id* entries,
                   fb_batch_plan* plan) {
  try {
    const BatchPlan p = form_batch(to_views(tasks, n), to_sched(*cfg));
    plan->predicted_ms = p.predicted_ms;
    plan->time_budget_used_ms = p.time_budget_used_ms;
    plan->token_budget_used = p.token_budget_used;
    plan->init_time_budget_ms = p.init_time_budget_ms;
    plan->entry_off = 0;
    plan->n_entries = static_cast<int64_t>(p.entries.size());
    for (size_t k = 0; k < p.entries.size(); ++k) {
      entries[k].request_id = p.entries[k].request_id;
      entries[k].new_tokens = p.entries[k].new_tokens;
      entries[k].reserved = 0;
    }
    return FB_OK;
  } catch (const std::exception& e) {
    return map_exception(e);
  }
}

int ref_pab(const fb_task_view* tasks, int64_t n, const fb_cost_model* model,
            int64_t ttft_us, int64_t tpot_us, int64_t* out) {
  try {
    *out = pab(to_views(tasks, n), to_model(*model), SloTargets{ttft_us, tpot_us});
    return FB_OK;
  } catch (const std::exception& e) {
    return map_exception(e);
  }
}

// Mirror-driven run with plan capture (digest + optional logs); check != 0
// additionally verifies the mirror against the real run_node.
int ref_run_instances(const fb_trace* rows, const fb_instance* inst, int64_t n_inst,
                      const fb_log_opts* lo, fb_instance_result* results,
                      fb_record* records, fb_log_counts* counts,
                      fb_step_log* steps, fb_plan_entry* entries,
                      fb_reject_log* rejects, int nthreads, int check) {
  std::vector<int64_t> rec_off(static_cast<size_t>(n_inst) + 1, 0);
  for (int64_t i = 0; i < n_inst; ++i) rec_off[i + 1] = rec_off[i] + inst[i].n_req;
  std::atomic<int64_t> next{0};
  std::atomic<int> status{FB_OK};
  auto worker = [&]() {
    for (;;) {
      const int64_t i = next.fetch_add(1);
      if (i >= n_inst) return;
      try {
        const bool lg = lo != nullptr;
        const int st = run_mirror(
            rows, inst[i], lo, &results[i], records ? records + rec_off[i] : nullptr,
            counts ? &counts[i] : nullptr,
            lg && steps ? steps + i * lo->step_cap : nullptr,
            lg && entries ? entries + i * lo->entry_cap : nullptr,
            lg && rejects ? rejects + i * lo->reject_cap : nullptr, check);
        if (st) status = st;
      } catch (const std::exception& e) {
        status = map_exception(e);
      }
    }
  };
  if (nthreads <= 1) {
    worker();
  } else {
    std::vector<std::thread> th;
    for (int k = 0; k < nthreads; ++k) th.emplace_back(worker);
    for (auto& x : th) x.join();
  }
  return status.load();
}

// The reference's own pipeline for timing: run_node (engine.cpp:266-288) +
// request_reports (metrics.cpp:60-116) per instance on a std::thread pool.
// Fills results[].steps / n_arrived / incomplete and records (may be NULL).
int ref_run_node_batch(const fb_trace* rows, const fb_instance* inst,
                       int64_t n_inst, fb_instance_result* results,
                       fb_record* records, int nthreads) {
  std::vector<int64_t> rec_off(static_cast<size_t>(n_inst) + 1, 0);
  for (int64_t i = 0; i < n_inst; ++i) rec_off[i + 1] = rec_off[i] + inst[i].n_req;
  std::atomic<int64_t> next{0};
  std::atomic<int> status{FB_OK};
  auto worker = [&]() {
    for (;;) {
      const int64_t i = next.fetch_add(1);
      if (i >= n_inst) return;
      try {
        const Trace tr = instance_trace(rows, inst[i]);
        const EventLog log = run_node(tr, to_engine(inst[i].cfg), inst[i].horizon_us);
        fb_instance_result& r = results[i];
        std::memset(&r, 0, sizeof(r));
        for (const auto& e : log.events) {
          if (e.kind == EventKind::kBatchStart) r.steps++;
          if (e.kind == EventKind::kArrival) r.n_arrived++;
          if (e.kind == EventKind::kAdmissionReject) r.n_rejected++;
        }
        r.incomplete = log.incomplete ? 1 : 0;
        if (records) {
          fill_records({log}, tr, records + rec_off[i]);
        } else {
          (void)request_reports({log});
        }
      } catch (const std::exception& e) {
        status = map_exception(e);
      }
    }
  };
  if (nthreads <= 1) {
    worker();
  } else {
    std::vector<std::thread> th;
    for (int k = 0; k < nthreads; ++k) th.emplace_back(worker);
    for (auto& x : th) x.join();
  }
  return status.load();
}

// The reference's own run_cluster (cluster.cpp:134-251), unmirrored, for
// timing: n_rep independent copies of one cluster case (the C5 replica
// baseline) on a std::thread pool, one copy per task.  Fills each copy's
// node steps / arrivals / rejects (counted from the node logs) and
// incomplete flag; records of copy 0 when `records` is non-NULL.
int ref_run_cluster_stock(const fb_trace* rows, const fb_engine_config* cfgs, int32_t n_nodes,
                          const fb_lb_config* lbc, int64_t horizon, int32_t n_rep,
                          fb_instance_result* node_results, fb_record* records, int nthreads) {
  fb_instance whole{};
  whole.trace_off = 0;
  whole.n_req = rows->n_rows;
  const Trace tr = instance_trace(rows, whole);
  LbConfig lb;
  lb.policy = lbc->policy == FB_LB_PAB ? LbPolicy::kPabLb : LbPolicy::kCountLb;
  lb.report_interval_steps = lbc->report_interval_steps;
  lb.report_latency = lbc->report_latency_us;
  lb.w_waiting = lbc->w_waiting;
  lb.w_running = lbc->w_running;
  lb.retry_reroute = lbc->retry_reroute != 0;
  std::vector<EngineConfig> ecfg;
  for (int i = 0; i < n_nodes; ++i) ecfg.push_back(to_engine(cfgs[i]));
  std::atomic<int> next{0};
  std::atomic<int> status{FB_OK};
  auto worker = [&]() {
    for (;;) {
      const int k = next.fetch_add(1);
      if (k >= n_rep) return;
      try {
        const ClusterResult res = run_cluster(tr, ecfg, lb, horizon);
        for (int i = 0; i < n_nodes; ++i) {
          fb_instance_result& r = node_results[static_cast<int64_t>(k) * n_nodes + i];
          std::memset(&r, 0, sizeof(r));
          for (const auto& e : res.node_logs[static_cast<size_t>(i)].events) {
            if (e.kind == EventKind::kBatchStart) r.steps++;
            if (e.kind == EventKind::kArrival) r.n_arrived++;
            if (e.kind == EventKind::kAdmissionReject) r.n_rejected++;
          }
          r.incomplete = res.incomplete ? 1 : 0;
        }
        if (records && k == 0) fill_records(res.node_logs, tr, records);
      } catch (const std::exception& e) {
        status = map_exception(e);
      }
    }
  };
  if (nthreads <= 1) {
    worker();
  } else {
    std::vector<std::thread> th;
    for (int k = 0; k < nthreads; ++k) th.emplace_back(worker);
    for (auto& x : th) x.join();
  }
  return status.load();
}

}  // extern "C"
