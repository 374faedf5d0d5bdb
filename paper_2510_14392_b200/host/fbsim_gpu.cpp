// fbsim_gpu.cpp -- the C++ host API (fbsim_gpu.h) over the C ABI of
// include/fbgpu.h.  Host work here is marshalling only: the scheduling, the
// step machine, the records and the cluster routing all run in libfbgpu.so
// on the GPU.  The event logs are rebuilt from the device plan logs with the
// rule of paper_2510_14392_b200/events.py (byte-identical to the reference's
// save_event_log, tests/test_gpu_parity.py).
#include "fbsim_gpu.h"

#include <algorithm>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <map>
#include <tuple>

#include "../../include/fbgpu.h"

namespace fbsim_gpu {

TimeUs ms_to_us(double ms) { return static_cast<TimeUs>(std::llround(ms * 1000.0)); }
double us_to_ms(TimeUs us) { return static_cast<double>(us) / 1000.0; }

namespace {

// Status codes -> the reference's exception taxonomy (errors.h:24-53).
void check(int st) {
  if (st == FB_OK) return;
  const std::string msg = fb_last_error() ? fb_last_error() : "";
  switch (st) {
    case FB_ERR_VALIDATION: throw ValidationError(msg);
    case FB_ERR_USAGE: throw UsageError(msg);
    case FB_ERR_CONFIG: throw ConfigError(msg);
    case FB_ERR_PARSE: throw ParseError(msg);
    default: throw CudaError(msg);
  }
}

fb_cost_model to_c(const CostModel& m) { return fb_cost_model{m.a_ms, m.b_ms, m.c_ms}; }

fb_scheduler_config to_c(const SchedulerConfig& c) {
  fb_scheduler_config o{};
  o.policy = static_cast<int32_t>(c.policy);
  o.max_chunk = c.max_chunk;
  o.token_budget = c.token_budget;
  o.model = to_c(c.model);
  return o;
}

fb_engine_config to_c(const EngineConfig& c) {
  fb_engine_config o{};
  o.scheduler = to_c(c.scheduler);
  o.truth_model = to_c(c.truth_model);
  o.noise_amplitude = c.noise.amplitude;
  o.noise_seed = c.noise.seed;
  o.global_ttft_us = c.global_slo.ttft_slo;
  o.global_tpot_us = c.global_slo.tpot_slo;
  o.max_active = c.max_active;
  return o;
}

std::vector<fb_task_view> to_c(const std::vector<TaskView>& tasks) {
  std::vector<fb_task_view> v(tasks.size());
  for (size_t i = 0; i < tasks.size(); ++i) {
    const TaskView& t = tasks[i];
    v[i].request_id = t.request_id;
    v[i].slack_us = t.slack;
    v[i].context = t.context;
    v[i].arrival_seq = t.arrival_seq;
    v[i].tpot_us = t.tpot_slo;
    v[i].new_tokens = t.new_tokens_available;
    v[i].phase = t.phase == Phase::kPrefill ? FB_PHASE_PREFILL : FB_PHASE_DECODE;
  }
  return v;
}

// Trace rows as the structure of arrays the device takes (row = position).
struct Rows {
  std::vector<int64_t> arrival, ttft, tpot;
  std::vector<int32_t> prompt, output;
  void add(const Trace& t) {
    for (const Request& r : t.requests) {
      arrival.push_back(r.arrival);
      prompt.push_back(r.prompt_len);
      output.push_back(r.output_len);
      ttft.push_back(r.ttft_slo);
      tpot.push_back(r.tpot_slo);
    }
  }
  fb_trace c() const {
    return fb_trace{arrival.data(), prompt.data(), output.data(), ttft.data(), tpot.data(),
                    static_cast<int64_t>(arrival.size())};
  }
};

struct Arena {
  fb_arena* a = nullptr;
  explicit Arena(int device) { check(fb_arena_create(device, nullptr, &a)); }
  ~Arena() { fb_arena_destroy(a); }
  Arena(const Arena&) = delete;
  Arena& operator=(const Arena&) = delete;
};

// One node's EventLog from its plan log.  At one instant the step
// completing comes first (token_emit / request_done in plan order,
// batch_end); then arrivals, rejects and the batch start ordered by (steps
// begun, rejects logged) -- an arrival tagged with its node's counts at
// enqueue falls after the events logged before it (a rerouted arrival can
// follow the node's own begin_step of that instant, cluster.cpp:222-237);
// untagged arrivals (-1) precede the instant's begin_step (run_node,
// engine.cpp:271-283).
struct Arrival {
  TimeUs t;
  int64_t row;
  int64_t rej_before, steps_before;
};

EventLog build_log(const Trace& tr, const std::vector<Arrival>& arrivals, bool incomplete,
                   const fb_log_counts& cnt, const fb_step_log* steps,
                   const fb_plan_entry* entries, const fb_reject_log* rejects) {
  if (cnt.truncated) throw CudaError("plan log truncated");
  constexpr int64_t kBig = int64_t(1) << 62;
  struct Item {
    TimeUs t;
    int cls;
    int64_t a, b, c, d;
    Event e;
  };
  std::vector<Item> items;
  for (size_t k = 0; k < arrivals.size(); ++k) {
    const Arrival& ar = arrivals[k];
    const Request& q = tr.requests[static_cast<size_t>(ar.row)];
    Event e;
    e.t = ar.t;
    e.kind = EventKind::kArrival;
    e.req_id = q.id;
    e.arrival = q.arrival;
    e.prompt_len = q.prompt_len;
    e.output_len = q.output_len;
    e.ttft_slo = q.ttft_slo;
    e.tpot_slo = q.tpot_slo;
    items.push_back({e.t, 1, ar.steps_before, ar.rej_before, 0, static_cast<int64_t>(k), e});
  }
  for (int32_t j = 0; j < cnt.rejects; ++j) {
    const fb_reject_log& rj = rejects[j];
    Event e;
    e.t = rj.t_us;
    e.kind = EventKind::kAdmissionReject;
    e.req_id = tr.requests[static_cast<size_t>(rj.req)].id;
    e.prompt_len = tr.requests[static_cast<size_t>(rj.req)].prompt_len;
    e.pab_tokens = rj.pab_tokens;
    items.push_back({e.t, 1, rj.step, j, 1, 0, e});
  }
  std::vector<int64_t> prefilled(std::max<size_t>(tr.requests.size(), 1), 0);
  std::vector<int32_t> nidx(prefilled.size(), 0);
  for (int32_t s = 0; s < cnt.steps; ++s) {
    const fb_step_log& st = steps[s];
    const TimeUs t0 = st.t_us, t1 = st.t_us + st.duration_us;
    Event b;
    b.t = t0;
    b.kind = EventKind::kBatchStart;
    b.step = s;
    b.new_tokens = st.total_new;
    b.context_tokens = st.total_ctx;
    b.predicted_ms = st.predicted_ms;
    items.push_back({t0, 1, s, kBig, 2, 0, b});
    int64_t sub = 0;
    for (int32_t k = 0; k < st.n_entries; ++k) {
      const fb_plan_entry& pe = entries[st.entry_off + k];
      const Request& q = tr.requests[static_cast<size_t>(pe.req)];
      bool emit = true;
      if (prefilled[pe.req] < q.prompt_len) {
        prefilled[pe.req] += pe.new_tokens;
        emit = prefilled[pe.req] >= q.prompt_len;  // the completing chunk yields token 0
      }
      if (!emit) continue;
      Event e;
      e.t = t1;
      e.kind = EventKind::kTokenEmit;
      e.req_id = q.id;
      e.token_idx = nidx[pe.req]++;
      items.push_back({t1, 0, s, sub++, 0, 0, e});
      if (nidx[pe.req] >= q.output_len) {
        Event d;
        d.t = t1;
        d.kind = EventKind::kRequestDone;
        d.req_id = q.id;
        items.push_back({t1, 0, s, sub++, 0, 0, d});
      }
    }
    Event end;
    end.t = t1;
    end.kind = EventKind::kBatchEnd;
    end.step = s;
    end.actual_ms = st.actual_ms;
    items.push_back({t1, 0, s, sub++, 0, 0, end});
  }
  std::stable_sort(items.begin(), items.end(), [](const Item& x, const Item& y) {
    return std::tie(x.t, x.cls, x.a, x.b, x.c, x.d) < std::tie(y.t, y.cls, y.a, y.b, y.c, y.d);
  });
  EventLog log;
  log.incomplete = incomplete;
  log.events.reserve(items.size());
  for (const Item& it : items) log.events.push_back(it.e);
  return log;
}

RequestReport report_from_record(const Request& q, const fb_record& r) {
  RequestReport o;
  o.req_id = q.id;
  o.arrival = q.arrival;
  o.ttft_slo = q.ttft_slo;
  o.tpot_slo = q.tpot_slo;
  o.output_len = q.output_len;
  o.tokens_emitted = r.tokens_emitted;
  o.rejected = (r.flags & FB_REC_REJECTED) != 0;
  o.finished = (r.flags & FB_REC_FINISHED) != 0;
  o.met_ttft = (r.flags & FB_REC_MET_TTFT) != 0;
  o.met_tpot = (r.flags & FB_REC_MET_TPOT) != 0;
  o.first_emit_rel = r.first_emit_us >= 0 ? r.first_emit_us - q.arrival : -1;
  o.max_tpot_cached = r.max_tpot_ms;
  o.max_tpot_alt_cached = r.max_tpot_alt_ms;
  return o;
}

}  // namespace

// ------------------------------------------------------------ policy names

const char* policy_name(Policy p) {
  switch (p) {
    case Policy::kPrefillFirst: return "prefill_first";
    case Policy::kSarathi: return "sarathi";
    case Policy::kFairBatch: return "fairbatch";
    case Policy::kFairBatchPab: return "fairbatch_pab";
  }
  return "?";
}

bool parse_policy(const std::string& name, Policy& out) {
  for (Policy p : {Policy::kPrefillFirst, Policy::kSarathi, Policy::kFairBatch,
                   Policy::kFairBatchPab}) {
    if (name == policy_name(p)) {
      out = p;
      return true;
    }
  }
  return false;
}

const char* event_kind_name(EventKind k) {
  switch (k) {
    case EventKind::kArrival: return "arrival";
    case EventKind::kAdmissionReject: return "admission_reject";
    case EventKind::kBatchStart: return "batch_start";
    case EventKind::kTokenEmit: return "token_emit";
    case EventKind::kRequestDone: return "request_done";
    case EventKind::kBatchEnd: return "batch_end";
  }
  return "?";
}

// ------------------------------------------------------------------ traces

Trace generate_bursty(const BurstProfile& p, TimeUs horizon) {
  fb_burst_profile c{};
  c.base_rate = p.base_rate;
  c.burst_rate = p.burst_rate;
  c.burst_duration_us = p.burst_duration;
  c.idle_duration_us = p.idle_duration;
  c.prompt_mean = p.prompt_len.mean;
  c.prompt_p90 = p.prompt_len.p90;
  c.output_mean = p.output_len.mean;
  c.output_p90 = p.output_len.p90;
  c.ttft_us = p.ttft_slo;
  c.tpot_us = p.tpot_slo;
  c.seed = p.seed;
  int64_t n = 0;
  int st = fb_generate_bursty(&c, horizon, 0, nullptr, nullptr, nullptr, nullptr, nullptr, &n);
  if (st != FB_OK && st != FB_ERR_CAPACITY) check(st);
  std::vector<int64_t> arr(n), tt(n), tp(n);
  std::vector<int32_t> pr(n), ou(n);
  check(fb_generate_bursty(&c, horizon, n, arr.data(), pr.data(), ou.data(), tt.data(), tp.data(),
                           &n));
  Trace t;
  t.name = "bursty";
  t.requests.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i)
    t.requests[i] = Request{i, arr[i], pr[i], ou[i], tt[i], tp[i]};
  return t;
}

Trace scale_trace(const Trace& trace, double factor) {
  std::vector<int64_t> arr;
  for (const Request& r : trace.requests) arr.push_back(r.arrival);
  check(fb_scale_trace(arr.data(), static_cast<int64_t>(arr.size()), factor));
  Trace t = trace;
  for (size_t i = 0; i < arr.size(); ++i) t.requests[i].arrival = arr[i];
  return t;
}

double offered_rps(const Trace& trace) {
  std::vector<int64_t> arr;
  for (const Request& r : trace.requests) arr.push_back(r.arrival);
  double rps = 0.0;
  check(fb_offered_rps(arr.data(), static_cast<int64_t>(arr.size()), &rps));
  return rps;
}

// ------------------------------------------------------------ pure scheduler

TimeUs init_time_budget(const std::vector<TaskView>& tasks, int device) {
  const std::vector<fb_task_view> v = to_c(tasks);
  const int64_t off[2] = {0, static_cast<int64_t>(v.size())};
  int64_t out = 0;
  check(fb_init_time_budget(device, v.data(), off, 1, &out));
  return out;
}

BatchPlan form_batch(const std::vector<TaskView>& tasks, const SchedulerConfig& cfg, int device) {
  const std::vector<fb_task_view> v = to_c(tasks);
  const int64_t off[2] = {0, static_cast<int64_t>(v.size())};
  const fb_scheduler_config c = to_c(cfg);
  std::vector<fb_plan_entry_id> e(std::max<size_t>(v.size(), 1));
  fb_batch_plan p{};
  check(fb_form_batch(device, v.data(), off, &c, 1, e.data(), &p));
  BatchPlan out;
  out.predicted_ms = p.predicted_ms;
  out.time_budget_used_ms = p.time_budget_used_ms;
  out.token_budget_used = p.token_budget_used;
  out.init_time_budget_ms = p.init_time_budget_ms;
  for (int64_t k = 0; k < p.n_entries; ++k)
    out.entries.push_back({e[p.entry_off + k].request_id, e[p.entry_off + k].new_tokens});
  return out;
}

std::int64_t pab(const std::vector<TaskView>& tasks, const CostModel& model,
                 const SloTargets& slo, int device) {
  const std::vector<fb_task_view> v = to_c(tasks);
  const int64_t off[2] = {0, static_cast<int64_t>(v.size())};
  const fb_cost_model m = to_c(model);
  int64_t out = 0;
  check(fb_pab(device, v.data(), off, &m, &slo.ttft_slo, &slo.tpot_slo, 1, &out));
  return out;
}

// ------------------------------------------------------------------- nodes

std::vector<EventLog> run_nodes(const std::vector<const Trace*>& traces,
                                const std::vector<EngineConfig>& cfgs, TimeUs horizon,
                                int device) {
  if (traces.size() != cfgs.size()) throw UsageError("run_nodes: one config per trace");
  const int64_t n = static_cast<int64_t>(traces.size());
  if (n == 0) return {};
  Rows rows;
  std::vector<fb_instance> inst(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    inst[i].cfg = to_c(cfgs[i]);
    inst[i].trace_off = static_cast<int64_t>(rows.arrival.size());
    inst[i].n_req = static_cast<int64_t>(traces[i]->requests.size());
    inst[i].horizon_us = horizon;
    rows.add(*traces[i]);
  }
  const fb_trace tr = rows.c();
  Arena a(device);
  // pass 1 sizes the plan logs exactly, pass 2 records them
  check(fb_arena_load(a.a, &tr, inst.data(), n, nullptr));
  check(fb_arena_run(a.a, 0, nullptr));
  std::vector<fb_instance_result> res(static_cast<size_t>(n));
  check(fb_arena_fetch_results(a.a, res.data()));
  fb_log_opts lo{1, 1, 1, 0};
  for (const fb_instance_result& r : res) {
    lo.step_cap = std::max<int32_t>(lo.step_cap, static_cast<int32_t>(r.steps));
    lo.entry_cap = std::max<int32_t>(lo.entry_cap, static_cast<int32_t>(r.sum_entries));
    lo.reject_cap = std::max<int32_t>(lo.reject_cap, static_cast<int32_t>(r.n_rejected));
  }
  check(fb_arena_load(a.a, &tr, inst.data(), n, &lo));
  check(fb_arena_run(a.a, 0, nullptr));
  check(fb_arena_fetch_results(a.a, res.data()));
  std::vector<fb_log_counts> cnt(static_cast<size_t>(n));
  check(fb_arena_fetch_log_counts(a.a, cnt.data()));
  std::vector<EventLog> logs;
  std::vector<fb_step_log> steps(static_cast<size_t>(lo.step_cap));
  std::vector<fb_plan_entry> entries(static_cast<size_t>(lo.entry_cap));
  std::vector<fb_reject_log> rejects(static_cast<size_t>(lo.reject_cap));
  for (int64_t i = 0; i < n; ++i) {
    check(res[i].status);
    check(fb_arena_fetch_log(a.a, i, steps.data(), entries.data(), rejects.data()));
    std::vector<Arrival> arrivals;
    for (int64_t r = 0; r < res[i].n_arrived; ++r)
      arrivals.push_back({traces[i]->requests[static_cast<size_t>(r)].arrival, r, -1, -1});
    logs.push_back(build_log(*traces[i], arrivals, res[i].incomplete != 0, cnt[i], steps.data(),
                             entries.data(), rejects.data()));
  }
  return logs;
}

EventLog run_node(const Trace& trace, const EngineConfig& cfg, TimeUs horizon, int device) {
  return run_nodes({&trace}, {cfg}, horizon, device)[0];
}

// -------------------------------------------------------------- NodeBatch

struct NodeBatch::Impl {
  Arena a;
  std::vector<const Trace*> traces;
  Rows rows;
  std::vector<fb_instance> inst;
  explicit Impl(int device) : a(device) {}
};

NodeBatch::NodeBatch(const std::vector<const Trace*>& traces,
                     const std::vector<EngineConfig>& cfgs, TimeUs horizon, int device)
    : impl_(nullptr) {
  if (traces.size() != cfgs.size()) throw UsageError("NodeBatch: one config per trace");
  Impl* m = new Impl(device);
  try {
    m->traces = traces;
    for (size_t i = 0; i < traces.size(); ++i) {
      fb_instance x{};
      x.cfg = to_c(cfgs[i]);
      x.trace_off = static_cast<int64_t>(m->rows.arrival.size());
      x.n_req = static_cast<int64_t>(traces[i]->requests.size());
      x.horizon_us = horizon;
      m->inst.push_back(x);
      m->rows.add(*traces[i]);
    }
    const fb_trace tr = m->rows.c();
    check(fb_arena_load(m->a.a, &tr, m->inst.data(), static_cast<int64_t>(m->inst.size()),
                        nullptr));
  } catch (...) {
    delete m;
    throw;
  }
  impl_ = m;
}

NodeBatch::~NodeBatch() { delete impl_; }

std::int64_t NodeBatch::step(std::int64_t max_events) {
  if (max_events < 1) throw UsageError("NodeBatch::step: max_events must be >= 1");
  int64_t active = 0;
  check(fb_arena_run(impl_->a.a, max_events, &active));
  return active;
}

void NodeBatch::run() { check(fb_arena_run(impl_->a.a, 0, nullptr)); }

std::vector<NodeSummary> NodeBatch::summaries() const {
  std::vector<fb_instance_result> res(impl_->inst.size());
  check(fb_arena_fetch_results(impl_->a.a, res.data()));
  std::vector<NodeSummary> out;
  for (const fb_instance_result& r : res) {
    check(r.status);
    out.push_back({r.steps, r.plan_digest, r.n_arrived, r.n_rejected, r.incomplete != 0});
  }
  return out;
}

std::vector<std::vector<RequestReport>> NodeBatch::reports() const {
  std::vector<fb_record> rec(static_cast<size_t>(std::max<int64_t>(fb_arena_record_rows(impl_->a.a), 1)));
  check(fb_arena_fetch_records(impl_->a.a, rec.data()));
  std::vector<std::vector<RequestReport>> out;
  for (size_t i = 0; i < impl_->traces.size(); ++i) {
    const Trace& t = *impl_->traces[i];
    std::vector<RequestReport> v;
    for (size_t q = 0; q < t.requests.size(); ++q)
      v.push_back(report_from_record(t.requests[q], rec[impl_->inst[i].trace_off + q]));
    out.push_back(std::move(v));
  }
  return out;
}

// ----------------------------------------------------------------- reports

double RequestReport::ttft_ms() const {
  if (!emits.empty()) return us_to_ms(emits[0]);
  return first_emit_rel >= 0 ? us_to_ms(first_emit_rel) : 0.0;
}

double RequestReport::max_tpot_ms() const {
  if (emits.empty()) return max_tpot_cached;
  double best = 0.0;  // metrics.cpp:42-49
  for (size_t j = 1; j < emits.size(); ++j)
    best = std::max(best, us_to_ms(emits[j] - emits[0]) / static_cast<double>(j));
  return best;
}

double RequestReport::max_tpot_alt_ms() const {
  if (emits.empty()) return max_tpot_alt_cached;
  double best = 0.0;  // metrics.cpp:53-60
  for (size_t j = 2; j < emits.size(); ++j)
    best = std::max(best, us_to_ms(emits[j] - emits[0]) / static_cast<double>(j - 1));
  return best;
}

std::vector<RequestReport> request_reports(const std::vector<EventLog>& logs) {
  std::map<int64_t, RequestReport> by_id;
  std::map<int64_t, bool> any_reject;
  for (const EventLog& log : logs) {
    for (const Event& e : log.events) {
      if (e.kind == EventKind::kArrival) {
        RequestReport& r = by_id[e.req_id];
        r.req_id = e.req_id;
        r.arrival = e.arrival;
        r.ttft_slo = e.ttft_slo;
        r.tpot_slo = e.tpot_slo;
        r.output_len = e.output_len;
      } else if (e.kind == EventKind::kAdmissionReject) {
        any_reject[e.req_id] = true;
      } else if (e.kind == EventKind::kTokenEmit) {
        RequestReport& r = by_id[e.req_id];
        r.emits.push_back(e.t - r.arrival);
      } else if (e.kind == EventKind::kRequestDone) {
        by_id[e.req_id].finished = true;
      }
    }
  }
  std::vector<RequestReport> out;
  for (auto& kv : by_id) {
    RequestReport& r = kv.second;
    r.tokens_emitted = static_cast<int32_t>(r.emits.size());
    // rejected only if never served anywhere (rerouting, metrics.cpp:96-98)
    r.rejected = any_reject.count(kv.first) > 0 && r.emits.empty();
    if (r.rejected) {
      r.met_ttft = r.met_tpot = false;
    } else {
      r.met_ttft = r.has_ttft() && r.emits[0] <= r.ttft_slo;
      bool ok = r.finished;
      for (size_t j = 1; j < r.emits.size() && ok; ++j)
        ok = r.emits[j] - r.emits[0] <= r.tpot_slo * static_cast<TimeUs>(j);
      r.met_tpot = ok;
    }
    if (r.has_ttft()) r.first_emit_rel = r.emits[0];
    out.push_back(r);
  }
  return out;
}

// ----------------------------------------------------------- JSONL writer

std::string event_log_jsonl(const EventLog& log) {
  std::string s;
  char buf[512];
  for (const Event& e : log.events) {
    switch (e.kind) {
      case EventKind::kArrival:
        std::snprintf(buf, sizeof(buf),
                      "{\"t_ms\":%.3f,\"kind\":\"arrival\",\"req_id\":%" PRId64
                      ",\"arrival_ms\":%.3f,\"prompt_tokens\":%d,\"output_tokens\":%d,"
                      "\"ttft_slo_ms\":%.3f,\"tpot_slo_ms\":%.3f}\n",
                      us_to_ms(e.t), e.req_id, us_to_ms(e.arrival), e.prompt_len, e.output_len,
                      us_to_ms(e.ttft_slo), us_to_ms(e.tpot_slo));
        break;
      case EventKind::kAdmissionReject:
        std::snprintf(buf, sizeof(buf),
                      "{\"t_ms\":%.3f,\"kind\":\"admission_reject\",\"req_id\":%" PRId64
                      ",\"prompt_tokens\":%d,\"pab_tokens\":%" PRId64 "}\n",
                      us_to_ms(e.t), e.req_id, e.prompt_len, e.pab_tokens);
        break;
      case EventKind::kBatchStart:
        std::snprintf(buf, sizeof(buf),
                      "{\"t_ms\":%.3f,\"kind\":\"batch_start\",\"step\":%" PRId64
                      ",\"new_tokens\":%" PRId64 ",\"context_tokens\":%" PRId64
                      ",\"predicted_ms\":%.6f}\n",
                      us_to_ms(e.t), e.step, e.new_tokens, e.context_tokens, e.predicted_ms);
        break;
      case EventKind::kTokenEmit:
        std::snprintf(buf, sizeof(buf),
                      "{\"t_ms\":%.3f,\"kind\":\"token_emit\",\"req_id\":%" PRId64
                      ",\"token_idx\":%d}\n",
                      us_to_ms(e.t), e.req_id, e.token_idx);
        break;
      case EventKind::kRequestDone:
        std::snprintf(buf, sizeof(buf),
                      "{\"t_ms\":%.3f,\"kind\":\"request_done\",\"req_id\":%" PRId64 "}\n",
                      us_to_ms(e.t), e.req_id);
        break;
      case EventKind::kBatchEnd:
        std::snprintf(buf, sizeof(buf),
                      "{\"t_ms\":%.3f,\"kind\":\"batch_end\",\"step\":%" PRId64
                      ",\"actual_ms\":%.6f}\n",
                      us_to_ms(e.t), e.step, e.actual_ms);
        break;
    }
    s += buf;
  }
  std::snprintf(buf, sizeof(buf), "{\"kind\":\"log_end\",\"node\":%d,\"incomplete\":%d}\n",
                log.node_id, log.incomplete ? 1 : 0);
  s += buf;
  return s;
}

void save_event_log(const EventLog& log, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw ParseError("cannot open for writing: " + path);
  out << event_log_jsonl(log);
}

// ----------------------------------------------------------------- cluster

ClusterResult run_cluster(const Trace& trace, const std::vector<EngineConfig>& node_cfgs,
                          const LbConfig& lb, TimeUs horizon, int device) {
  Rows rows;
  rows.add(trace);
  const fb_trace tr = rows.c();
  std::vector<fb_engine_config> cfgs;
  for (const EngineConfig& c : node_cfgs) cfgs.push_back(to_c(c));
  fb_lb_config l{};
  l.policy = lb.policy == LbPolicy::kPabLb ? FB_LB_PAB : FB_LB_COUNT;
  l.report_interval_steps = lb.report_interval_steps;
  l.report_latency_us = lb.report_latency;
  l.w_waiting = lb.w_waiting;
  l.w_running = lb.w_running;
  l.retry_reroute = lb.retry_reroute ? 1 : 0;
  const size_t nr = trace.requests.size(), nn = node_cfgs.size();
  std::vector<fb_instance_result> res(std::max<size_t>(nn, 1));
  std::vector<fb_record> rec(std::max<size_t>(nr, 1));
  std::vector<int32_t> route(std::max<size_t>(nr, 1));
  int32_t inc = 0;
  ClusterResult out;
  // pass 1 sizes the node plan logs, pass 2 records them with the routing log
  check(fb_run_cluster(device, &tr, cfgs.data(), static_cast<int32_t>(nn), &l, horizon,
                       res.data(), rec.data(), route.data(), &inc, &out.device_ms));
  fb_log_opts lo{1, 1, 1, 0};
  for (size_t i = 0; i < nn; ++i) {
    lo.step_cap = std::max<int32_t>(lo.step_cap, static_cast<int32_t>(res[i].steps));
    lo.entry_cap = std::max<int32_t>(lo.entry_cap, static_cast<int32_t>(res[i].sum_entries));
    lo.reject_cap = std::max<int32_t>(lo.reject_cap, static_cast<int32_t>(res[i].n_rejected));
  }
  std::vector<fb_log_counts> cnt(std::max<size_t>(nn, 1));
  std::vector<fb_step_log> steps(nn * lo.step_cap);
  std::vector<fb_plan_entry> entries(nn * lo.entry_cap);
  std::vector<fb_reject_log> rejects(nn * lo.reject_cap);
  const int64_t cap = static_cast<int64_t>(lb.retry_reroute ? 2 * nr + 1 : nr + 1);
  std::vector<fb_route_log> routes(static_cast<size_t>(cap));
  std::vector<double> snaps(static_cast<size_t>(cap) * nn);
  int64_t n_routes = 0;
  check(fb_run_cluster_logged(device, &tr, cfgs.data(), static_cast<int32_t>(nn), &l, horizon,
                              &lo, res.data(), rec.data(), route.data(), &inc, cnt.data(),
                              steps.data(), entries.data(), rejects.data(), routes.data(),
                              snaps.data(), cap, &n_routes));
  out.incomplete = inc != 0;
  for (size_t i = 0; i < nn; ++i)
    out.nodes.push_back({res[i].steps, res[i].plan_digest, res[i].n_arrived, res[i].n_rejected,
                         res[i].incomplete != 0});
  for (int64_t k = 0; k < n_routes; ++k) {
    const fb_route_log& e = routes[static_cast<size_t>(k)];
    RoutingLogEntry r;
    r.t = e.t_us;
    r.req_id = trace.requests[static_cast<size_t>(e.req)].id;
    r.node = e.node;
    r.view_snapshot.assign(snaps.begin() + k * nn, snaps.begin() + (k + 1) * nn);
    out.routing.push_back(std::move(r));
  }
  for (size_t q = 0; q < nr; ++q)
    if (route[q] >= 0) out.reports.push_back(report_from_record(trace.requests[q], rec[q]));
  // each node's EventLog: its arrivals are the requests routed to it, at
  // their routing times
  for (size_t i = 0; i < nn; ++i) {
    std::vector<Arrival> arrivals;
    for (int64_t k = 0; k < n_routes; ++k) {
      const fb_route_log& e = routes[static_cast<size_t>(k)];
      if (e.node == static_cast<int32_t>(i))
        arrivals.push_back({e.t_us, e.req, e.rej_before, e.steps_before});
    }
    EventLog log = build_log(trace, arrivals, out.incomplete, cnt[i], steps.data() + i * lo.step_cap,
                             entries.data() + i * lo.entry_cap, rejects.data() + i * lo.reject_cap);
    log.node_id = static_cast<int>(i);
    out.node_logs.push_back(std::move(log));
  }
  return out;
}

const char* lb_policy_name(LbPolicy p) { return p == LbPolicy::kPabLb ? "pab_lb" : "count_lb"; }

void save_routing_log(const std::vector<RoutingLogEntry>& log, LbPolicy policy,
                      const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw ParseError("cannot open for writing: " + path);
  char buf[256];
  for (const RoutingLogEntry& e : log) {
    std::snprintf(buf, sizeof(buf),
                  "{\"t_ms\":%.3f,\"req_id\":%" PRId64 ",\"node\":%d,\"policy\":\"%s\","
                  "\"view_snapshot\":[",
                  us_to_ms(e.t), e.req_id, e.node, lb_policy_name(policy));
    out << buf;
    for (size_t i = 0; i < e.view_snapshot.size(); ++i) {
      std::snprintf(buf, sizeof(buf), "%s%.3f", i ? "," : "", e.view_snapshot[i]);
      out << buf;
    }
    out << "]}\n";
  }
}

}  // namespace fbsim_gpu
