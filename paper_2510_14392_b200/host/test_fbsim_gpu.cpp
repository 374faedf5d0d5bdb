// test_fbsim_gpu.cpp -- tests of the C++ host API (fbsim_gpu.h), driven by
// tests/test_host_cpp.py.
//
//   test_fbsim_gpu nogpu                 host-only checks + every device entry
//                                        point must throw CudaError (no CPU
//                                        fallback)
//   test_fbsim_gpu kat                   the reference's known answers through
//                                        the C++ API on the GPU (test_sched.cpp,
//                                        test_engine.cpp, test_cluster.cpp)
//   test_fbsim_gpu eventlog IN OUT       run_node on the instance described in
//                                        IN, save_event_log to OUT (the caller
//                                        compares it with the reference's log)
//   test_fbsim_gpu clusterlogs IN DIR    run_cluster on the cluster in IN; its
//                                        node logs + routing log into DIR
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <string>

#include "fbsim_gpu.h"

using namespace fbsim_gpu;

static int g_fail = 0;
#define CHECK(c)                                                    \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #c); \
      ++g_fail;                                                     \
    }                                                               \
  } while (0)

template <typename E>
static bool throws(const std::function<void()>& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

// test_sched.cpp:17-53 helpers
static TaskView decode_task(int64_t id, double slack_ms, int64_t ctx, double tpot_ms = 50.0,
                            int64_t seq = -1) {
  TaskView v;
  v.request_id = id;
  v.phase = Phase::kDecode;
  v.slack = ms_to_us(slack_ms);
  v.new_tokens_available = 1;
  v.context = ctx;
  v.arrival_seq = seq < 0 ? id : seq;
  v.tpot_slo = ms_to_us(tpot_ms);
  return v;
}
static TaskView prefill_task(int64_t id, double slack_ms, int32_t tokens, int64_t ctx = 0,
                             double tpot_ms = 50.0) {
  TaskView v;
  v.request_id = id;
  v.phase = Phase::kPrefill;
  v.slack = ms_to_us(slack_ms);
  v.new_tokens_available = tokens;
  v.context = ctx;
  v.arrival_seq = id;
  v.tpot_slo = ms_to_us(tpot_ms);
  return v;
}
static const CostModel kModel{5.0, 0.01, 0.0001};
static SchedulerConfig fb_config(int64_t budget = 8192, Policy p = Policy::kFairBatch) {
  SchedulerConfig c;
  c.policy = p;
  c.token_budget = budget;
  c.max_chunk = static_cast<int32_t>(budget);
  c.model = kModel;
  return c;
}
static EngineConfig node_config(Policy p, int64_t budget = 8192, int32_t max_chunk = 8192) {
  EngineConfig c;  // test_engine.cpp / test_cluster.cpp node_config
  c.scheduler.policy = p;
  c.scheduler.token_budget = budget;
  c.scheduler.max_chunk = max_chunk;
  c.scheduler.model = kModel;
  c.truth_model = kModel;
  c.global_slo = {ms_to_us(500.0), ms_to_us(50.0)};
  return c;
}
static Request make_request(int64_t id, double arrival_ms, int32_t prompt, int32_t output) {
  return Request{id, ms_to_us(arrival_ms), prompt, output, ms_to_us(500.0), ms_to_us(50.0)};
}

static int run_nogpu() {
  // host-side pieces work without a device
  BurstProfile p;  // 931 requests
  p.base_rate = p.burst_rate = 4.0;
  p.burst_duration = ms_to_us(1500.0);
  p.idle_duration = ms_to_us(3500.0);
  p.prompt_len = {892.0, 1776.0};
  p.output_len = {377.0, 742.0};
  p.ttft_slo = ms_to_us(500.0);
  p.tpot_slo = ms_to_us(50.0);
  p.seed = 33;
  const Trace t = generate_bursty(p, ms_to_us(250000.0));
  CHECK(t.requests.size() == 931);
  CHECK(std::string(policy_name(Policy::kFairBatchPab)) == "fairbatch_pab");
  Policy q;
  CHECK(parse_policy("sarathi", q) && q == Policy::kSarathi && !parse_policy("fifo", q));
  EventLog log;
  Event a;
  a.t = a.arrival = 1000;
  a.req_id = 0;
  a.prompt_len = 10;
  a.output_len = 2;
  a.ttft_slo = 500000;
  a.tpot_slo = 50000;
  log.events.push_back(a);
  const std::string js = event_log_jsonl(log);
  CHECK(js ==
        "{\"t_ms\":1.000,\"kind\":\"arrival\",\"req_id\":0,\"arrival_ms\":1.000,"
        "\"prompt_tokens\":10,\"output_tokens\":2,\"ttft_slo_ms\":500.000,"
        "\"tpot_slo_ms\":50.000}\n{\"kind\":\"log_end\",\"node\":0,\"incomplete\":0}\n");
  // the device entry points fail loudly
  CHECK(throws<CudaError>([] { init_time_budget({decode_task(0, 30, 100)}); }));
  CHECK(throws<CudaError>([] { form_batch({decode_task(0, 30, 100)}, fb_config()); }));
  CHECK(throws<CudaError>([&] { run_node(t, node_config(Policy::kFairBatch), 1000); }));
  CHECK(throws<CudaError>([&] {
    run_cluster(t, {node_config(Policy::kFairBatch)}, LbConfig{}, 1000);
  }));
  return g_fail;
}

static int run_kat() {
  // test_sched.cpp:57-78
  CHECK(init_time_budget({decode_task(0, 30, 100), decode_task(1, 80, 100)}) == 50000);
  CHECK(init_time_budget({decode_task(0, 120, 100)}) == 120000);
  CHECK(init_time_budget({decode_task(0, -20, 100)}) == 50000);
  CHECK(init_time_budget({prefill_task(0, 300, 1000, 0, 80.0), prefill_task(1, 200, 500, 0, 60.0)}) ==
        60000);
  CHECK(throws<UsageError>([] { init_time_budget({}); }));
  // test_sched.cpp:80-89
  BatchPlan b = form_batch({decode_task(7, 40, 1000)}, fb_config());
  CHECK(b.entries.size() == 1 && b.entries[0].request_id == 7 && b.entries[0].new_tokens == 1);
  CHECK(std::fabs(b.predicted_ms - 5.11) < 1e-12 && b.init_time_budget_ms == 50.0);
  // test_sched.cpp:133-166: tie-break and the empty plan
  b = form_batch({decode_task(0, 20, 500), decode_task(1, 10, 500), prefill_task(2, 100, 50000)},
                 fb_config());
  CHECK(b.entries.size() >= 2 && b.entries[0].request_id == 1 && b.entries[1].request_id == 0);
  b = form_batch({decode_task(0, 10, 600000)}, fb_config());
  CHECK(b.entries.empty() && b.predicted_ms == 0.0);
  // test_sched.cpp:401-421
  const SloTargets slo{500000, 50000};
  CHECK(pab({}, kModel, slo) == 49009);
  CHECK(pab({decode_task(0, 100, 2000)}, kModel, slo) == 44883);
  CHECK(pab({decode_task(0, 100, 2000), prefill_task(1, 500, 10000)}, kModel, slo) == 34883);

  // test_engine.cpp:72-92: a 100-token prompt, 3 outputs, emits at 6000,
  // 11020, 16040 us
  Trace t1;
  t1.requests.push_back(make_request(0, 0.0, 100, 3));
  EventLog log = run_node(t1, node_config(Policy::kFairBatch), ms_to_us(60000.0));
  std::vector<TimeUs> emits;
  for (const Event& e : log.events)
    if (e.kind == EventKind::kTokenEmit) emits.push_back(e.t);
  CHECK(emits == (std::vector<TimeUs>{6000, 11020, 16040}));
  CHECK(!log.incomplete);
  std::vector<RequestReport> rep = request_reports({log});
  CHECK(rep.size() == 1 && rep[0].finished && rep[0].met_ttft && rep[0].tokens_emitted == 3);
  CHECK(std::fabs(rep[0].ttft_ms() - 6.0) < 1e-12);
  // test_engine.cpp:202-219: the empty node's PAB 49009 rejects a 60000 prompt
  Trace t2;
  t2.requests.push_back(make_request(0, 0.0, 60000, 4));
  t2.requests.push_back(make_request(1, 0.0, 100, 4));
  log = run_node(t2, node_config(Policy::kFairBatchPab), ms_to_us(60000.0));
  int rejects = 0;
  for (const Event& e : log.events)
    if (e.kind == EventKind::kAdmissionReject) {
      ++rejects;
      CHECK(e.req_id == 0 && e.pab_tokens == 49009);
    }
  CHECK(rejects == 1);
  rep = request_reports({log});
  CHECK(rep.size() == 2 && rep[0].rejected && !rep[1].rejected && rep[1].finished);
  // test_engine.cpp:221-243: 600-token prompt in 256-token chunks
  Trace t3;
  t3.requests.push_back(make_request(0, 0.0, 600, 3));
  log = run_node(t3, node_config(Policy::kSarathi, 512, 256), ms_to_us(60000.0));
  std::vector<int64_t> takes;
  for (const Event& e : log.events)
    if (e.kind == EventKind::kBatchStart) takes.push_back(e.new_tokens);
  CHECK(takes == (std::vector<int64_t>{256, 256, 88, 1, 1}));
  // batched run_node: each instance equals its single run
  const std::vector<EventLog> logs =
      run_nodes({&t1, &t3}, {node_config(Policy::kFairBatch), node_config(Policy::kSarathi, 512, 256)},
                ms_to_us(60000.0));
  CHECK(logs.size() == 2 && event_log_jsonl(logs[1]) == event_log_jsonl(log));
  CHECK(throws<ValidationError>([] {
    Trace bad;
    bad.requests.push_back(make_request(0, 0.0, 0, 3));  // prompt_len must be >= 1
    run_node(bad, node_config(Policy::kFairBatch), 1000);
  }));
  // the step machine: one event-loop iteration per step() reaches the same
  // state as a run to quiescence
  {
    NodeBatch nb({&t1, &t2, &t3},
                 {node_config(Policy::kFairBatch), node_config(Policy::kFairBatchPab),
                  node_config(Policy::kSarathi, 512, 256)},
                 ms_to_us(60000.0));
    int calls = 0;
    while (nb.step(1) > 0) ++calls;
    CHECK(calls >= 3);
    NodeBatch all({&t1, &t2, &t3},
                  {node_config(Policy::kFairBatch), node_config(Policy::kFairBatchPab),
                   node_config(Policy::kSarathi, 512, 256)},
                  ms_to_us(60000.0));
    all.run();
    const std::vector<NodeSummary> a = nb.summaries(), b2 = all.summaries();
    CHECK(a.size() == 3 && a[0].steps == 3 && a[1].n_rejected == 1);
    for (size_t i = 0; i < a.size(); ++i)
      CHECK(a[i].plan_digest == b2[i].plan_digest && a[i].steps == b2[i].steps);
    const auto rp = nb.reports();
    CHECK(rp[0][0].finished && std::fabs(rp[0][0].ttft_ms() - 6.0) < 1e-12);
    CHECK(rp[1][0].rejected && rp[1][1].finished);
    CHECK(throws<UsageError>([&] { nb.step(0); }));
  }
  CHECK(throws<ValidationError>([&] {  // Node ctor: validate_scheduler_config
    run_node(t1, node_config(Policy::kFairBatch, 100, 256), 1000);  // budget < max_chunk
  }));

  // test_cluster.cpp:76-113 through a 2-node cluster: pab_lb picks the
  // roomiest node that fits, ties to the lowest id
  Trace t4;
  t4.requests = {make_request(0, 0.0, 800, 4), make_request(1, 0.0, 100, 4),
                 make_request(2, 0.0, 50000, 4)};
  ClusterResult cr = run_cluster(t4, {node_config(Policy::kFairBatchPab), node_config(Policy::kFairBatchPab)},
                                 LbConfig{}, ms_to_us(60000.0));
  CHECK(cr.routing.size() == 3 && cr.routing[0].node == 0 && cr.routing[1].node == 1 &&
        cr.routing[2].node == 1);
  // test_cluster.cpp:225-250: with retry_reroute the request rejected behind
  // the giant prompts finishes on the other node
  Trace t5;
  t5.requests = {make_request(0, 0.0, 45000, 300), make_request(1, 1.0, 45000, 300),
                 make_request(2, 2.0, 9000, 20)};
  LbConfig lb;
  lb.retry_reroute = true;
  cr = run_cluster(t5, {node_config(Policy::kFairBatchPab), node_config(Policy::kFairBatchPab)}, lb,
                   ms_to_us(3600000.0));
  CHECK(cr.reports.size() == 3 && cr.reports[2].finished && !cr.reports[2].rejected);
  std::printf("kat: %d failures\n", g_fail);
  return g_fail;
}

// IN: "horizon policy token_budget max_chunk a b c ta tb tc noise_amp
// noise_seed ttft tpot max_active" then n, then n rows "arrival prompt
// output ttft tpot" (the arrival order is the row order).
static int run_eventlog(const char* in_path, const char* out_path) {
  std::ifstream in(in_path);
  int64_t horizon, budget, ttft, tpot;
  int policy, max_chunk, max_active;
  double a, b, c, ta, tb, tc, amp;
  unsigned long long seed;
  size_t n;
  in >> horizon >> policy >> budget >> max_chunk >> a >> b >> c >> ta >> tb >> tc >> amp >> seed >>
      ttft >> tpot >> max_active >> n;
  EngineConfig cfg;
  cfg.scheduler.policy = static_cast<Policy>(policy);
  cfg.scheduler.token_budget = budget;
  cfg.scheduler.max_chunk = max_chunk;
  cfg.scheduler.model = {a, b, c};
  cfg.truth_model = {ta, tb, tc};
  cfg.noise = {amp, seed};
  cfg.global_slo = {ttft, tpot};
  cfg.max_active = max_active;
  Trace t;
  for (size_t i = 0; i < n; ++i) {
    Request r;
    r.id = static_cast<int64_t>(i);
    in >> r.arrival >> r.prompt_len >> r.output_len >> r.ttft_slo >> r.tpot_slo;
    t.requests.push_back(r);
  }
  if (!in) {
    std::fprintf(stderr, "bad input\n");
    return 2;
  }
  save_event_log(run_node(t, cfg, horizon), out_path);
  return 0;
}

static EngineConfig read_cfg(std::istream& in) {
  int policy, max_chunk, max_active;
  int64_t budget, ttft, tpot;
  double a, b, c, ta, tb, tc, amp;
  unsigned long long seed;
  in >> policy >> budget >> max_chunk >> a >> b >> c >> ta >> tb >> tc >> amp >> seed >> ttft >>
      tpot >> max_active;
  EngineConfig cfg;
  cfg.scheduler.policy = static_cast<Policy>(policy);
  cfg.scheduler.token_budget = budget;
  cfg.scheduler.max_chunk = max_chunk;
  cfg.scheduler.model = {a, b, c};
  cfg.truth_model = {ta, tb, tc};
  cfg.noise = {amp, seed};
  cfg.global_slo = {ttft, tpot};
  cfg.max_active = max_active;
  return cfg;
}

// IN: "n_nodes horizon policy(0 count, 1 pab) interval latency_us w_w w_r
// reroute", one config line per node (as eventlog's, without the horizon),
// n, then n rows.  Writes OUT/node<i>.jsonl and OUT/routing.jsonl.
static int run_clusterlogs(const char* in_path, const std::string& out_dir) {
  std::ifstream in(in_path);
  int n_nodes, pol, interval, reroute;
  int64_t horizon, latency;
  double ww, wr;
  in >> n_nodes >> horizon >> pol >> interval >> latency >> ww >> wr >> reroute;
  std::vector<EngineConfig> cfgs;
  for (int i = 0; i < n_nodes; ++i) cfgs.push_back(read_cfg(in));
  size_t n;
  in >> n;
  Trace t;
  for (size_t i = 0; i < n; ++i) {
    Request r;
    r.id = static_cast<int64_t>(i);
    in >> r.arrival >> r.prompt_len >> r.output_len >> r.ttft_slo >> r.tpot_slo;
    t.requests.push_back(r);
  }
  if (!in) {
    std::fprintf(stderr, "bad input\n");
    return 2;
  }
  LbConfig lb;
  lb.policy = pol ? LbPolicy::kPabLb : LbPolicy::kCountLb;
  lb.report_interval_steps = interval;
  lb.report_latency = latency;
  lb.w_waiting = ww;
  lb.w_running = wr;
  lb.retry_reroute = reroute != 0;
  const ClusterResult res = run_cluster(t, cfgs, lb, horizon);
  for (size_t i = 0; i < res.node_logs.size(); ++i)
    save_event_log(res.node_logs[i], out_dir + "/node" + std::to_string(i) + ".jsonl");
  save_routing_log(res.routing, lb.policy, out_dir + "/routing.jsonl");
  return 0;
}

// IN: K, then K instance blocks in eventlog's format.  NodeBatch over all
// of them; prints per instance "steps digest n_rejected" (hex digest).
static int run_batch_digests(const char* in_path) {
  std::ifstream in(in_path);
  size_t k;
  in >> k;
  std::vector<Trace> traces(k);
  std::vector<EngineConfig> cfgs;
  TimeUs horizon = 0;
  for (size_t i = 0; i < k; ++i) {
    in >> horizon;
    cfgs.push_back(read_cfg(in));
    size_t n;
    in >> n;
    for (size_t j = 0; j < n; ++j) {
      Request r;
      r.id = static_cast<int64_t>(j);
      in >> r.arrival >> r.prompt_len >> r.output_len >> r.ttft_slo >> r.tpot_slo;
      traces[i].requests.push_back(r);
    }
  }
  if (!in) {
    std::fprintf(stderr, "bad input\n");
    return 2;
  }
  std::vector<const Trace*> tp;
  for (const Trace& t : traces) tp.push_back(&t);
  NodeBatch nb(tp, cfgs, horizon);
  nb.run();
  for (const NodeSummary& s : nb.summaries())
    std::printf("%llu %016llx %lld\n", static_cast<unsigned long long>(s.steps),
                static_cast<unsigned long long>(s.plan_digest), static_cast<long long>(s.n_rejected));
  return 0;
}

// IN as for `batch` (all instances share the horizon); run_nodes over all of
// them, each log written with save_event_log to DIR/out<i>.jsonl.
static int run_eventlogs(const char* in_path, const std::string& out_dir) {
  std::ifstream in(in_path);
  size_t k;
  in >> k;
  std::vector<Trace> traces(k);
  std::vector<EngineConfig> cfgs;
  TimeUs horizon = 0;
  for (size_t i = 0; i < k; ++i) {
    in >> horizon;
    cfgs.push_back(read_cfg(in));
    size_t n;
    in >> n;
    for (size_t j = 0; j < n; ++j) {
      Request r;
      r.id = static_cast<int64_t>(j);
      in >> r.arrival >> r.prompt_len >> r.output_len >> r.ttft_slo >> r.tpot_slo;
      traces[i].requests.push_back(r);
    }
  }
  if (!in) {
    std::fprintf(stderr, "bad input\n");
    return 2;
  }
  std::vector<const Trace*> tp;
  for (const Trace& t : traces) tp.push_back(&t);
  const std::vector<EventLog> logs = run_nodes(tp, cfgs, horizon);
  for (size_t i = 0; i < logs.size(); ++i)
    save_event_log(logs[i], out_dir + "/out" + std::to_string(i) + ".jsonl");
  return 0;
}

// run_scenario on a scenario file; one line of report fields.
static int run_scenario_file(const char* path) {
  try {
    const ScenarioReport r = run_scenario(load_scenario(path));
    std::printf("{\"name\":\"%s\",\"total\":%zu,\"rejected\":%zu,\"finished\":%zu,"
                "\"good\":%zu,\"offered\":%.17g,\"effective\":%.17g,\"violation\":%.17g,"
                "\"ttft\":[%.17g,%.17g,%.17g,%zu],\"tpot\":[%.17g,%.17g,%.17g,%zu]}\n",
                r.name.c_str(), r.total_requests, r.rejected, r.finished, r.good, r.offered_rps,
                r.effective_rps, r.slo_violation_rate, r.ttft_ms.p50, r.ttft_ms.p95, r.ttft_ms.p99,
                r.ttft_ms.count, r.max_tpot_ms.p50, r.max_tpot_ms.p95, r.max_tpot_ms.p99,
                r.max_tpot_ms.count);
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 1;  // commands.h:30-33
  } catch (const ValidationError& e) {
    std::fprintf(stderr, "validation error: %s\n", e.what());
    return 2;
  }
  return 0;
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "";
  try {
    if (mode == "nogpu") return run_nogpu() ? 1 : 0;
    if (mode == "kat") return run_kat() ? 1 : 0;
    if (mode == "eventlog" && argc == 4) return run_eventlog(argv[2], argv[3]);
    if (mode == "clusterlogs" && argc == 4) return run_clusterlogs(argv[2], argv[3]);
    if (mode == "scenario" && argc == 3) return run_scenario_file(argv[2]);
    if (mode == "batch" && argc == 3) return run_batch_digests(argv[2]);
    if (mode == "eventlogs" && argc == 4) return run_eventlogs(argv[2], argv[3]);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "uncaught: %s\n", e.what());
    return 3;
  }
  std::fprintf(stderr, "usage: test_fbsim_gpu nogpu | kat | eventlog IN OUT\n");
  return 2;
}
