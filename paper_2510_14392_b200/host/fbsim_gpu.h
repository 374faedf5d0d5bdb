// fbsim_gpu.h -- the C++ host API of the B200 scheduling path.
//
// Mirrors the reference simulator's public interfaces (namespace fbsim:
// workload.h, sched.h, costmodel.h, slo.h, engine.h, metrics.h, cluster.h,
// errors.h) -- same type and field names, same argument meaning, same
// exception taxonomy -- so a caller of fbsim::form_batch / pab / run_node /
// run_cluster / request_reports can switch to this namespace.  Everything
// runs on the GPU through the C ABI of include/fbgpu.h (libfbgpu.so); there
// is no CPU fallback: without a CUDA device the device entry points throw
// CudaError.
//
// Differences from fbsim, by design:
//   * run_nodes() is the batched form of run_node (thousands of nodes in one
//     device arena) -- the sweep drivers' hot loop (commands.cpp:100-116);
//   * ClusterResult also carries per-request reports and per-node digests;
//   * RequestReport built from a device record (cluster runs) carries the
//     first-token time and the max-TPOT figures instead of every emission.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace fbsim_gpu {

using TimeUs = std::int64_t;  // time.h:23-34
TimeUs ms_to_us(double ms);   // llround(ms * 1000), time.h:30-32
double us_to_ms(TimeUs us);

// ---------------------------------------------------------------- errors.h
class ParseError : public std::runtime_error {
 public:
  explicit ParseError(const std::string& w) : std::runtime_error(w) {}
};
class ValidationError : public std::runtime_error {
 public:
  explicit ValidationError(const std::string& w) : std::runtime_error(w) {}
};
class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};
class UsageError : public std::logic_error {
 public:
  explicit UsageError(const std::string& w) : std::logic_error(w) {}
};
// Device missing, CUDA runtime failure, capacity or exchange timeout.
class CudaError : public std::runtime_error {
 public:
  explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};

// -------------------------------------------------------------- workload.h
struct Request {
  std::int64_t id = 0;
  TimeUs arrival = 0;
  std::int32_t prompt_len = 0;
  std::int32_t output_len = 0;
  TimeUs ttft_slo = 0;
  TimeUs tpot_slo = 0;
};
struct Trace {
  std::string name;
  std::vector<Request> requests;  // sorted by arrival, ids unique
};
struct LengthDist {
  double mean = 1.0;
  double p90 = 1.0;
};
struct BurstProfile {
  double base_rate = 0.0;
  double burst_rate = 0.0;
  TimeUs burst_duration = 0;
  TimeUs idle_duration = 0;
  LengthDist prompt_len;
  LengthDist output_len;
  TimeUs ttft_slo = 0;
  TimeUs tpot_slo = 0;
  std::uint64_t seed = 0;
};
Trace generate_bursty(const BurstProfile& profile, TimeUs horizon);  // workload.cpp:244-298
Trace scale_trace(const Trace& trace, double factor);                // workload.cpp:211-221
double offered_rps(const Trace& trace);                              // workload.cpp:315-321

// ------------------------------------------- costmodel.h / slo.h / sched.h
struct CostModel {
  double a_ms = 0.0;
  double b_ms = 0.0;
  double c_ms = 0.0;
};
struct NoiseSpec {
  double amplitude = 0.0;
  std::uint64_t seed = 0;
};
struct SloTargets {
  TimeUs ttft_slo = 0;
  TimeUs tpot_slo = 0;
};
enum class Phase { kPrefill, kDecode };
struct TaskView {
  std::int64_t request_id = 0;
  Phase phase = Phase::kDecode;
  TimeUs slack = 0;
  std::int32_t new_tokens_available = 0;
  std::int64_t context = 0;
  std::int64_t arrival_seq = 0;
  TimeUs tpot_slo = 0;
};
struct BatchPlanEntry {
  std::int64_t request_id = 0;
  std::int32_t new_tokens = 0;
};
struct BatchPlan {
  std::vector<BatchPlanEntry> entries;
  double predicted_ms = 0.0;
  double time_budget_used_ms = 0.0;
  std::int64_t token_budget_used = 0;
  double init_time_budget_ms = 0.0;
};
enum class Policy { kPrefillFirst, kSarathi, kFairBatch, kFairBatchPab };
const char* policy_name(Policy p);
bool parse_policy(const std::string& name, Policy& out);
struct SchedulerConfig {
  Policy policy = Policy::kFairBatch;
  std::int64_t token_budget = 2048;
  std::int32_t max_chunk = 2048;
  CostModel model;
};

// Pure scheduler (sched.h:81-109), one task set per call; device selects the
// GPU.  Batched forms: fb_form_batch / fb_init_time_budget / fb_pab.
TimeUs init_time_budget(const std::vector<TaskView>& tasks, int device = 0);
BatchPlan form_batch(const std::vector<TaskView>& tasks, const SchedulerConfig& cfg,
                     int device = 0);
std::int64_t pab(const std::vector<TaskView>& tasks, const CostModel& model,
                 const SloTargets& slo, int device = 0);

// ---------------------------------------------------------------- engine.h
enum class EventKind { kArrival, kAdmissionReject, kBatchStart, kTokenEmit, kRequestDone, kBatchEnd };
const char* event_kind_name(EventKind k);
struct Event {
  TimeUs t = 0;
  EventKind kind = EventKind::kArrival;
  std::int64_t req_id = -1;
  TimeUs arrival = 0;
  std::int32_t prompt_len = 0;
  std::int32_t output_len = 0;
  TimeUs ttft_slo = 0;
  TimeUs tpot_slo = 0;
  std::int64_t pab_tokens = 0;
  std::int64_t step = -1;
  std::int64_t new_tokens = 0;
  std::int64_t context_tokens = 0;
  double predicted_ms = 0.0;
  double actual_ms = 0.0;
  std::int32_t token_idx = -1;
};
struct EventLog {
  int node_id = 0;
  bool incomplete = false;
  std::vector<Event> events;
};
struct EngineConfig {
  SchedulerConfig scheduler;
  CostModel truth_model;
  NoiseSpec noise;
  SloTargets global_slo;
  std::int32_t max_active = 0;
};
// The reference's JSONL writer format (engine.cpp:395-451).
void save_event_log(const EventLog& log, const std::string& path);
std::string event_log_jsonl(const EventLog& log);

// run_node (engine.cpp:266-288): the node's whole EventLog, rebuilt from
// the device plan log (every step, entry and reject) -- byte-identical to
// the reference's when written with save_event_log.
EventLog run_node(const Trace& trace, const EngineConfig& cfg, TimeUs horizon, int device = 0);
// run_node over many (trace, config) pairs in one device arena.
std::vector<EventLog> run_nodes(const std::vector<const Trace*>& traces,
                                const std::vector<EngineConfig>& cfgs, TimeUs horizon,
                                int device = 0);

// The step machine, batched: many nodes (one per trace) resident on the
// device, advanced together by step(max_events) -- max_events iterations of
// each node's run_node event loop (engine.cpp:271-283: complete the step in
// flight, enqueue the arrivals at t, begin_step) -- until every node is
// quiescent.  reports() / summaries() read the current state at any point.
struct NodeSummary;
struct RequestReport;
class NodeBatch {
 public:
  NodeBatch(const std::vector<const Trace*>& traces, const std::vector<EngineConfig>& cfgs,
            TimeUs horizon, int device = 0);
  ~NodeBatch();
  NodeBatch(const NodeBatch&) = delete;
  NodeBatch& operator=(const NodeBatch&) = delete;
  // Returns the number of nodes still running (0: all quiescent).
  std::int64_t step(std::int64_t max_events = 1);
  void run();  // to quiescence
  std::vector<NodeSummary> summaries() const;
  // Per node, one RequestReport per request of its trace (in trace order).
  std::vector<std::vector<RequestReport>> reports() const;

 private:
  struct Impl;
  Impl* impl_;
};

// --------------------------------------------------------------- metrics.h
struct NodeSummary {
  std::uint64_t steps = 0, plan_digest = 0;  // steps_completed; rolling plan digest
  std::int64_t n_arrived = 0, n_rejected = 0;
  bool incomplete = false;
};
struct RequestReport {
  std::int64_t req_id = -1;
  TimeUs arrival = 0;
  TimeUs ttft_slo = 0;
  TimeUs tpot_slo = 0;
  std::int32_t output_len = 0;
  std::int32_t tokens_emitted = 0;
  bool rejected = false;
  bool finished = false;
  std::vector<TimeUs> emits;  // arrival-relative emission times (empty for device records)
  TimeUs first_emit_rel = -1;  // emits[0] when emits is empty
  double max_tpot_cached = 0.0, max_tpot_alt_cached = 0.0;
  bool has_ttft() const { return tokens_emitted >= 1; }
  double ttft_ms() const;
  double max_tpot_ms() const;      // metrics.cpp:42-49
  double max_tpot_alt_ms() const;  // metrics.cpp:53-60
  bool met_ttft = false;
  bool met_tpot = false;
  bool good() const { return !rejected && finished && met_ttft && met_tpot; }
};
// request_reports (metrics.cpp:60-116) over one or more event logs.
std::vector<RequestReport> request_reports(const std::vector<EventLog>& logs);

// --------------------------------------------------------------- cluster.h
enum class LbPolicy { kCountLb, kPabLb };
struct LbConfig {
  LbPolicy policy = LbPolicy::kPabLb;
  int report_interval_steps = 1;
  TimeUs report_latency = 0;
  double w_waiting = 1.0;
  double w_running = 1.0;
  bool retry_reroute = false;
};
const char* lb_policy_name(LbPolicy p);
struct RoutingLogEntry {
  TimeUs t = 0;
  std::int64_t req_id = -1;
  int node = 0;
  std::vector<double> view_snapshot;  // per-node score after the decision
};
// The reference's routing-log JSONL (cluster.cpp:114-131).
void save_routing_log(const std::vector<RoutingLogEntry>& log, LbPolicy policy,
                      const std::string& path);

struct ClusterResult {
  std::vector<EventLog> node_logs;
  std::vector<RoutingLogEntry> routing;  // one entry per routing decision
  std::vector<RequestReport> reports;  // every routed request, by id
  std::vector<NodeSummary> nodes;
  bool incomplete = false;
  double device_ms = 0.0;
};
// run_cluster (cluster.cpp:134-251) on one GPU.
ClusterResult run_cluster(const Trace& trace, const std::vector<EngineConfig>& node_cfgs,
                          const LbConfig& lb, TimeUs horizon, int device = 0);

// ------------------------------------------------- metrics.h / scenario.h
struct PercentileRow {
  double p50 = 0.0, p95 = 0.0, p99 = 0.0;
  std::size_t count = 0;
};
PercentileRow percentiles(std::vector<double> values);  // nearest rank, metrics.cpp:118-135
struct ScenarioReport {                                  // metrics.h:74-88
  std::string name;
  std::size_t total_requests = 0, rejected = 0, finished = 0, good = 0;
  double slo_violation_rate = 0.0, offered_rps = 0.0, effective_rps = 0.0;
  PercentileRow ttft_ms, max_tpot_ms, max_tpot_alt_ms;
};
// scenario_report (metrics.cpp:171-205) over the arrived requests' reports.
ScenarioReport scenario_report(const std::vector<RequestReport>& reports, double offered_rps,
                               const std::string& name, bool alt_tpot = false);

struct Scenario {  // scenario.h:31-61
  std::string name = "scenario";
  std::string trace_file, trace_format = "jsonl";
  bool bursty = false;
  BurstProfile burst;
  TimeUs burst_horizon = 0;
  std::int64_t max_requests = 0;
  double scale = 1.0;
  SloTargets slo;
  SchedulerConfig scheduler;
  CostModel truth;
  double noise_amplitude = 0.0;
  int nodes = 1;
  LbConfig lb;
  TimeUs horizon = 0;
  std::uint64_t seed = 0;
  std::string out_dir = "out";
  std::int32_t max_active = 0;
  TimeUs lead_bucket = 1000000;
  bool alt_tpot = false;
};
// load_scenario / scenario_from_json (scenario.cpp:77-222, 280-289): the
// JSON schema with unknown-key rejection; ConfigError on any violation,
// ValidationError for an invalid scheduler configuration.
Scenario load_scenario(const std::string& path);
Scenario scenario_from_json(const std::string& text);
Trace materialize_trace(const Scenario& sc);      // scenario.cpp:298-308
EngineConfig engine_config(const Scenario& sc);   // scenario.cpp:310-319
// run_scenario (commands.cpp:59-85) without the file writers.
ScenarioReport run_scenario(const Scenario& sc, int device = 0);

}  // namespace fbsim_gpu
