// fbsim_gpu_scenario.cpp -- scenario loading and run_scenario for the C++
// host API (fbsim_gpu.h): the reference's JSON scenario schema
// (scenario.cpp:77-222, unknown keys rejected), trace materialisation
// (scenario.cpp:298-308, load_trace workload.cpp:185-209) and the scenario
// report (metrics.cpp:118-135, 171-205).  Host tooling over the device path:
// the runs go through run_nodes / run_cluster.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <fstream>
#include <map>
#include <memory>
#include <set>
#include <sstream>

#include "fbsim_gpu.h"

namespace fbsim_gpu {

namespace {

// ------------------------------------------------------ a small JSON reader

struct Json {
  enum Kind { kNull, kBool, kNum, kStr, kArr, kObj } kind = kNull;
  bool b = false;
  double num = 0.0;
  bool is_int = false;
  std::int64_t i = 0;
  std::string str;
  std::vector<Json> arr;
  std::map<std::string, Json> obj;
};

class Reader {
 public:
  explicit Reader(const std::string& s) : s_(s) {}
  Json parse() {
    Json v = value();
    ws();
    if (p_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  size_t p_ = 0;
  [[noreturn]] void fail(const std::string& what) {
    throw ConfigError("scenario JSON: " + what + " at offset " + std::to_string(p_));
  }
  void ws() {
    while (p_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[p_]))) ++p_;
  }
  bool eat(char c) {
    ws();
    if (p_ < s_.size() && s_[p_] == c) {
      ++p_;
      return true;
    }
    return false;
  }
  Json value() {
    ws();
    if (p_ >= s_.size()) fail("unexpected end");
    const char c = s_[p_];
    Json v;
    if (c == '{') {
      ++p_;
      v.kind = Json::kObj;
      if (eat('}')) return v;
      do {
        ws();
        const std::string k = string();
        if (!eat(':')) fail("expected ':'");
        v.obj[k] = value();
      } while (eat(','));
      if (!eat('}')) fail("expected '}'");
    } else if (c == '[') {
      ++p_;
      v.kind = Json::kArr;
      if (eat(']')) return v;
      do v.arr.push_back(value());
      while (eat(','));
      if (!eat(']')) fail("expected ']'");
    } else if (c == '"') {
      v.kind = Json::kStr;
      v.str = string();
    } else if (s_.compare(p_, 4, "true") == 0) {
      p_ += 4;
      v.kind = Json::kBool;
      v.b = true;
    } else if (s_.compare(p_, 5, "false") == 0) {
      p_ += 5;
      v.kind = Json::kBool;
    } else if (s_.compare(p_, 4, "null") == 0) {
      p_ += 4;
    } else {
      const size_t b = p_;
      while (p_ < s_.size() && std::strchr("+-0123456789.eE", s_[p_])) ++p_;
      if (b == p_) fail("unexpected character");
      const std::string tok = s_.substr(b, p_ - b);
      v.kind = Json::kNum;
      v.num = std::strtod(tok.c_str(), nullptr);
      v.is_int = tok.find_first_of(".eE") == std::string::npos;
      if (v.is_int) v.i = std::strtoll(tok.c_str(), nullptr, 10);
    }
    return v;
  }
  std::string string() {
    if (p_ >= s_.size() || s_[p_] != '"') fail("expected a string");
    ++p_;
    std::string out;
    while (p_ < s_.size() && s_[p_] != '"') {
      char c = s_[p_++];
      if (c == '\\' && p_ < s_.size()) {
        const char e = s_[p_++];
        c = e == 'n' ? '\n' : e == 't' ? '\t' : e;
      }
      out += c;
    }
    if (p_ >= s_.size()) fail("unterminated string");
    ++p_;
    return out;
  }
};

void keys(const Json& j, const std::string& section, std::set<std::string> allowed) {
  for (const auto& kv : j.obj)
    if (!allowed.count(kv.first))
      throw ConfigError("unknown key '" + (section.empty() ? "" : section + ".") + kv.first + "'");
}

const Json* find(const Json& j, const std::string& k) {
  auto it = j.obj.find(k);
  return it == j.obj.end() ? nullptr : &it->second;
}

double num(const Json& j, const std::string& section, const std::string& k, const double* def) {
  const Json* v = find(j, k);
  if (!v) {
    if (!def) throw ConfigError("missing required key '" + section + "." + k + "'");
    return *def;
  }
  if (v->kind != Json::kNum) throw ConfigError("'" + section + "." + k + "' must be a number");
  return v->num;
}
double num(const Json& j, const std::string& section, const std::string& k) {
  return num(j, section, k, nullptr);
}
double num(const Json& j, const std::string& section, const std::string& k, double def) {
  return num(j, section, k, &def);
}

const Json* section(const Json& j, const char* k) {
  const Json* v = find(j, k);
  if (!v) throw ConfigError(std::string("missing section '") + k + "'");
  return v;
}

CostModel model(const Json& j, const std::string& sec) {
  keys(j, sec, {"a_ms", "b_ms_per_token", "c_ms_per_context_token"});
  return CostModel{num(j, sec, "a_ms"), num(j, sec, "b_ms_per_token"),
                   num(j, sec, "c_ms_per_context_token")};
}

std::uint64_t splitmix64(std::uint64_t& s) {  // rng.h:25-30
  std::uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
std::uint64_t derive_seed(std::uint64_t base, std::uint64_t stream) {  // rng.h:33-37
  std::uint64_t s = base ^ (0x9e3779b97f4a7c15ULL * (stream + 1));
  splitmix64(s);
  return splitmix64(s);
}

std::string slurp(const std::string& path, const char* what) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ConfigError(std::string("cannot open ") + what + ": " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

// load_trace (workload.cpp:185-209): JSONL or CSV records, SLOs defaulted,
// stably re-sorted by arrival, ids assigned in sorted order.
Trace load_trace(const std::string& path, const std::string& fmt, TimeUs ttft, TimeUs tpot) {
  const std::string text = slurp(path, "trace file");
  struct Rec {
    TimeUs arrival, ttft, tpot;
    int32_t prompt, output;
  };
  std::vector<Rec> recs;
  std::istringstream lines(text);
  std::string line;
  std::vector<std::string> header;
  auto field_of = [](const Json& j, const char* k) -> const Json* {
    auto it = j.obj.find(k);
    return it == j.obj.end() ? nullptr : &it->second;
  };
  while (std::getline(lines, line)) {
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    std::map<std::string, double> r;
    if (fmt == "jsonl") {
      const Json j = Reader(line).parse();
      for (const char* k : {"arrival_ms", "prompt_tokens", "output_tokens", "ttft_slo_ms",
                            "tpot_slo_ms"})
        if (const Json* v = field_of(j, k)) r[k] = v->num;
    } else {
      std::vector<std::string> cells;
      std::stringstream cs(line);
      std::string cell;
      while (std::getline(cs, cell, ',')) cells.push_back(cell);
      if (header.empty()) {
        header = cells;
        continue;
      }
      for (size_t i = 0; i < cells.size() && i < header.size(); ++i)
        if (!cells[i].empty()) r[header[i]] = std::strtod(cells[i].c_str(), nullptr);
    }
    if (!r.count("arrival_ms") || !r.count("prompt_tokens") || !r.count("output_tokens"))
      throw ParseError("trace record missing a required field: " + line);
    recs.push_back({ms_to_us(r["arrival_ms"]),
                    r.count("ttft_slo_ms") ? ms_to_us(r["ttft_slo_ms"]) : ttft,
                    r.count("tpot_slo_ms") ? ms_to_us(r["tpot_slo_ms"]) : tpot,
                    static_cast<int32_t>(r["prompt_tokens"]),
                    static_cast<int32_t>(r["output_tokens"])});
  }
  std::stable_sort(recs.begin(), recs.end(),
                   [](const Rec& a, const Rec& b) { return a.arrival < b.arrival; });
  Trace t;
  t.name = path;
  for (size_t i = 0; i < recs.size(); ++i)
    t.requests.push_back({static_cast<int64_t>(i), recs[i].arrival, recs[i].prompt,
                          recs[i].output, recs[i].ttft, recs[i].tpot});
  return t;
}

}  // namespace

// ---------------------------------------------------------------- scenario

Scenario scenario_from_json(const std::string& text) {
  const Json j = Reader(text).parse();
  if (j.kind != Json::kObj) throw ConfigError("scenario JSON must be an object");
  keys(j, "", {"name", "trace", "slo", "scheduler", "cost_model", "cluster", "run"});
  Scenario sc;
  if (const Json* n = find(j, "name")) sc.name = n->str;
  const Json& jt = *section(j, "trace");
  keys(jt, "trace", {"file", "format", "bursty", "max_requests", "scale"});
  if (const Json* f = find(jt, "file")) {
    sc.trace_file = f->str;
    if (const Json* fm = find(jt, "format")) sc.trace_format = fm->str;
    if (sc.trace_format != "jsonl" && sc.trace_format != "csv")
      throw ConfigError("trace.format must be 'jsonl' or 'csv', got '" + sc.trace_format + "'");
  }
  if (const Json* jb = find(jt, "bursty")) {
    const std::string s = "trace.bursty";
    keys(*jb, s, {"base_rate", "burst_rate", "burst_duration_ms", "idle_duration_ms",
                  "prompt_mean", "prompt_p90", "output_mean", "output_p90", "seed",
                  "horizon_ms"});
    sc.bursty = true;
    sc.burst.base_rate = num(*jb, s, "base_rate");
    sc.burst.burst_rate = num(*jb, s, "burst_rate");
    sc.burst.burst_duration = ms_to_us(num(*jb, s, "burst_duration_ms"));
    sc.burst.idle_duration = ms_to_us(num(*jb, s, "idle_duration_ms"));
    sc.burst.prompt_len = {num(*jb, s, "prompt_mean"), num(*jb, s, "prompt_p90")};
    sc.burst.output_len = {num(*jb, s, "output_mean"), num(*jb, s, "output_p90")};
    sc.burst_horizon = ms_to_us(num(*jb, s, "horizon_ms"));
    const Json* seed = find(*jb, "seed");
    if (!seed) throw ConfigError("missing required key 'trace.bursty.seed'");
    sc.burst.seed = static_cast<std::uint64_t>(seed->is_int ? seed->i : static_cast<int64_t>(seed->num));
  }
  if (sc.trace_file.empty() == !sc.bursty)
    throw ConfigError("trace must name exactly one of 'file' or 'bursty'");
  sc.max_requests = static_cast<int64_t>(num(jt, "trace", "max_requests", 0.0));
  sc.scale = num(jt, "trace", "scale", 1.0);
  if (!(sc.scale > 0.0)) throw ConfigError("trace.scale must be > 0");
  const Json& js = *section(j, "slo");
  keys(js, "slo", {"ttft_ms", "tpot_ms"});
  sc.slo = {ms_to_us(num(js, "slo", "ttft_ms")), ms_to_us(num(js, "slo", "tpot_ms"))};
  if (sc.slo.ttft_slo <= 0 || sc.slo.tpot_slo <= 0) throw ConfigError("slo targets must be positive");
  sc.burst.ttft_slo = sc.slo.ttft_slo;
  sc.burst.tpot_slo = sc.slo.tpot_slo;
  const Json& jc = *section(j, "cost_model");
  keys(jc, "cost_model", {"truth", "noise_amplitude"});
  const Json* truth = find(jc, "truth");
  if (!truth) throw ConfigError("missing required key 'cost_model.truth'");
  sc.truth = model(*truth, "cost_model.truth");
  sc.noise_amplitude = num(jc, "cost_model", "noise_amplitude", 0.0);
  if (!(sc.noise_amplitude >= 0.0 && sc.noise_amplitude < 1.0))
    throw ConfigError("cost_model.noise_amplitude must be in [0, 1)");
  const Json& jsch = *section(j, "scheduler");
  keys(jsch, "scheduler", {"policy", "token_budget", "max_chunk", "model"});
  const Json* pol = find(jsch, "policy");
  if (!pol || !parse_policy(pol->str, sc.scheduler.policy))
    throw ConfigError("scheduler.policy must be one of prefill_first, sarathi, fairbatch, "
                      "fairbatch_pab; got '" + (pol ? pol->str : std::string()) + "'");
  sc.scheduler.token_budget = static_cast<int64_t>(num(jsch, "scheduler", "token_budget", 2048.0));
  sc.scheduler.max_chunk = static_cast<int32_t>(
      num(jsch, "scheduler", "max_chunk", static_cast<double>(sc.scheduler.token_budget)));
  const Json* m = find(jsch, "model");
  sc.scheduler.model = m ? model(*m, "scheduler.model") : sc.truth;
  static const Json kEmpty = [] {
    Json e;
    e.kind = Json::kObj;
    return e;
  }();
  const Json* jclp = find(j, "cluster");
  const Json& jcl = jclp ? *jclp : kEmpty;
  keys(jcl, "cluster", {"nodes", "policy", "report_interval_steps", "report_latency_ms",
                        "w_waiting", "w_running", "retry_reroute"});
  sc.nodes = static_cast<int>(num(jcl, "cluster", "nodes", 1.0));
  if (sc.nodes < 1) throw ConfigError("cluster.nodes must be >= 1");
  const Json* lbp = find(jcl, "policy");
  const std::string lbs = lbp ? lbp->str : "pab_lb";
  if (lbs != "pab_lb" && lbs != "count_lb")
    throw ConfigError("cluster.policy must be count_lb or pab_lb; got '" + lbs + "'");
  sc.lb.policy = lbs == "pab_lb" ? LbPolicy::kPabLb : LbPolicy::kCountLb;
  sc.lb.report_interval_steps = static_cast<int>(num(jcl, "cluster", "report_interval_steps", 1.0));
  const double lat = num(jcl, "cluster", "report_latency_ms", 0.0);
  if (lat < 0) throw ConfigError("cluster.report_latency_ms must be >= 0");
  sc.lb.report_latency = ms_to_us(lat);
  sc.lb.w_waiting = num(jcl, "cluster", "w_waiting", 1.0);
  sc.lb.w_running = num(jcl, "cluster", "w_running", 1.0);
  if (const Json* rr = find(jcl, "retry_reroute")) sc.lb.retry_reroute = rr->b;
  const Json& jr = *section(j, "run");
  keys(jr, "run", {"horizon_ms", "seed", "out_dir", "max_active", "lead_bucket_ms", "alt_tpot"});
  sc.horizon = ms_to_us(num(jr, "run", "horizon_ms"));
  if (sc.horizon <= 0) throw ConfigError("run.horizon_ms must be > 0");
  const Json* seed = find(jr, "seed");
  if (!seed) throw ConfigError("missing required key 'run.seed' (seeds are explicit)");
  sc.seed = static_cast<std::uint64_t>(seed->is_int ? seed->i : static_cast<int64_t>(seed->num));
  if (const Json* od = find(jr, "out_dir")) sc.out_dir = od->str;
  sc.max_active = static_cast<int32_t>(num(jr, "run", "max_active", 0.0));
  sc.lead_bucket = ms_to_us(num(jr, "run", "lead_bucket_ms", 1000.0));
  if (const Json* at = find(jr, "alt_tpot")) sc.alt_tpot = at->b;
  const SchedulerConfig& s = sc.scheduler;  // validate_scheduler_config, sched.cpp:81-88
  if (s.max_chunk < 1 || s.token_budget < s.max_chunk || s.model.a_ms < 0 || s.model.b_ms <= 0 ||
      s.model.c_ms < 0)
    throw ValidationError("invalid scheduler configuration");
  return sc;
}

Scenario load_scenario(const std::string& path) {
  return scenario_from_json(slurp(path, "scenario file"));
}

Trace materialize_trace(const Scenario& sc) {
  Trace t = sc.bursty ? generate_bursty(sc.burst, sc.burst_horizon)
                      : load_trace(sc.trace_file, sc.trace_format, sc.slo.ttft_slo, sc.slo.tpot_slo);
  if (sc.scale != 1.0) t = scale_trace(t, sc.scale);
  if (sc.max_requests > 0 && static_cast<size_t>(sc.max_requests) < t.requests.size())
    t.requests.resize(static_cast<size_t>(sc.max_requests));  // truncate_trace
  return t;
}

EngineConfig engine_config(const Scenario& sc) {
  EngineConfig c;
  c.scheduler = sc.scheduler;
  c.truth_model = sc.truth;
  c.noise = {sc.noise_amplitude, derive_seed(sc.seed, 3)};
  c.global_slo = sc.slo;
  c.max_active = sc.max_active;
  return c;
}

// ----------------------------------------------------------------- reports

PercentileRow percentiles(std::vector<double> v) {
  PercentileRow row;
  row.count = v.size();
  if (v.empty()) return row;
  std::sort(v.begin(), v.end());
  auto rank = [&](double p) {
    size_t r = static_cast<size_t>(std::ceil(p / 100.0 * static_cast<double>(v.size())));
    r = std::min(std::max<size_t>(r, 1), v.size());
    return v[r - 1];
  };
  row.p50 = rank(50.0);
  row.p95 = rank(95.0);
  row.p99 = rank(99.0);
  return row;
}

ScenarioReport scenario_report(const std::vector<RequestReport>& reports, double offered_rps,
                               const std::string& name, bool alt_tpot) {
  ScenarioReport rep;
  rep.name = name;
  rep.offered_rps = offered_rps;
  rep.total_requests = reports.size();
  std::vector<double> ttft, tpot, alt;
  for (const RequestReport& r : reports) {
    rep.rejected += r.rejected;
    rep.finished += r.finished;
    rep.good += r.good();
    if (r.has_ttft()) ttft.push_back(r.ttft_ms());
    if (r.tokens_emitted >= 2) tpot.push_back(r.max_tpot_ms());
    if (alt_tpot && r.tokens_emitted >= 3) alt.push_back(r.max_tpot_alt_ms());
  }
  const double frac = rep.total_requests == 0
                          ? 0.0
                          : static_cast<double>(rep.good) / static_cast<double>(rep.total_requests);
  rep.slo_violation_rate = 1.0 - frac;
  rep.effective_rps = offered_rps * frac;
  rep.ttft_ms = percentiles(std::move(ttft));
  rep.max_tpot_ms = percentiles(std::move(tpot));
  rep.max_tpot_alt_ms = percentiles(std::move(alt));
  return rep;
}

ScenarioReport run_scenario(const Scenario& sc, int device) {
  const Trace trace = materialize_trace(sc);
  const EngineConfig cfg = engine_config(sc);
  std::vector<RequestReport> reports;
  if (sc.nodes == 1) {
    NodeBatch nb({&trace}, {cfg}, sc.horizon, device);
    nb.run();
    // run_node enqueues in trace order: the first n_arrived rows arrived
    std::vector<RequestReport> all = nb.reports()[0];
    const size_t n_arrived = static_cast<size_t>(nb.summaries()[0].n_arrived);
    reports.assign(all.begin(), all.begin() + static_cast<std::ptrdiff_t>(std::min(n_arrived, all.size())));
  } else {
    reports = run_cluster(trace, std::vector<EngineConfig>(static_cast<size_t>(sc.nodes), cfg),
                          sc.lb, sc.horizon, device)
                  .reports;
  }
  return scenario_report(reports, offered_rps(trace), sc.name, sc.alt_tpot);
}

}  // namespace fbsim_gpu
