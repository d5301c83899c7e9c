// C ABI over the host controller (include/msw_host.h).
#include <chrono>
#include <memory>
#include <cstring>
#include <sstream>
#include <string>

#include "modeswitch/classifier.hpp"
#include "modeswitch/energy.hpp"
#include "modeswitch/executor.hpp"
#include "modeswitch/routing.hpp"
#include "modeswitch/trace_io.hpp"
#include "modeswitch/workload.hpp"
#include "msw_host.h"

namespace ms = modeswitch;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& body) {
  try {
    body();
    return MSW_OK;
  } catch (const ms::ConfigError& e) {
    g_err = e.what();
    return MSW_ERR_CONFIG;
  } catch (const ms::DataError& e) {
    g_err = e.what();
    return MSW_ERR_DATA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MSW_ERR_OTHER;
  } catch (...) {
    g_err = "unknown error";
    return MSW_ERR_OTHER;
  }
}

ms::RequestDescriptor to_cpp(const msw_descriptor& d) {
  ms::RequestDescriptor r;
  if (d.request_id == nullptr) throw ms::DataError("request_id is NULL");
  r.request_id = d.request_id;
  r.prompt_tokens = d.prompt_tokens;
  r.expected_output_tokens = d.expected_output_tokens;
  r.shared_prefix = d.shared_prefix != 0;
  r.memory_pressure = d.memory_pressure != 0;
  r.batch_pressure = d.batch_pressure;
  if (d.workload_tag >= 0) {
    if (d.workload_tag >= ms::kFamilyCount)
      throw ms::DataError("workload_tag out of range");
    r.workload_tag = static_cast<ms::WorkloadFamily>(d.workload_tag);
  } else if (d.workload_tag != -1) {
    throw ms::DataError("workload_tag out of range");
  }
  return r;
}

ms::ClassifierConfig to_cpp(const msw_classifier_cfg* c) {
  ms::ClassifierConfig cfg;
  if (c) {
    cfg.long_prompt_threshold = c->long_prompt_threshold;
    cfg.long_output_threshold = c->long_output_threshold;
    cfg.decode_heavy_ratio = c->decode_heavy_ratio;
    cfg.batch_threshold = c->batch_threshold;
  }
  ms::validate(cfg);
  return cfg;
}

void fill(const ms::RequestDescriptor& r, const ms::ClassifierConfig& cfg,
          const ms::RoutingDecision& d, msw_route_out* out) {
  out->mode = static_cast<int32_t>(d.mode);
  out->reason = static_cast<int32_t>(d.reason);
  out->workload_class =
      static_cast<int32_t>(ms::classify(ms::extract_features(r), cfg));
  out->family = static_cast<int32_t>(ms::resolve_family(r, cfg));
  out->overhead_ms = d.overhead_ms;
}

std::vector<ms::RequestDescriptor> parse_ndjson(const char* text) {
  if (text == nullptr) throw ms::DataError("trace text is NULL");
  std::vector<ms::RequestDescriptor> out;
  std::istringstream in(text);
  std::string line;
  for (size_t lineno = 1; std::getline(in, line); ++lineno) {
    if (line.empty()) continue;
    try {
      out.push_back(ms::parse_trace_line(line));
    } catch (const ms::DataError& e) {
      throw ms::DataError("line " + std::to_string(lineno) + ": " + e.what());
    }
  }
  return out;
}

void copy_out(const std::string& s, char* buf, size_t cap, size_t* needed) {
  if (needed) *needed = s.size() + 1;
  if (buf == nullptr || cap < s.size() + 1)
    throw ms::Error("output buffer too small");
  std::memcpy(buf, s.c_str(), s.size() + 1);
}

}  // namespace

extern "C" {

int msw_route_rule(const msw_descriptor* d, const msw_classifier_cfg* c,
                   msw_route_out* out) {
  return guarded([&] {
    if (!d || !out) throw ms::DataError("NULL argument");
    const ms::RequestDescriptor r = to_cpp(*d);
    ms::validate(r);
    const ms::ClassifierConfig cfg = to_cpp(c);
    const ms::RulePolicy policy(cfg);
    fill(r, cfg, policy.route(r), out);
  });
}

int msw_route_ndjson(const char* ndjson, const msw_classifier_cfg* c,
                     int32_t n_max, msw_route_out* out, int32_t* n_out) {
  return guarded([&] {
    const auto trace = parse_ndjson(ndjson);
    if (n_out) *n_out = static_cast<int32_t>(trace.size());
    if (static_cast<int64_t>(trace.size()) > n_max)
      throw ms::Error("output array too small");
    const ms::ClassifierConfig cfg = to_cpp(c);
    const ms::RulePolicy policy(cfg);
    for (size_t i = 0; i < trace.size(); ++i)
      fill(trace[i], cfg, policy.route(trace[i]), &out[i]);
  });
}

int msw_trace_parse_line(const char* line, msw_descriptor* out, char* id_buf,
                         size_t id_cap) {
  return guarded([&] {
    if (!line || !out) throw ms::DataError("NULL argument");
    const ms::RequestDescriptor r = ms::parse_trace_line(line);
    copy_out(r.request_id, id_buf, id_cap, nullptr);
    out->request_id = id_buf;
    out->prompt_tokens = r.prompt_tokens;
    out->expected_output_tokens = r.expected_output_tokens;
    out->shared_prefix = r.shared_prefix;
    out->memory_pressure = r.memory_pressure;
    out->batch_pressure = r.batch_pressure;
    out->workload_tag = r.workload_tag ? static_cast<int32_t>(*r.workload_tag) : -1;
  });
}

int msw_trace_format_line(const msw_descriptor* d, char* buf, size_t cap,
                          size_t* needed) {
  return guarded([&] {
    if (!d) throw ms::DataError("NULL argument");
    copy_out(ms::format_trace_line(to_cpp(*d)), buf, cap, needed);
  });
}

int msw_trace_generate(const int32_t counts[11], double jitter, uint64_t seed,
                       int32_t batch_pressure, double batched_fraction,
                       char* buf, size_t cap, size_t* needed) {
  return guarded([&] {
    ms::TraceSpec spec;
    for (int i = 0; i < ms::kFamilyCount; ++i)
      if (counts[i] != 0) spec.counts[static_cast<ms::WorkloadFamily>(i)] = counts[i];
    spec.jitter = jitter;
    spec.seed = seed;
    spec.batch_pressure = batch_pressure;
    spec.batched_fraction = batched_fraction;
    std::string text;
    for (const auto& r : ms::generate_trace(spec))
      text += ms::format_trace_line(r) + "\n";
    copy_out(text, buf, cap, needed);
  });
}

int msw_route_cost(const char* ndjson, int32_t passes, double* mean_stamp_ms,
                   double* wall_ms_per_decision) {
  return guarded([&] {
    const auto trace = parse_ndjson(ndjson);
    if (trace.empty() || passes < 1) throw ms::ConfigError("nothing to route");
    const ms::RulePolicy policy;
    double stamped = 0.0;
    long n = 0;
    volatile int sink = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int p = 0; p < passes; ++p)
      for (const auto& r : trace) {
        const auto d = policy.route(r);
        stamped += d.overhead_ms;
        sink = sink + static_cast<int>(d.mode);
        ++n;
      }
    const double wall = std::chrono::duration<double, std::milli>(
                            std::chrono::steady_clock::now() - t0)
                            .count();
    if (mean_stamp_ms) *mean_stamp_ms = stamped / double(n);
    if (wall_ms_per_decision) *wall_ms_per_decision = wall / double(n);
  });
}

int msw_execute_trace(struct msw_engine* engine, int32_t vocab, const char* ndjson,
                      const msw_classifier_cfg* c, const msw_exec_opts* opts, int32_t n_max,
                      msw_exec_row* rows, int32_t* n_out, msw_exec_summary* summary) {
  return guarded([&] {
    if (!engine || !opts) throw ms::ConfigError("NULL engine/options");
    const auto trace = parse_ndjson(ndjson);
    if (n_out) *n_out = static_cast<int32_t>(trace.size());
    if (static_cast<int64_t>(trace.size()) > n_max) throw ms::Error("output array too small");
    ms::ExecOptions o;
    o.classifier = to_cpp(c);
    o.fallback_enabled = opts->fallback_enabled != 0;
    o.zero_overhead = opts->zero_overhead != 0;
    o.extra_overhead_ms = opts->extra_overhead_ms;
    o.measure_fp16_baseline = opts->measure_fp16_baseline != 0;
    o.token_seed = opts->token_seed;
    o.prefix_len = opts->prefix_len;
    o.max_output_tokens = opts->max_output_tokens;
    o.max_prompt_tokens = opts->max_prompt_tokens;
    o.cohort_max = opts->cohort_max > 0 ? opts->cohort_max : 64;
    o.vocab = vocab;
    o.constraints.quality_floor_pp = opts->quality_floor_pp;
    o.constraints.energy_ratio_max = opts->energy_ratio_max;
    o.constraints.memory_ratio_max = opts->memory_ratio_max;
    ms::validate(o.constraints);
    o.power_device = opts->power_device;
    o.prefix_groups = opts->prefix_groups > 1 ? opts->prefix_groups : 1;
    if (opts->quality_delta_pp)
      for (int m = 0; m < ms::kModeCount; ++m)
        o.quality_delta_pp[static_cast<ms::InferenceMode>(m)] = opts->quality_delta_pp[m];
    const ms::RulePolicy policy(o.classifier);
    const ms::ExecRunResult run = ms::run_policy(trace, policy, engine, o);
    for (size_t i = 0; i < run.results.size(); ++i) {
      const auto& r = run.results[i];
      msw_exec_row& w = rows[i];
      w.mode = static_cast<int32_t>(r.decision.mode);
      w.reason = static_cast<int32_t>(r.decision.reason);
      w.executed_mode = static_cast<int32_t>(r.executed_mode);
      w.family = static_cast<int32_t>(r.family);
      w.prompt_tokens = r.prompt_tokens;
      w.output_tokens = r.output_tokens;
      w.fallback_used = r.fallback_used;
      w.spec_proposed = r.spec_proposed;
      w.spec_accepted = r.spec_accepted;
      w.prefix_hit_tokens = r.prefix_hit_tokens;
      w.fp16_latency_ms = r.fp16_latency_ms;
      w.mode_latency_ms = r.mode_latency_ms;
      w.speedup = r.speedup;
      w.overhead_ms = r.overhead_ms;
      w.prefill_ms = r.prefill_ms;
      w.decode_ms = r.decode_ms;
      w.energy_j = r.energy_j;
      w.energy_ratio = r.energy_ratio;
      w.memory_ratio = r.memory_ratio;
      w.quality_delta_pp = r.quality_delta_pp;
      w.constraint_violated = r.constraint_violated;
    }
    if (opts->results_csv) ms::write_results_csv(run.results, opts->results_csv);
    if (opts->comparison_csv) ms::write_comparison_csv({run}, opts->comparison_csv);
    if (summary) {
      const auto& p = run.report;
      summary->request_count = p.request_count;
      summary->fallback_count = p.fallback_count;
      summary->mean_speedup = p.mean_speedup;
      summary->aggregate_latency_speedup = p.aggregate_latency_speedup;
      summary->collapsed_mean_speedup = p.collapsed_mean_speedup;
      summary->mean_overhead_ms = p.mean_overhead_ms;
      summary->mode_time_ms = p.mode_time_ms;
      summary->generated_tokens = p.generated_tokens;
      summary->mean_energy_ratio = p.mean_energy_ratio;
      summary->mean_memory_ratio = p.mean_memory_ratio;
      summary->mean_quality_delta_pp = p.mean_quality_delta_pp;
      summary->collapsed_mean_energy_ratio = p.collapsed_mean_energy_ratio;
      summary->constraint_violation_rate = p.constraint_violation_rate;
      const ms::ExecQualityGate gate = ms::evaluate_quality_gate(run.results);
      summary->quality_gate_passed = gate.passed;
      summary->collapsed_benchmark_delta_pp = gate.collapsed_benchmark_delta_pp;
    }
  });
}

int msw_write_decisions_csv(const char* ndjson, const msw_exec_row* rows, int32_t n,
                            const char* path) {
  return guarded([&] {
    if (!ndjson || !rows || !path) throw ms::ConfigError("msw_write_decisions_csv: NULL argument");
    std::istringstream in(ndjson);
    std::string line;
    std::vector<ms::ExecRequestResult> res;
    while (std::getline(in, line) && int32_t(res.size()) < n) {
      if (line.empty()) continue;
      const ms::RequestDescriptor d = ms::parse_trace_line(line);
      ms::ExecRequestResult r;
      const msw_exec_row& w = rows[res.size()];
      r.request_id = d.request_id;
      r.decision.mode = static_cast<ms::InferenceMode>(w.mode);
      r.decision.reason = static_cast<ms::RoutingReason>(w.reason);
      r.decision.overhead_ms = w.overhead_ms;
      res.push_back(std::move(r));
    }
    if (int32_t(res.size()) != n) throw ms::DataError("msw_write_decisions_csv: fewer trace lines than rows");
    ms::write_decisions_csv(res, path);
  });
}

struct msw_power_sampler {
  ms::PowerSampler impl;
  msw_power_sampler(int d, double p) : impl(d, p) {}
};

int msw_power_start(int32_t device, double period_ms, msw_power_sampler** out) {
  return guarded([&] {
    if (!out) throw ms::ConfigError("msw_power_start: out is NULL");
    if (!(period_ms > 0.0)) throw ms::ConfigError("msw_power_start: period_ms must be positive");
    auto* s = new msw_power_sampler(device, period_ms);
    s->impl.start();
    *out = s;
  });
}

int msw_power_stop(msw_power_sampler* s, const char* csv_path, int32_t tokens,
                   double* joules_per_token, int32_t* n_samples, double* counter_joules) {
  return guarded([&] {
    if (!s) throw ms::ConfigError("msw_power_stop: sampler is NULL");
    std::unique_ptr<msw_power_sampler> own(s);
    const ms::PowerTrace tr = own->impl.stop();
    if (counter_joules) *counter_joules = own->impl.counter_joules();
    if (n_samples) *n_samples = int32_t(tr.samples.size());
    if (csv_path && *csv_path) ms::write_power_trace(tr, csv_path);
    if (joules_per_token) *joules_per_token = ms::energy_from_power_trace(tr, tokens);
  });
}

int msw_energy_from_trace(const char* csv_path, int32_t tokens, double* joules_per_token) {
  return guarded([&] {
    if (!csv_path || !joules_per_token) throw ms::ConfigError("msw_energy_from_trace: NULL argument");
    *joules_per_token = ms::energy_from_power_trace(ms::read_power_trace(csv_path), tokens);
  });
}

const char* msw_host_last_error(void) { return g_err.c_str(); }

}  // extern "C"
