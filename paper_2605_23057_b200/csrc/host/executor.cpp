// Mode executor: the reference's simulate_request / run_policy / summarize
// (sim.cpp:80-263) with the latency model replaced by execution on the B200
// engine through its C ABI. See include/modeswitch/executor.hpp.
#include "modeswitch/executor.hpp"

#include <cmath>
#include <cstdio>
#include <fstream>
#include <limits>
#include <map>

#include "modeswitch/energy.hpp"
#include "msw_engine.h"

namespace modeswitch {
namespace {

std::uint64_t mix64(std::uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

std::uint64_t hash_str(const std::string& s) {  // FNV-1a 64
  std::uint64_t h = 0xcbf29ce484222325ull;
  for (unsigned char c : s) h = (h ^ c) * 0x100000001b3ull;
  return h;
}

bool is_shared_prefix(const RequestDescriptor& r) {
  return r.shared_prefix ||
         (r.workload_tag && *r.workload_tag == WorkloadFamily::SharedPrefixChat);
}

void check(int rc, const char* what) {
  if (rc == 0) return;
  const std::string msg = std::string(what) + ": " + msw_last_error();
  if (rc == 2) throw ConfigError(msg);
  if (rc == 3) throw DataError(msg);
  throw Error(msg);
}

struct RunOut {
  int rc = 0;
  std::vector<std::int32_t> tokens;
  msw_result res{};
};

RunOut run_one(msw_engine* e, int mode, const std::vector<std::int32_t>& prompt, int n_new) {
  RunOut o;
  o.tokens.assign(n_new, 0);
  msw_request req{};
  req.mode = mode;
  req.prompt_ids = prompt.data();
  req.prompt_len = static_cast<int32_t>(prompt.size());
  req.max_new_tokens = n_new;
  req.prefix_group = -1;
  o.res.out_ids = o.tokens.data();
  o.rc = msw_engine_run(e, &req, &o.res);
  return o;
}

int output_len(const RequestDescriptor& r, const ExecOptions& o) {
  int n = r.expected_output_tokens;
  if (o.max_output_tokens > 0 && n > o.max_output_tokens) n = o.max_output_tokens;
  return n;
}

double charged_overhead(const RoutingDecision& d, const ExecOptions& o) {
  return (o.zero_overhead ? 0.0 : d.overhead_ms) + o.extra_overhead_ms;
}

// Joules of one engine call on o.power_device: the driver's energy counter
// over the call, or the trapezoid of the sampled power trace when the counter
// did not advance (short windows); -1 when energy is not measured.
template <typename F>
double measured_joules(const ExecOptions& o, F&& call) {
  if (o.power_device < 0) {
    call();
    return -1.0;
  }
  PowerSampler ps(o.power_device, 2.0);
  ps.start();
  call();
  const PowerTrace tr = ps.stop();
  const double cj = ps.counter_joules();
  if (cj > 0.0) return cj;
  return tr.samples.size() >= 2 ? energy_from_power_trace(tr, 1) : -1.0;
}

double memory_bytes(msw_engine* e, InferenceMode mode, int tokens) {
  int64_t b = 0;
  check(msw_engine_memory_bytes(e, static_cast<int32_t>(mode), tokens, &b), "memory bytes");
  return static_cast<double>(b);
}

// SimRequestResult fields that follow from the measured runs (sim.cpp:136-143)
void finish_ratios(msw_engine* e, ExecRequestResult& r, double fp16_joules, const ExecOptions& o) {
  const int tokens = r.prompt_tokens + r.output_tokens;
  r.memory_ratio = memory_bytes(e, r.executed_mode, tokens) /
                   memory_bytes(e, InferenceMode::FP16, tokens);
  if (r.energy_j > 0.0 && fp16_joules > 0.0) r.energy_ratio = r.energy_j / fp16_joules;
  const auto q = o.quality_delta_pp.find(r.executed_mode);
  r.quality_delta_pp = q == o.quality_delta_pp.end() ? 0.0 : q->second;
  r.constraint_violated = !(r.quality_delta_pp >= o.constraints.quality_floor_pp &&
                            r.energy_ratio <= o.constraints.energy_ratio_max &&
                            r.memory_ratio <= o.constraints.memory_ratio_max);
}

}  // namespace

int prefix_group(const std::string& request_id, int groups) {
  if (groups <= 1) return 0;
  return static_cast<int>(hash_str(request_id) % static_cast<std::uint64_t>(groups));
}

std::vector<std::int32_t> synth_prompt(const RequestDescriptor& r, std::uint64_t seed, int vocab,
                                       int prefix_len, int prompt_cap, int prefix_groups) {
  if (vocab < 2) throw ConfigError("synth_prompt: vocab must be >= 2");
  int n = r.prompt_tokens;
  if (prompt_cap > 0 && n > prompt_cap) n = prompt_cap;
  std::vector<std::int32_t> ids(n);
  const std::uint64_t rkey = mix64(seed ^ hash_str(r.request_id));
  const std::string group = "prefix-group-" + std::to_string(prefix_group(r.request_id, prefix_groups));
  const std::uint64_t pkey = mix64(seed ^ hash_str(group));
  const int shared = is_shared_prefix(r) ? std::min(prefix_len, n - 1) : 0;
  for (int i = 0; i < n; ++i) {
    const std::uint64_t k = i < shared ? pkey : rkey;
    ids[i] = static_cast<std::int32_t>(mix64(k + static_cast<std::uint64_t>(i)) %
                                       static_cast<std::uint64_t>(vocab));
  }
  return ids;
}

ExecRequestResult execute_request(msw_engine* e, const RequestDescriptor& request,
                                  const RoutingDecision& decision, const ExecOptions& o) {
  validate(request);
  ExecRequestResult out;
  out.request_id = request.request_id;
  out.decision = decision;
  out.family = resolve_family(request, o.classifier);
  const auto prompt = synth_prompt(request, o.token_seed, o.vocab, o.prefix_len, o.max_prompt_tokens,
                                   o.prefix_groups);
  const int n_new = output_len(request, o);
  out.prompt_tokens = static_cast<int>(prompt.size());
  out.output_tokens = n_new;

  // batching guard (sim.cpp:104-106): batching-only modes need co-scheduled work
  int mode = static_cast<int>(decision.mode);
  std::string problem;
  if (requires_batching(decision.mode) && request.batch_pressure <= 1)
    problem = std::string(to_string(decision.mode)) + " applies only to batched requests";
  RunOut run;
  double joules = -1.0;
  if (problem.empty()) {
    joules = measured_joules(o, [&] { run = run_one(e, mode, prompt, n_new); });
    if (run.rc != 0) problem = msw_last_error();
  }
  if (!problem.empty()) {
    if (!o.fallback_enabled)
      throw DataError("request '" + request.request_id + "': " + problem +
                      " and FP16 fallback is disabled");
    mode = static_cast<int>(InferenceMode::FP16);
    joules = measured_joules(o, [&] { run = run_one(e, mode, prompt, n_new); });
    check(run.rc, "FP16 fallback");
    out.fallback_used = true;
  }
  out.executed_mode = static_cast<InferenceMode>(mode);
  out.overhead_ms = charged_overhead(decision, o);
  out.mode_latency_ms = run.res.total_ms + out.overhead_ms;
  out.prefill_ms = run.res.prefill_ms;
  out.decode_ms = run.res.decode_ms;
  out.spec_proposed = run.res.spec_proposed;
  out.spec_accepted = run.res.spec_accepted;
  out.prefix_hit_tokens = run.res.prefix_hit_tokens;
  out.tokens = std::move(run.tokens);
  out.energy_j = joules;
  double fp16_joules = -1.0;
  if (o.measure_fp16_baseline) {
    if (mode == static_cast<int>(InferenceMode::FP16)) {
      out.fp16_latency_ms = run.res.total_ms;
      fp16_joules = joules;
    } else {
      RunOut base;
      fp16_joules = measured_joules(
          o, [&] { base = run_one(e, static_cast<int>(InferenceMode::FP16), prompt, n_new); });
      check(base.rc, "FP16 baseline");
      out.fp16_latency_ms = base.res.total_ms;
    }
    out.speedup = speedup(out.fp16_latency_ms, out.mode_latency_ms);
  }
  finish_ratios(e, out, fp16_joules, o);
  return out;
}

ExecRunResult run_policy(const std::vector<RequestDescriptor>& trace, const RoutingPolicy& policy,
                         msw_engine* e, const ExecOptions& o) {
  if (trace.empty()) throw DataError("run_policy: empty trace");
  ExecRunResult run;
  run.report.policy = policy.name();
  run.results.resize(trace.size());
  std::vector<RoutingDecision> decisions(trace.size());
  for (size_t i = 0; i < trace.size(); ++i) decisions[i] = policy.route(trace[i]);

  const auto cb = InferenceMode::INT8PlusContinuousBatching;
  for (size_t i = 0; i < trace.size();) {
    if (decisions[i].mode != cb || trace[i].batch_pressure <= 1) {
      run.results[i] = execute_request(e, trace[i], decisions[i], o);
      ++i;
      continue;
    }
    // continuous-batching cohort: maximal run of consecutive CB-routed requests
    size_t j = i;
    while (j < trace.size() && j - i < static_cast<size_t>(o.cohort_max) &&
           decisions[j].mode == cb && trace[j].batch_pressure > 1)
      ++j;
    const size_t n = j - i;
    std::vector<std::vector<std::int32_t>> prompts(n), toks(n);
    std::vector<msw_request> reqs(n);
    std::vector<msw_result> res(n);
    for (size_t q = 0; q < n; ++q) {
      prompts[q] = synth_prompt(trace[i + q], o.token_seed, o.vocab, o.prefix_len,
                                o.max_prompt_tokens, o.prefix_groups);
      const int n_new = output_len(trace[i + q], o);
      toks[q].assign(n_new, 0);
      reqs[q] = msw_request{static_cast<int32_t>(cb), prompts[q].data(),
                            static_cast<int32_t>(prompts[q].size()), n_new, -1, 0, i + q};
      res[q] = msw_result{};
      res[q].out_ids = toks[q].data();
    }
    int rc = 0;
    const double cohort_joules = measured_joules(
        o, [&] { rc = msw_engine_run_batch(e, reqs.data(), static_cast<int32_t>(n), res.data()); });
    long long cohort_tokens = 0;
    for (size_t q = 0; q < n; ++q) cohort_tokens += static_cast<long long>(toks[q].size());
    if (rc != 0) {  // whole cohort falls back to batch-1 FP16 (flagged per request)
      if (!o.fallback_enabled) check(rc, "continuous batching");
      for (size_t q = 0; q < n; ++q) {
        RoutingDecision d = decisions[i + q];
        ExecRequestResult r = execute_request(e, trace[i + q], route_static(InferenceMode::FP16), o);
        r.decision = d;
        r.fallback_used = true;
        run.results[i + q] = std::move(r);
      }
      i = j;
      continue;
    }
    for (size_t q = 0; q < n; ++q) {
      ExecRequestResult& r = run.results[i + q];
      r.request_id = trace[i + q].request_id;
      r.decision = decisions[i + q];
      r.executed_mode = cb;
      r.family = resolve_family(trace[i + q], o.classifier);
      r.prompt_tokens = static_cast<int>(prompts[q].size());
      r.output_tokens = static_cast<int>(toks[q].size());
      r.overhead_ms = charged_overhead(r.decision, o);
      r.mode_latency_ms = res[q].total_ms + r.overhead_ms;
      r.prefill_ms = res[q].prefill_ms;
      r.decode_ms = res[q].decode_ms;
      r.tokens = std::move(toks[q]);
      // the cohort's energy, split by generated tokens
      if (cohort_joules > 0.0 && cohort_tokens > 0)
        r.energy_j = cohort_joules * static_cast<double>(r.output_tokens) /
                     static_cast<double>(cohort_tokens);
      double fp16_joules = -1.0;
      if (o.measure_fp16_baseline) {
        RunOut base;
        fp16_joules = measured_joules(o, [&] {
          base = run_one(e, static_cast<int>(InferenceMode::FP16), prompts[q], r.output_tokens);
        });
        check(base.rc, "FP16 baseline");
        r.fp16_latency_ms = base.res.total_ms;
        r.speedup = speedup(r.fp16_latency_ms, r.mode_latency_ms);
      }
      finish_ratios(e, r, fp16_joules, o);
    }
    i = j;
  }

  // summarize (sim.cpp:149-207): unweighted means, per-family, collapsed, aggregate
  ExecReport& rep = run.report;
  rep.request_count = static_cast<int>(run.results.size());
  double tot_fp16 = 0.0, tot_mode = 0.0;
  std::map<WorkloadFamily, ExecFamilySummary> fam;
  int violations = 0;
  for (const auto& r : run.results) {
    rep.mean_speedup += r.speedup;
    rep.mean_energy_ratio += r.energy_ratio;
    rep.mean_memory_ratio += r.memory_ratio;
    rep.mean_quality_delta_pp += r.quality_delta_pp;
    if (r.constraint_violated) ++violations;
    rep.mean_overhead_ms += r.overhead_ms;
    tot_fp16 += r.fp16_latency_ms;
    tot_mode += r.mode_latency_ms;
    rep.generated_tokens += r.output_tokens;
    if (r.fallback_used) ++rep.fallback_count;
    ExecFamilySummary& f = fam[r.family];
    f.family = r.family;
    f.count += 1;
    f.mean_speedup += r.speedup;
    f.mean_energy_ratio += r.energy_ratio;
    f.mean_memory_ratio += r.memory_ratio;
    f.mean_quality_delta_pp += r.quality_delta_pp;
  }
  const double n = static_cast<double>(run.results.size());
  rep.mean_speedup /= n;
  rep.mean_energy_ratio /= n;
  rep.mean_memory_ratio /= n;
  rep.mean_quality_delta_pp /= n;
  rep.constraint_violation_rate = violations / n;
  rep.mean_overhead_ms /= n;
  rep.aggregate_latency_speedup = tot_mode > 0.0 ? tot_fp16 / tot_mode : 0.0;
  rep.mode_time_ms = tot_mode;
  for (auto& kv : fam) {
    ExecFamilySummary& f = kv.second;
    f.mean_speedup /= f.count;
    f.mean_energy_ratio /= f.count;
    f.mean_memory_ratio /= f.count;
    f.mean_quality_delta_pp /= f.count;
    rep.per_family.push_back(f);
    rep.collapsed_mean_speedup += f.mean_speedup;
    rep.collapsed_mean_energy_ratio += f.mean_energy_ratio;
  }
  rep.collapsed_mean_speedup /= static_cast<double>(rep.per_family.size());
  rep.collapsed_mean_energy_ratio /= static_cast<double>(rep.per_family.size());
  return run;
}

void write_decisions_csv(const std::vector<ExecRequestResult>& results,
                         const std::filesystem::path& path) {
  std::ofstream out(path);
  if (!out) throw DataError("cannot write decisions file: " + path.string());
  out << "request_id,mode,reason,overhead_ms\n";
  char buf[64];
  for (const auto& r : results) {
    std::snprintf(buf, sizeof(buf), "%.17g", r.decision.overhead_ms);
    out << r.request_id << ',' << to_string(r.decision.mode) << ',' << to_string(r.decision.reason)
        << ',' << buf << '\n';
  }
}

ExecQualityGate evaluate_quality_gate(const std::vector<ExecRequestResult>& results,
                                      double threshold_pp) {
  ExecQualityGate gate;
  std::map<WorkloadFamily, ExecFamilySummary> fam;
  for (const auto& r : results) {
    if (!is_benchmark_family(r.family)) continue;
    ExecFamilySummary& f = fam[r.family];
    f.family = r.family;
    f.count += 1;
    f.mean_quality_delta_pp += r.quality_delta_pp;
    f.mean_speedup += r.speedup;
    f.mean_energy_ratio += r.energy_ratio;
    f.mean_memory_ratio += r.memory_ratio;
  }
  if (fam.empty()) return gate;  // no benchmark traffic, nothing to gate
  double collapsed = 0.0;
  for (auto& kv : fam) {
    ExecFamilySummary& f = kv.second;
    f.mean_quality_delta_pp /= f.count;
    f.mean_speedup /= f.count;
    f.mean_energy_ratio /= f.count;
    f.mean_memory_ratio /= f.count;
    collapsed += f.mean_quality_delta_pp;
    gate.benchmark_families.push_back(f);
  }
  collapsed /= static_cast<double>(fam.size());
  gate.collapsed_benchmark_delta_pp = collapsed;
  gate.passed = std::abs(collapsed) <= threshold_pp;
  return gate;
}

namespace {
std::string fmt17(double v) {  // the reference's format_double (report.cpp:9-13)
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}
}  // namespace

void write_comparison_csv(const std::vector<ExecRunResult>& runs,
                          const std::filesystem::path& path) {
  std::ofstream out(path);
  if (!out) throw DataError("cannot write comparison CSV: " + path.string());
  out << "policy,request_count,mean_speedup,mean_energy_ratio,"
         "mean_memory_ratio,mean_quality_delta_pp,collapsed_mean_speedup,"
         "collapsed_mean_energy_ratio,aggregate_latency_speedup,"
         "oracle_match_rate,constraint_violation_rate,mean_overhead_ms,"
         "synthesized_cell_usage,fallback_count,oracle_capture\n";
  const double nan = std::numeric_limits<double>::quiet_NaN();
  for (const auto& run : runs) {
    const ExecReport& p = run.report;
    out << p.policy << ',' << p.request_count << ',' << fmt17(p.mean_speedup) << ','
        << fmt17(p.mean_energy_ratio) << ',' << fmt17(p.mean_memory_ratio) << ','
        << fmt17(p.mean_quality_delta_pp) << ',' << fmt17(p.collapsed_mean_speedup) << ','
        << fmt17(p.collapsed_mean_energy_ratio) << ',' << fmt17(p.aggregate_latency_speedup) << ','
        << fmt17(nan) << ',' << fmt17(p.constraint_violation_rate) << ','
        << fmt17(p.mean_overhead_ms) << ',' << fmt17(0.0) << ',' << p.fallback_count << ','
        << fmt17(nan) << '\n';
  }
}

void write_results_csv(const std::vector<ExecRequestResult>& results,
                       const std::filesystem::path& path) {
  std::ofstream out(path);
  if (!out) throw DataError("cannot write results CSV: " + path.string());
  out << "request_id,mode,reason,overhead_ms,simulated_mode,family,fp16_latency_ms,"
         "mode_latency_ms,speedup,energy_ratio,memory_ratio,quality_delta_pp,energy_j,"
         "constraint_violated,used_synthesized_cell,fallback_used\n";
  for (const auto& r : results) {
    out << r.request_id << ',' << to_string(r.decision.mode) << ','
        << to_string(r.decision.reason) << ',' << fmt17(r.decision.overhead_ms) << ','
        << to_string(r.executed_mode) << ',' << to_string(r.family) << ','
        << fmt17(r.fp16_latency_ms) << ',' << fmt17(r.mode_latency_ms) << ','
        << fmt17(r.speedup) << ',' << fmt17(r.energy_ratio) << ',' << fmt17(r.memory_ratio)
        << ',' << fmt17(r.quality_delta_pp) << ',' << fmt17(r.energy_j) << ','
        << (r.constraint_violated ? 1 : 0) << ",0," << (r.fallback_used ? 1 : 0) << '\n';
  }
}

}  // namespace modeswitch
