// modeswitch-b200 host: the mode executor seam.
//
// Replaces the reference's simulator step (sim.hpp:92-122, sim.cpp:80-263):
// instead of mode_latency = fp16_latency / cell.latency_speedup + overhead
// (sim.cpp:132-135), the routed mode is EXECUTED on a B200 through the C ABI
// (include/msw_engine.h) and the measured latency is used. Everything around
// that step keeps the reference's semantics:
//   * FP16 emergency fallback when the routed mode cannot run (mode not
//     resident, or a batching-only mode on an unbatched request: the batching
//     guard of sim.cpp:104-106), flagged in the result (sim.cpp:112-124);
//   * per-request speedup = FP16 latency / mode latency on the SAME request
//     (domain.cpp:118-123), FP16 measured on the same GPU;
//   * aggregation = unweighted mean over requests, per-family means, the
//     collapsed one-vote-per-family mean and sum(fp16)/sum(mode)
//     (summarize, sim.cpp:149-207); results in trace order;
//   * the rest of SimRequestResult (sim.hpp:40-56), measured instead of read
//     from a profile cell: energy_j / energy_ratio from the driver's energy
//     counter around the mode run and the FP16 run of the same request
//     (ExecOptions::power_device), memory_ratio from the HBM footprint of
//     the mode (weights + this request's KV) over FP16's
//     (msw_engine_memory_bytes), constraint_violated against a ConstraintSet
//     (routing.cpp:56-61 on the measured ratios). quality_delta_pp cannot be
//     measured on random-init weights: it comes from ExecOptions (e.g. the
//     reference profile's cell values), 0 when absent.
#pragma once

#include <cstdint>
#include <filesystem>
#include <map>
#include <string>
#include <vector>

#include "modeswitch/classifier.hpp"
#include "modeswitch/domain.hpp"
#include "modeswitch/routing.hpp"

struct msw_engine;

namespace modeswitch {

struct ExecOptions {
  bool fallback_enabled = true;
  bool zero_overhead = false;       // ignore the measured routing overhead
  double extra_overhead_ms = 0.0;   // injected synthetic routing overhead
  ClassifierConfig classifier;
  bool measure_fp16_baseline = true;
  std::uint64_t token_seed = 0;     // synthetic token ids
  int prefix_len = 768;             // shared-prefix tokens of SharedPrefixChat requests
  int prefix_groups = 1;            // shared-prefix requests split into this many groups
  int max_output_tokens = 0;        // > 0 caps generation (bounded samples)
  int max_prompt_tokens = 0;        // > 0 caps prompt length
  int vocab = 0;                    // engine vocabulary (required)
  int cohort_max = 64;              // continuous-batching cohort size
  ConstraintSet constraints;        // violation accounting (sim.cpp:143)
  int power_device = -1;            // >= 0: measure energy on this CUDA device
  std::map<InferenceMode, double> quality_delta_pp;  // per mode; absent = 0
};

struct ExecRequestResult {
  std::string request_id;
  RoutingDecision decision;
  InferenceMode executed_mode = InferenceMode::FP16;  // FP16 when the fallback hit
  WorkloadFamily family = WorkloadFamily::SyntheticSS;
  int prompt_tokens = 0;
  int output_tokens = 0;
  double fp16_latency_ms = 0.0;   // measured (same request, FP16 mode)
  double mode_latency_ms = 0.0;   // measured + charged overhead
  double speedup = 1.0;
  double overhead_ms = 0.0;
  double prefill_ms = 0.0;
  double decode_ms = 0.0;
  int spec_proposed = 0;
  int spec_accepted = 0;
  int prefix_hit_tokens = 0;
  bool fallback_used = false;
  // reference SimRequestResult fields (sim.hpp:48-53), measured
  double energy_j = -1.0;         // mode run, driver energy counter; -1 = not measured
  double energy_ratio = 1.0;      // (mode J/token) / (FP16 J/token), same request
  double memory_ratio = 1.0;      // mode HBM footprint / FP16's, same request
  double quality_delta_pp = 0.0;  // from ExecOptions::quality_delta_pp
  bool constraint_violated = false;
  std::vector<std::int32_t> tokens;
};

struct ExecFamilySummary {
  WorkloadFamily family = WorkloadFamily::SyntheticSS;
  int count = 0;
  double mean_speedup = 0.0;
  double mean_energy_ratio = 0.0;
  double mean_memory_ratio = 0.0;
  double mean_quality_delta_pp = 0.0;
};

struct ExecReport {
  std::string policy;
  int request_count = 0;
  double mean_speedup = 0.0;
  double aggregate_latency_speedup = 0.0;
  double collapsed_mean_speedup = 0.0;
  double mean_overhead_ms = 0.0;
  int fallback_count = 0;
  double mean_energy_ratio = 0.0;
  double mean_memory_ratio = 0.0;
  double mean_quality_delta_pp = 0.0;
  double collapsed_mean_energy_ratio = 0.0;
  double constraint_violation_rate = 0.0;
  std::vector<ExecFamilySummary> per_family;
  long long generated_tokens = 0;
  double mode_time_ms = 0.0;  // sum of mode latencies
};

struct ExecRunResult {
  ExecReport report;
  std::vector<ExecRequestResult> results;  // trace order
};

// Deterministic synthetic prompt ids: hash(seed, request_id, pos) mod vocab;
// SharedPrefixChat / shared_prefix requests share their first prefix_len ids
// with the other requests of their prefix group (prefix_group()).
std::vector<std::int32_t> synth_prompt(const RequestDescriptor& request, std::uint64_t seed,
                                       int vocab, int prefix_len, int prompt_cap = 0,
                                       int prefix_groups = 1);

// Prefix group of a request: FNV-1a-64(request_id) mod groups (0 for one
// group). The multi-GPU dispatcher pins each group to one GPU with the same
// rule (paper_2605_23057_b200/dispatch.py), so cache hits stay local.
int prefix_group(const std::string& request_id, int groups);

ExecRequestResult execute_request(msw_engine* engine, const RequestDescriptor& request,
                                  const RoutingDecision& decision, const ExecOptions& options);

// Routes every request with `policy`, executes it (continuous-batching
// cohorts = maximal runs of consecutive requests routed to
// INT8PlusContinuousBatching, up to cohort_max), and summarises.
ExecRunResult run_policy(const std::vector<RequestDescriptor>& trace, const RoutingPolicy& policy,
                         msw_engine* engine, const ExecOptions& options);

// The reference's decisions CSV (report.cpp:49-61): header
// "request_id,mode,reason,overhead_ms", one row per request in trace order,
// overhead as %.17g, so its read_decisions_csv (report.cpp:63-81) and any diff
// against its own routing output work on executed B200 runs.
void write_decisions_csv(const std::vector<ExecRequestResult>& results,
                         const std::filesystem::path& path);

// The reference's benchmark quality gate (sim.cpp:265-296) over executed
// requests: collapsed mean quality delta of the benchmark families within
// +-threshold_pp; traces without benchmark traffic pass.
struct ExecQualityGate {
  bool passed = true;
  double collapsed_benchmark_delta_pp = 0.0;
  std::vector<ExecFamilySummary> benchmark_families;
};
ExecQualityGate evaluate_quality_gate(const std::vector<ExecRequestResult>& results,
                                      double threshold_pp = 1.5);

// The reference's comparison.csv (report.cpp:83-111), one row per executed
// policy run, same header and %.17g formatting. oracle_match_rate and
// oracle_capture need the constraint oracle over the reference's profile
// store (evaluation-only) and are written as nan;
// synthesized_cell_usage is 0 (every number is measured).
void write_comparison_csv(const std::vector<ExecRunResult>& runs,
                          const std::filesystem::path& path);

// Per-request results with the reference's SimRequestResult fields (sim.hpp:40-56),
// one CSV row per request in trace order, for the reference's own consumers
// (oracle/_ref/ref_exec_interop rebuilds SimRequestResult from it):
// request_id,mode,reason,overhead_ms,simulated_mode,family,fp16_latency_ms,
// mode_latency_ms,speedup,energy_ratio,memory_ratio,quality_delta_pp,energy_j,
// constraint_violated,used_synthesized_cell,fallback_used
void write_results_csv(const std::vector<ExecRequestResult>& results,
                       const std::filesystem::path& path);

}  // namespace modeswitch
