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
//     (summarize, sim.cpp:149-207); results in trace order.
#pragma once

#include <cstdint>
#include <filesystem>
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
  int max_output_tokens = 0;        // > 0 caps generation (bounded samples)
  int max_prompt_tokens = 0;        // > 0 caps prompt length
  int vocab = 0;                    // engine vocabulary (required)
  int cohort_max = 64;              // continuous-batching cohort size
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
  std::vector<std::int32_t> tokens;
};

struct ExecFamilySummary {
  WorkloadFamily family = WorkloadFamily::SyntheticSS;
  int count = 0;
  double mean_speedup = 0.0;
};

struct ExecReport {
  std::string policy;
  int request_count = 0;
  double mean_speedup = 0.0;
  double aggregate_latency_speedup = 0.0;
  double collapsed_mean_speedup = 0.0;
  double mean_overhead_ms = 0.0;
  int fallback_count = 0;
  std::vector<ExecFamilySummary> per_family;
  long long generated_tokens = 0;
  double mode_time_ms = 0.0;  // sum of mode latencies
};

struct ExecRunResult {
  ExecReport report;
  std::vector<ExecRequestResult> results;  // trace order
};

// Deterministic synthetic prompt ids: hash(seed, request_id, pos) mod vocab;
// SharedPrefixChat / shared_prefix requests share their first prefix_len ids.
std::vector<std::int32_t> synth_prompt(const RequestDescriptor& request, std::uint64_t seed,
                                       int vocab, int prefix_len, int prompt_cap = 0);

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

}  // namespace modeswitch
