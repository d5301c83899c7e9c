// Host controller: domain vocabulary, feature extraction, classifier and the
// seven-rule router. Behaviour restated from the reference
//   domain.cpp:5-133, classifier.cpp:13-136, routing.cpp:9-229
// (bit-exact routing is checked against reference-generated goldens in
// tests/test_host_controller.py and by compiling the reference's
// tests/test_domain.cpp against this library).
#include <chrono>
#include <cmath>

#include "modeswitch/classifier.hpp"
#include "modeswitch/domain.hpp"
#include "modeswitch/routing.hpp"

namespace modeswitch {
namespace {

constexpr std::string_view kFamilyNames[kFamilyCount] = {
    "SyntheticSS",   "SyntheticSL",
    "SyntheticLS",   "SyntheticLL",
    "SharedPrefixChat", "MemoryPressureLongContext",
    "MMLUPro",       "GSM8K",
    "TruthfulQA",    "GPQA",
    "MLU"};

constexpr std::string_view kModeNames[kModeCount] = {
    "fp16",
    "int8",
    "gptq4",
    "awq4",
    "speculative_decoding",
    "prefix_caching",
    "chunked_prefill",
    "continuous_batching",
    "cuda_graphs",
    "kv_cache_compression",
    "gptq_prefix_caching",
    "int8_continuous_batching"};

constexpr int kClassCount = 6;
constexpr std::string_view kClassNames[kClassCount] = {
    "batched",      "shared_prefix", "memory_pressure",
    "prefill_heavy", "decode_heavy", "balanced"};

constexpr std::string_view kReasonNames[kRoutingReasonCount] = {
    "rule1_batched",          "rule2_shared_prefix",
    "rule3_memory_pressure",  "rule4_synthetic_shape",
    "rule5_decode_heavy",     "rule6_choice_benchmark",
    "rule7_default",          "oracle_feasible_fastest",
    "oracle_fallback_fp16",   "static",
    "learned_vote"};

// Benchmark sub-index (MMLUPro=0 .. MLU=4), -1 for non-benchmarks.
int benchmark_index(WorkloadFamily family) {
  const int v = static_cast<int>(family);
  const int first = static_cast<int>(WorkloadFamily::MMLUPro);
  return v >= first ? v - first : -1;
}

template <int N>
std::string_view name_of(const std::string_view (&table)[N], int v,
                         const char* what) {
  if (v < 0 || v >= N) throw DataError(std::string("unknown ") + what + " value");
  return table[v];
}

using SteadyClock = std::chrono::steady_clock;
double ms_since(SteadyClock::time_point t0) {
  return std::chrono::duration<double, std::milli>(SteadyClock::now() - t0)
      .count();
}

}  // namespace

// ---- domain -------------------------------------------------------------

bool is_benchmark_family(WorkloadFamily family) {
  return benchmark_index(family) >= 0;
}

bool is_choice_scored(WorkloadFamily family) {
  return is_benchmark_family(family) && family != WorkloadFamily::GSM8K;
}

bool requires_batching(InferenceMode mode) {
  return mode == InferenceMode::ContinuousBatching ||
         mode == InferenceMode::INT8PlusContinuousBatching;
}

std::string_view to_string(WorkloadFamily family) {
  return name_of(kFamilyNames, static_cast<int>(family), "WorkloadFamily");
}
std::string_view to_string(InferenceMode mode) {
  return name_of(kModeNames, static_cast<int>(mode), "InferenceMode");
}
std::string_view to_string(WorkloadClass cls) {
  return name_of(kClassNames, static_cast<int>(cls), "WorkloadClass");
}

WorkloadFamily family_from_string(std::string_view name) {
  for (int i = 0; i < kFamilyCount; ++i)
    if (kFamilyNames[i] == name) return static_cast<WorkloadFamily>(i);
  throw DataError("unknown workload family: '" + std::string(name) + "'");
}
InferenceMode mode_from_string(std::string_view name) {
  for (int i = 0; i < kModeCount; ++i)
    if (kModeNames[i] == name) return static_cast<InferenceMode>(i);
  throw DataError("unknown inference mode: '" + std::string(name) + "'");
}
WorkloadClass workload_class_from_string(std::string_view name) {
  for (int i = 0; i < kClassCount; ++i)
    if (kClassNames[i] == name) return static_cast<WorkloadClass>(i);
  throw DataError("unknown workload class: '" + std::string(name) + "'");
}

void validate(const RequestDescriptor& r) {
  if (r.request_id.empty()) throw DataError("request_id must be nonempty");
  const std::string who = "request '" + r.request_id + "': ";
  if (r.prompt_tokens < 1) throw DataError(who + "prompt_tokens must be >= 1");
  if (r.expected_output_tokens < 1)
    throw DataError(who + "expected_output_tokens must be >= 1");
  if (r.batch_pressure < 1) throw DataError(who + "batch_pressure must be >= 1");
}

double speedup(double fp16_latency_ms, double mode_latency_ms) {
  // Negated comparisons so NaN is rejected too.
  if (!(fp16_latency_ms > 0.0 && mode_latency_ms > 0.0))
    throw DataError("speedup requires positive latencies");
  return fp16_latency_ms / mode_latency_ms;
}

double ratio_vs_baseline(double mode_value, double fp16_value) {
  if (!(fp16_value > 0.0))
    throw DataError("ratio_vs_baseline requires a positive baseline value");
  if (mode_value < 0.0)
    throw DataError("ratio_vs_baseline requires a nonnegative mode value");
  return mode_value / fp16_value;
}

// ---- classifier ---------------------------------------------------------

std::array<double, kFeatureCount> to_array(const FeatureVector& f) {
  return {double(f.prompt_tokens),     double(f.expected_output_tokens),
          double(f.shared_prefix),     double(f.memory_pressure),
          double(f.batch_pressure),    double(f.workload_tag_code),
          f.output_to_prompt_ratio,    double(f.benchmark_family_code),
          double(f.eval_mode_code)};
}

const std::array<std::string, kFeatureCount>& feature_names() {
  static const std::array<std::string, kFeatureCount> names{
      "prompt_tokens",          "expected_output_tokens", "shared_prefix",
      "memory_pressure",        "batch_pressure",         "workload_tag_code",
      "output_to_prompt_ratio", "benchmark_family_code",  "eval_mode_code"};
  return names;
}

FeatureVector features_from_array(const std::array<double, kFeatureCount>& v) {
  auto as_int = [](double x) { return static_cast<int>(std::llround(x)); };
  FeatureVector f;
  f.prompt_tokens = as_int(v[0]);
  f.expected_output_tokens = as_int(v[1]);
  f.shared_prefix = as_int(v[2]);
  f.memory_pressure = as_int(v[3]);
  f.batch_pressure = as_int(v[4]);
  f.workload_tag_code = as_int(v[5]);
  f.output_to_prompt_ratio = v[6];
  f.benchmark_family_code = as_int(v[7]);
  f.eval_mode_code = as_int(v[8]);
  return f;
}

void validate(const ClassifierConfig& c) {
  if (c.long_prompt_threshold < 1 || c.long_output_threshold < 1 ||
      c.batch_threshold < 1)
    throw ConfigError("classifier thresholds must be >= 1");
  if (!(c.decode_heavy_ratio > 0.0))
    throw ConfigError("decode_heavy_ratio must be > 0");
}

FeatureVector extract_features(const RequestDescriptor& r) {
  FeatureVector f;
  f.prompt_tokens = r.prompt_tokens;
  f.expected_output_tokens = r.expected_output_tokens;
  f.shared_prefix = int(r.shared_prefix);
  f.memory_pressure = int(r.memory_pressure);
  f.batch_pressure = r.batch_pressure;
  f.output_to_prompt_ratio =
      double(r.expected_output_tokens) / double(r.prompt_tokens);
  if (r.workload_tag.has_value()) {
    const WorkloadFamily tag = *r.workload_tag;
    f.workload_tag_code = static_cast<int>(tag);
    f.benchmark_family_code = benchmark_index(tag);
    f.eval_mode_code = is_choice_scored(tag) ? 1 : 0;
  }
  return f;
}

WorkloadClass classify(const FeatureVector& f, const ClassifierConfig& c) {
  validate(c);  // the reference re-validates on every call (classifier.cpp:89)
  if (f.batch_pressure >= c.batch_threshold) return WorkloadClass::Batched;
  if (f.shared_prefix) return WorkloadClass::SharedPrefix;
  if (f.memory_pressure) return WorkloadClass::MemoryPressure;
  const int out = f.expected_output_tokens;
  const bool long_out_ratio =
      out >= c.long_output_threshold &&
      f.output_to_prompt_ratio >= c.decode_heavy_ratio;
  const bool long_out_short_prompt =
      out > c.long_output_threshold && f.prompt_tokens < c.long_prompt_threshold;
  if (long_out_ratio || long_out_short_prompt) return WorkloadClass::DecodeHeavy;
  if (f.prompt_tokens >= c.long_prompt_threshold && out < c.long_output_threshold)
    return WorkloadClass::PrefillHeavy;
  return WorkloadClass::Balanced;
}

WorkloadFamily resolve_family(const RequestDescriptor& r,
                              const ClassifierConfig& c) {
  if (r.workload_tag) return *r.workload_tag;
  if (r.shared_prefix) return WorkloadFamily::SharedPrefixChat;
  if (r.memory_pressure) return WorkloadFamily::MemoryPressureLongContext;
  const bool lp = r.prompt_tokens >= c.long_prompt_threshold;
  const bool lo = r.expected_output_tokens >= c.long_output_threshold;
  static constexpr WorkloadFamily quadrant[2][2] = {
      {WorkloadFamily::SyntheticSS, WorkloadFamily::SyntheticSL},
      {WorkloadFamily::SyntheticLS, WorkloadFamily::SyntheticLL}};
  return quadrant[lp][lo];
}

// ---- routing ------------------------------------------------------------

std::string_view to_string(RoutingReason reason) {
  return name_of(kReasonNames, static_cast<int>(reason), "RoutingReason");
}

RoutingReason routing_reason_from_string(std::string_view name) {
  for (int i = 0; i < kRoutingReasonCount; ++i)
    if (kReasonNames[i] == name) return static_cast<RoutingReason>(i);
  throw DataError("unknown routing reason: '" + std::string(name) + "'");
}

RoutingDecision route_rule(const RequestDescriptor& r, WorkloadClass cls,
                           const ClassifierConfig& /*config*/) {
  const auto t0 = SteadyClock::now();
  using M = InferenceMode;
  using R = RoutingReason;
  using F = WorkloadFamily;
  const bool tagged = r.workload_tag.has_value();
  const F tag = tagged ? *r.workload_tag : F::SyntheticSS;

  RoutingDecision d;
  auto pick = [&d](M m, R why) {
    d.mode = m;
    d.reason = why;
  };
  // Rules are evaluated strictly in order; the first match wins.
  if (cls == WorkloadClass::Batched) {
    pick(M::INT8PlusContinuousBatching, R::Rule1Batched);
  } else if (cls == WorkloadClass::SharedPrefix) {
    pick(M::GPTQPlusPrefixCaching, R::Rule2SharedPrefix);
  } else if (cls == WorkloadClass::MemoryPressure) {
    pick(M::GPTQ4, R::Rule3MemoryPressure);
  } else if (tagged && (tag == F::SyntheticSS || tag == F::SyntheticLS ||
                        tag == F::SyntheticLL)) {
    pick(M::GPTQ4, R::Rule4SyntheticShape);
  } else if (cls == WorkloadClass::DecodeHeavy || (tagged && tag == F::GSM8K)) {
    pick(M::SpeculativeDecoding, R::Rule5DecodeHeavy);
  } else if (tagged && (is_choice_scored(tag) ||
                        (cls == WorkloadClass::PrefillHeavy &&
                         is_benchmark_family(tag)))) {
    pick(M::INT8, R::Rule6ChoiceBenchmark);
  } else {
    pick(M::INT8, R::Rule7Default);
  }
  d.overhead_ms = ms_since(t0);
  return d;
}

void validate(const ConstraintSet& c) {
  if (!(c.energy_ratio_max > 0.0) || !(c.memory_ratio_max > 0.0))
    throw ConfigError("constraint caps must be positive");
}

RoutingDecision route_static(InferenceMode mode) {
  RoutingDecision d;
  d.mode = mode;
  d.reason = RoutingReason::Static;
  d.overhead_ms = 0.0;  // no decision work; keeps the FP16 identity exact
  return d;
}

RulePolicy::RulePolicy(ClassifierConfig config) : config_(config) {
  validate(config_);
}

RoutingDecision RulePolicy::route(const RequestDescriptor& request) const {
  const auto t0 = SteadyClock::now();
  RoutingDecision d =
      route_rule(request, classify(extract_features(request), config_), config_);
  d.overhead_ms = ms_since(t0);  // extraction + classification + rules
  return d;
}

StaticPolicy::StaticPolicy(InferenceMode mode) : mode_(mode) {}

std::string StaticPolicy::name() const {
  return mode_ == InferenceMode::FP16 ? std::string("fp16")
                                      : "static:" + std::string(to_string(mode_));
}

RoutingDecision StaticPolicy::route(const RequestDescriptor&) const {
  return route_static(mode_);
}

}  // namespace modeswitch
