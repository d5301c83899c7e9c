// modeswitch-b200 host controller: request vocabulary.
//
// Drop-in re-implementation of the reference's domain layer
// (reference: proj/core/include/modeswitch/domain.hpp:10-180,
//  proj/core/src/domain.cpp:5-133). Names, enum values and the error
// hierarchy are kept identical so reference callers (and the reference's own
// tests/test_domain.cpp) compile unchanged against this header.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>

namespace modeswitch {

// ConfigError -> exit code 2, DataError -> exit code 3 (reference
// tools/modeswitch.cpp:26-30). The C ABI mirrors these as return codes.
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ConfigError : public Error {
 public:
  using Error::Error;
};
class DataError : public Error {
 public:
  using Error::Error;
};

// Closed enumerations. Integer values are part of the ABI (msw_request.mode
// is static_cast<int>(InferenceMode)).
enum class WorkloadFamily : int {
  SyntheticSS = 0,
  SyntheticSL = 1,
  SyntheticLS = 2,
  SyntheticLL = 3,
  SharedPrefixChat = 4,
  MemoryPressureLongContext = 5,
  MMLUPro = 6,
  GSM8K = 7,
  TruthfulQA = 8,
  GPQA = 9,
  MLU = 10,
};
inline constexpr int kFamilyCount = 11;

enum class InferenceMode : int {
  FP16 = 0,
  INT8 = 1,
  GPTQ4 = 2,
  AWQ4 = 3,
  SpeculativeDecoding = 4,
  PrefixCaching = 5,
  ChunkedPrefill = 6,
  ContinuousBatching = 7,
  CudaGraphs = 8,
  KVCacheCompression = 9,
  GPTQPlusPrefixCaching = 10,
  INT8PlusContinuousBatching = 11,
};
inline constexpr int kModeCount = 12;

enum class WorkloadClass : int {
  Batched = 0,
  SharedPrefix = 1,
  MemoryPressure = 2,
  PrefillHeavy = 3,
  DecodeHeavy = 4,
  Balanced = 5,
};

constexpr std::array<WorkloadFamily, kFamilyCount> all_families() {
  std::array<WorkloadFamily, kFamilyCount> out{};
  for (int i = 0; i < kFamilyCount; ++i) out[i] = static_cast<WorkloadFamily>(i);
  return out;
}

constexpr std::array<InferenceMode, kModeCount> all_modes() {
  std::array<InferenceMode, kModeCount> out{};
  for (int i = 0; i < kModeCount; ++i) out[i] = static_cast<InferenceMode>(i);
  return out;
}

// The controller's candidate set (reference domain.hpp:103-112), in the
// reference's listed order.
constexpr std::array<InferenceMode, 6> controller_candidates() {
  return {InferenceMode::GPTQ4, InferenceMode::SpeculativeDecoding,
          InferenceMode::GPTQPlusPrefixCaching,
          InferenceMode::INT8PlusContinuousBatching, InferenceMode::INT8,
          InferenceMode::FP16};
}

// Five-class label space, fixed tie-break order (reference domain.hpp:116-120).
constexpr std::array<InferenceMode, 5> oracle_classes() {
  return {InferenceMode::FP16, InferenceMode::INT8, InferenceMode::GPTQ4,
          InferenceMode::SpeculativeDecoding,
          InferenceMode::GPTQPlusPrefixCaching};
}

bool is_benchmark_family(WorkloadFamily family);
bool is_choice_scored(WorkloadFamily family);
bool requires_batching(InferenceMode mode);

std::string_view to_string(WorkloadFamily family);
std::string_view to_string(InferenceMode mode);
std::string_view to_string(WorkloadClass cls);

WorkloadFamily family_from_string(std::string_view name);
InferenceMode mode_from_string(std::string_view name);
WorkloadClass workload_class_from_string(std::string_view name);

// One routable request. Token counts only; token ids are synthesised by the
// executor (see executor.hpp).
struct RequestDescriptor {
  std::string request_id;
  int prompt_tokens = 1;
  int expected_output_tokens = 1;
  bool shared_prefix = false;
  bool memory_pressure = false;
  int batch_pressure = 1;
  std::optional<WorkloadFamily> workload_tag;
};

void validate(const RequestDescriptor& request);

struct RequestMetrics {
  double latency_ms = 0.0;
  double energy_per_token_j = 0.0;
  double throughput_tps = 0.0;
  double memory_ratio = 1.0;
  double quality_delta_pp = 0.0;
  double routing_overhead_ms = 0.0;
};

double speedup(double fp16_latency_ms, double mode_latency_ms);
double ratio_vs_baseline(double mode_value, double fp16_value);

}  // namespace modeswitch
