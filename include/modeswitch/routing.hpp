// modeswitch-b200 host controller: routing policies.
//
// Interface kept from reference proj/core/include/modeswitch/routing.hpp:14-129
// (RoutingReason, RoutingDecision, RoutingPolicy, RulePolicy, StaticPolicy).
// The constraint-aware oracle policy needs the reference's profile store and
// is evaluation-only, so it is not part of this drop-in.
#pragma once

#include <string>
#include <string_view>

#include "modeswitch/classifier.hpp"
#include "modeswitch/domain.hpp"

namespace modeswitch {

enum class RoutingReason : int {
  Rule1Batched = 0,
  Rule2SharedPrefix = 1,
  Rule3MemoryPressure = 2,
  Rule4SyntheticShape = 3,
  Rule5DecodeHeavy = 4,
  Rule6ChoiceBenchmark = 5,
  Rule7Default = 6,
  OracleFeasibleFastest = 7,
  OracleFallbackFP16 = 8,
  Static = 9,
  LearnedVote = 10,
};
inline constexpr int kRoutingReasonCount = 11;

std::string_view to_string(RoutingReason reason);
RoutingReason routing_reason_from_string(std::string_view name);

struct RoutingDecision {
  InferenceMode mode = InferenceMode::FP16;
  RoutingReason reason = RoutingReason::Static;
  double overhead_ms = 0.0;  // wall-clock cost of the decision itself
};

// Feasibility envelope (reference routing.hpp:38-47): quality is a one-sided
// floor, energy and memory one-sided caps. The executor checks every executed
// request's measured ratios against it (SimRequestResult::constraint_violated).
struct ConstraintSet {
  double quality_floor_pp = -1.5;
  double energy_ratio_max = 1.0;
  double memory_ratio_max = 1.10;
};

void validate(const ConstraintSet& constraints);

// Seven ordered rules (reference routing.cpp:63-100). Never returns FP16.
RoutingDecision route_rule(const RequestDescriptor& request, WorkloadClass cls,
                           const ClassifierConfig& config);

RoutingDecision route_static(InferenceMode mode);

// Stateless after construction, safe to share across dispatcher threads.
class RoutingPolicy {
 public:
  virtual ~RoutingPolicy() = default;
  virtual std::string name() const = 0;
  virtual RoutingDecision route(const RequestDescriptor& request) const = 0;
};

class RulePolicy final : public RoutingPolicy {
 public:
  explicit RulePolicy(ClassifierConfig config = {});
  std::string name() const override { return "rule"; }
  RoutingDecision route(const RequestDescriptor& request) const override;

 private:
  ClassifierConfig config_;
};

class StaticPolicy final : public RoutingPolicy {
 public:
  explicit StaticPolicy(InferenceMode mode);
  std::string name() const override;
  RoutingDecision route(const RequestDescriptor& request) const override;

 private:
  InferenceMode mode_;
};

}  // namespace modeswitch
