// Golden-fixture generator. TEST INFRASTRUCTURE ONLY: links the reference's
// own proj/core library (compiled from /root/reference by oracle/Makefile
// into oracle/_ref/, never copied) and writes the routing/trace fixtures that
// pin the host controller under tests/golden/.
//
// Usage: ref_golden <out_dir>
// Outputs (all deterministic):
//   balanced_55_seed7.ndjson        reference write_trace(balanced_family_trace(55, 7))
//   <name>.ndjson / <name>.decisions.csv for every trace below; each decision
//   row is request_id,mode,reason,class,family from the reference's
//   RulePolicy::route, classify(extract_features()) and resolve_family.
//   power_<k>.csv + power_golden.csv: power traces written by the reference's
//   write_power_trace and their energy_from_power_trace (J/token, %.17g) or
//   the DataError it raises (sim.cpp:10-78).
#include <cstdio>
#include <fstream>
#include <random>
#include <string>
#include <vector>

#include "modeswitch/classifier.hpp"
#include "modeswitch/routing.hpp"
#include "modeswitch/profile.hpp"
#include "modeswitch/report.hpp"
#include "modeswitch/sim.hpp"
#include "modeswitch/trace_io.hpp"
#include "modeswitch/workload.hpp"

namespace ms = modeswitch;

static void emit(const std::string& dir, const std::string& name,
                 const std::vector<ms::RequestDescriptor>& trace) {
  ms::write_trace(trace, dir + "/" + name + ".ndjson");
  std::ofstream out(dir + "/" + name + ".decisions.csv");
  out << "request_id,mode,reason,class,family\n";
  const ms::RulePolicy policy;
  const ms::ClassifierConfig cfg;
  for (const auto& r : trace) {
    const auto d = policy.route(r);
    out << r.request_id << ',' << ms::to_string(d.mode) << ','
        << ms::to_string(d.reason) << ','
        << ms::to_string(ms::classify(ms::extract_features(r), cfg)) << ','
        << ms::to_string(ms::resolve_family(r, cfg)) << '\n';
  }
}

int main(int argc, char** argv) {
  if (argc == 3 && std::string(argv[1]) == "--check-decisions") {
    // the reference's own read_decisions_csv (report.cpp:63-81) on a CSV written by this repo
    try {
      for (const auto& r : ms::read_decisions_csv(argv[2]))
        std::printf("%s,%s,%s\n", r.request_id.c_str(), std::string(ms::to_string(r.mode)).c_str(),
                    std::string(ms::to_string(r.reason)).c_str());
      return 0;
    } catch (const std::exception& e) {
      std::printf("error %s\n", e.what());
      return 3;
    }
  }
  if (argc == 3 && std::string(argv[1]) == "--check-profile") {
    // the reference's own loader + validate() on a profile written by this repo
    try {
      const ms::ProfileTable t = ms::load_profile(argv[2]);
      std::printf("ok %zu families\n", t.families().size());
      return 0;
    } catch (const std::exception& e) {
      std::printf("error %s\n", e.what());
      return 3;
    }
  }
  if (argc != 2) {
    std::fprintf(stderr, "usage: %s <out_dir>\n", argv[0]);
    return 2;
  }
  const std::string dir = argv[1];

  // (1) SURVEY §8c golden: balanced_family_trace(55, seed 7), 605 lines.
  emit(dir, "balanced_55_seed7", ms::balanced_family_trace(55, 7));

  // (2) canonical families, zero jitter, unbatched and batch_pressure 4
  //     (SPEC acceptance criterion 4).
  {
    ms::TraceSpec spec;
    spec.jitter = 0.0;
    spec.batched_fraction = 0.5;
    spec.batch_pressure = 4;
    for (auto f : ms::all_families()) spec.counts[f] = 2;
    emit(dir, "canonical_families", ms::generate_trace(spec));
  }

  // (3) BASELINE config 1 workload: 5 per family, jitter 0.10, seed 7,
  //     batched_fraction 0.2, batch_pressure 4.
  {
    ms::TraceSpec spec;
    spec.seed = 7;
    spec.batched_fraction = 0.2;
    for (auto f : ms::all_families()) spec.counts[f] = 5;
    emit(dir, "config1_mixed", ms::generate_trace(spec));
  }

  // (4) BASELINE config 5 deployment-mix families, tagged and untagged.
  //     (the 8K variant is derived from the MemoryPressure rows by the host
  //     code; routing does not depend on prompt length for memory_pressure.)
  {
    ms::TraceSpec spec;
    spec.seed = 7;
    spec.counts[ms::WorkloadFamily::SyntheticSS] = 64;
    spec.counts[ms::WorkloadFamily::SyntheticSL] = 32;
    spec.counts[ms::WorkloadFamily::GSM8K] = 32;
    spec.counts[ms::WorkloadFamily::SharedPrefixChat] = 64;
    spec.counts[ms::WorkloadFamily::MemoryPressureLongContext] = 64;
    auto trace = ms::generate_trace(spec);
    emit(dir, "deploy_mix_tagged", trace);
    for (auto& r : trace) r.workload_tag.reset();
    emit(dir, "deploy_mix_untagged", trace);
  }

  // (5) boundary fuzz: random descriptors concentrated around the classifier
  //     thresholds (prompt 512, output 64, ratio 0.5, batch 2).
  {
    std::mt19937_64 rng(2605);
    auto pick = [&rng](std::initializer_list<int> v) {
      return *(v.begin() + rng() % v.size());
    };
    std::vector<ms::RequestDescriptor> trace;
    for (int i = 0; i < 3000; ++i) {
      ms::RequestDescriptor r;
      r.request_id = "fuzz-" + std::to_string(i);
      const int mode = int(rng() % 3);
      if (mode == 0) {
        r.prompt_tokens = pick({1, 2, 63, 64, 65, 127, 128, 255, 256, 257, 511,
                                512, 513, 1024, 2048, 8192});
        r.expected_output_tokens =
            pick({1, 16, 31, 32, 63, 64, 65, 128, 255, 256, 257, 512, 1024});
      } else if (mode == 1) {
        // ratio exactly 0.5 and its neighbours
        const int out = 64 + int(rng() % 200);
        r.expected_output_tokens = out;
        r.prompt_tokens = 2 * out + int(rng() % 3) - 1;
      } else {
        r.prompt_tokens = 1 + int(rng() % 9000);
        r.expected_output_tokens = 1 + int(rng() % 1100);
      }
      r.shared_prefix = (rng() % 5) == 0;
      r.memory_pressure = (rng() % 5) == 0;
      r.batch_pressure = pick({1, 1, 1, 1, 2, 3, 4, 64});
      if (rng() % 3 != 0) r.workload_tag = ms::all_families()[rng() % 11];
      trace.push_back(r);
    }
    emit(dir, "boundary_fuzz", trace);
  }
    // (power) energy per token over deterministic traces, incl. error cases
  {
    std::ofstream g(dir + "/power_golden.csv");
    g << "name,tokens,joules_per_token\n";
    std::mt19937_64 rng(20260517);
    std::uniform_real_distribution<double> watts(120.0, 1000.0), step(5.0, 80.0);
    const int lens[] = {2, 3, 17, 200};
    const int toks[] = {1, 7, 128, 1000};
    for (int k = 0; k < 6; ++k) {
      ms::PowerTrace tr;
      const int n = k < 4 ? lens[k] : 12;
      double t = 1000.0 * k;
      for (int i = 0; i < n; ++i) {
        tr.samples.push_back({t, watts(rng)});
        t += step(rng);
      }
      if (k == 4) tr.samples[5].timestamp_ms = tr.samples[4].timestamp_ms;  // not increasing
      if (k == 5) tr.samples[3].power_w = -1.0;                             // negative power
      const std::string name = "power_" + std::to_string(k);
      ms::write_power_trace(tr, dir + "/" + name + ".csv");
      const int tokens = toks[k % 4];
      char buf[64];
      try {
        std::snprintf(buf, sizeof(buf), "%.17g",
                      ms::energy_from_power_trace(ms::read_power_trace(dir + "/" + name + ".csv"), tokens));
        g << name << ',' << tokens << ',' << buf << '\n';
      } catch (const ms::DataError&) {
        g << name << ',' << tokens << ",DataError\n";
      }
    }
  }
  return 0;
}
