// Executor -> reference interop checker. TEST INFRASTRUCTURE ONLY: links the
// reference's own proj/core library (compiled from /root/reference by
// oracle/Makefile into oracle/_ref/, never copied).
//
// Usage: ref_exec_interop <results.csv> <comparison.csv> <out_dir>
//   results.csv    the B200 executor's per-request SimRequestResult fields
//                  (modeswitch::write_results_csv, executor.hpp)
//   comparison.csv the executor's comparison.csv (write_comparison_csv)
// Rebuilds the reference's SimRequestResult for every executed request from
// results.csv (read with the reference's read_csv) and feeds them to the
// reference's own consumers:
//   * evaluate_quality_gate (sim.cpp:265-296) -> printed as JSON;
//   * write_decisions_csv (report.cpp:49-61) -> <out_dir>/decisions.csv, read
//     back with read_decisions_csv (row count printed);
//   * comparison.csv parsed with read_csv, its report scalars placed in a
//     reference PolicyComparison and re-emitted with the reference's
//     write_comparison_csv -> <out_dir>/comparison.csv (byte-compared by the
//     test against the executor's file).
#include <cstdio>
#include <limits>
#include <string>
#include <vector>

#include "modeswitch/report.hpp"
#include "modeswitch/sim.hpp"

namespace ms = modeswitch;

int main(int argc, char** argv) {
  if (argc != 4) {
    std::fprintf(stderr, "usage: %s results.csv comparison.csv out_dir\n", argv[0]);
    return 2;
  }
  try {
    const ms::CsvTable t = ms::read_csv(argv[1]);
    auto col = [&](const char* name) {
      for (size_t i = 0; i < t.header.size(); ++i)
        if (t.header[i] == name) return i;
      throw ms::DataError(std::string("results.csv: missing column ") + name);
    };
    std::vector<ms::SimRequestResult> results;
    for (const auto& row : t.rows) {
      ms::SimRequestResult r;
      r.request_id = row[col("request_id")];
      r.decision.mode = ms::mode_from_string(row[col("mode")]);
      r.decision.reason = ms::routing_reason_from_string(row[col("reason")]);
      r.decision.overhead_ms = std::stod(row[col("overhead_ms")]);
      r.simulated_mode = ms::mode_from_string(row[col("simulated_mode")]);
      r.family = ms::family_from_string(row[col("family")]);
      r.fp16_latency_ms = std::stod(row[col("fp16_latency_ms")]);
      r.mode_latency_ms = std::stod(row[col("mode_latency_ms")]);
      r.speedup = std::stod(row[col("speedup")]);
      r.energy_ratio = std::stod(row[col("energy_ratio")]);
      r.memory_ratio = std::stod(row[col("memory_ratio")]);
      r.quality_delta_pp = std::stod(row[col("quality_delta_pp")]);
      r.energy_j = std::stod(row[col("energy_j")]);
      r.overhead_ms = r.decision.overhead_ms;
      r.constraint_violated = row[col("constraint_violated")] == "1";
      r.used_synthesized_cell = row[col("used_synthesized_cell")] == "1";
      r.fallback_used = row[col("fallback_used")] == "1";
      results.push_back(r);
    }
    const ms::QualityGateResult gate = ms::evaluate_quality_gate(results);
    const std::string dir = argv[3];
    ms::write_decisions_csv(results, dir + "/decisions.csv");
    const auto records = ms::read_decisions_csv(dir + "/decisions.csv");

    const ms::CsvTable c = ms::read_csv(argv[2]);
    ms::PolicyComparison cmp;
    for (const auto& row : c.rows) {
      auto f = [&](size_t i) { return std::stod(row[i]); };
      ms::PolicyRunResult run;
      ms::PolicyReport& p = run.report;
      p.policy = row[0];
      p.request_count = std::stoi(row[1]);
      p.mean_speedup = f(2);
      p.mean_energy_ratio = f(3);
      p.mean_memory_ratio = f(4);
      p.mean_quality_delta_pp = f(5);
      p.collapsed_mean_speedup = f(6);
      p.collapsed_mean_energy_ratio = f(7);
      p.aggregate_latency_speedup = f(8);
      p.oracle_match_rate = f(9);
      p.constraint_violation_rate = f(10);
      p.mean_overhead_ms = f(11);
      p.synthesized_cell_usage = f(12);
      p.fallback_count = std::stoi(row[13]);
      cmp.runs.push_back(run);
      cmp.oracle_capture.push_back(f(14));
    }
    ms::write_comparison_csv(cmp, dir + "/comparison.csv");
    std::printf("{\"requests\": %zu, \"gate_passed\": %d, \"collapsed_benchmark_delta_pp\": %s, "
                "\"benchmark_families\": %zu, \"decisions_read_back\": %zu}\n",
                results.size(), gate.passed ? 1 : 0,
                ms::format_double(gate.collapsed_benchmark_delta_pp).c_str(),
                gate.benchmark_families.size(), records.size());
  } catch (const std::exception& ex) {
    std::fprintf(stderr, "error: %s\n", ex.what());
    return 3;
  }
  return 0;
}
