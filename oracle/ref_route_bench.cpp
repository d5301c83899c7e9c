// Reference routing-cost timer. TEST/BENCH INFRASTRUCTURE ONLY: links the
// reference's own proj/core (oracle/_ref) and times RulePolicy::route with the
// reference's own steady_clock stamp (routing.cpp:186-194), the CPU half of
// the hot path, on the host it runs on.
//
// Usage: ref_route_bench <trace.ndjson> <passes>
// Prints one JSON line: {"decisions": N, "mean_overhead_ms": x, "wall_ms": y}
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "modeswitch/routing.hpp"
#include "modeswitch/trace_io.hpp"

int main(int argc, char** argv) {
  if (argc != 3) {
    std::fprintf(stderr, "usage: %s <trace.ndjson> <passes>\n", argv[0]);
    return 2;
  }
  const auto trace = modeswitch::read_trace(argv[1]);
  const int passes = std::atoi(argv[2]);
  const modeswitch::RulePolicy policy;
  double stamped = 0.0;
  long n = 0;
  int sink = 0;
  const auto t0 = std::chrono::steady_clock::now();
  for (int p = 0; p < passes; ++p) {
    for (const auto& r : trace) {
      const auto d = policy.route(r);
      stamped += d.overhead_ms;
      sink += static_cast<int>(d.mode);
      ++n;
    }
  }
  const double wall =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
          .count();
  std::printf("{\"decisions\": %ld, \"mean_overhead_ms\": %.9g, \"wall_ms\": %.6g, \"sink\": %d}\n",
              n, stamped / double(n), wall, sink);
  return 0;
}
