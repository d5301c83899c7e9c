// modeswitch-b200 host: GPU power traces and energy per token.
//
// Same types, names and semantics as the reference's power-trace API
// (sim.hpp:14-31, sim.cpp:10-78): a CSV with header "timestamp_ms,power_w",
// strictly increasing timestamps, nonnegative power, and energy per token by
// trapezoidal integration divided by the generated tokens, with the same
// DataError conditions. The reference only reads traces recorded elsewhere;
// here PowerSampler records them on the B200 (NVML power polling in a host
// thread, libnvidia-ml loaded at run time) around the executed requests, which
// is the paper's second headline metric (J/token, energy ratio vs FP16).
#pragma once

#include <atomic>
#include <filesystem>
#include <mutex>
#include <thread>
#include <vector>

namespace modeswitch {

struct PowerTrace {
  struct Sample {
    double timestamp_ms = 0.0;
    double power_w = 0.0;
  };
  std::vector<Sample> samples;
};

PowerTrace read_power_trace(const std::filesystem::path& path);
void write_power_trace(const PowerTrace& trace, const std::filesystem::path& path);
// Joules per token: sum of 0.5 (p_i + p_i+1) (t_i+1 - t_i) / 1000 over
// consecutive samples, divided by tokens (reference sim.cpp:57-78).
double energy_from_power_trace(const PowerTrace& trace, int tokens);

// Samples the instantaneous board power of CUDA device `device` (NVML device
// resolved by PCI bus id; NVML_FI_DEV_POWER_INSTANT, falling back to
// nvmlDeviceGetPowerUsage) every period_ms into a PowerTrace (timestamps:
// steady clock, ms since start()), and reads the driver's total-energy
// counter at start() and stop(). Throws ConfigError when NVML is unavailable.
class PowerSampler {
 public:
  explicit PowerSampler(int device, double period_ms = 10.0);
  ~PowerSampler();
  void start();
  PowerTrace stop();  // always appends one final sample so short windows integrate
  // Joules between start() and stop() from nvmlDeviceGetTotalEnergyConsumption
  // (the driver's integrated counter); -1 when the device does not expose it.
  double counter_joules() const;

 private:
  void sample_once();
  bool read_energy_mj(unsigned long long* mj);
  bool have_energy_ = false;
  unsigned long long e0_ = 0, e1_ = 0;
  int device_;
  double period_ms_;
  void* dev_handle_ = nullptr;
  std::thread thread_;
  std::atomic<bool> running_{false};
  std::mutex mu_;
  PowerTrace trace_;
  double t0_ = 0.0;
};

}  // namespace modeswitch
