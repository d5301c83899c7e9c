// Power traces and energy per token (include/modeswitch/energy.hpp).
#include "modeswitch/energy.hpp"

#include <dlfcn.h>

#include <chrono>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>

#include "modeswitch/domain.hpp"
#include "msw_engine.h"

namespace modeswitch {

PowerTrace read_power_trace(const std::filesystem::path& path) {
  std::ifstream in(path);
  if (!in) throw DataError("cannot open power trace: " + path.string());
  std::string line;
  if (!std::getline(in, line) || line != "timestamp_ms,power_w")
    throw DataError("power trace " + path.string() + ": expected header 'timestamp_ms,power_w'");
  PowerTrace trace;
  size_t no = 1;
  while (std::getline(in, line)) {
    ++no;
    if (line.empty()) continue;
    const size_t comma = line.find(',');
    if (comma == std::string::npos || comma + 1 >= line.size())
      throw DataError(path.string() + ":" + std::to_string(no) + ": malformed power sample");
    try {
      trace.samples.push_back({std::stod(line.substr(0, comma)), std::stod(line.substr(comma + 1))});
    } catch (const std::exception&) {
      throw DataError(path.string() + ":" + std::to_string(no) + ": non-numeric power sample");
    }
  }
  return trace;
}

void write_power_trace(const PowerTrace& trace, const std::filesystem::path& path) {
  std::ofstream out(path);
  if (!out) throw DataError("cannot write power trace: " + path.string());
  out << "timestamp_ms,power_w\n";
  char buf[96];
  for (const auto& s : trace.samples) {
    std::snprintf(buf, sizeof(buf), "%.17g,%.17g", s.timestamp_ms, s.power_w);
    out << buf << '\n';
  }
}

double energy_from_power_trace(const PowerTrace& trace, int tokens) {
  if (trace.samples.size() < 2) throw DataError("power trace needs at least 2 samples to integrate");
  if (tokens < 1) throw DataError("energy_from_power_trace: tokens must be positive");
  double joules = 0.0;
  for (size_t i = 0; i + 1 < trace.samples.size(); ++i) {
    const auto& a = trace.samples[i];
    const auto& b = trace.samples[i + 1];
    if (!(b.timestamp_ms > a.timestamp_ms))
      throw DataError("power trace timestamps must be strictly increasing");
    if (a.power_w < 0.0 || b.power_w < 0.0) throw DataError("power trace samples must be nonnegative");
    joules += 0.5 * (a.power_w + b.power_w) * (b.timestamp_ms - a.timestamp_ms) / 1000.0;
  }
  return joules / tokens;
}

// ---- NVML, resolved at run time (no link dependency on the driver library)
namespace {
struct NvmlField {  // nvmlFieldValue_t (nvml.h)
  unsigned field_id, scope_id;
  long long timestamp, latency_usec;
  int value_type, nvml_return;
  union {
    double d;
    unsigned ui;
    unsigned long ul;
    unsigned long long ull;
    long long sll;
    int si;
  } value;
};
constexpr unsigned kFieldPowerInstant = 186;  // NVML_FI_DEV_POWER_INSTANT (mW)

struct Nvml {
  using InitFn = int (*)();
  using HandleIdxFn = int (*)(unsigned, void**);
  using HandleBusFn = int (*)(const char*, void**);
  using PowerFn = int (*)(void*, unsigned*);
  using FieldsFn = int (*)(void*, int, NvmlField*);
  using EnergyFn = int (*)(void*, unsigned long long*);
  InitFn init = nullptr;
  HandleIdxFn handle_idx = nullptr;
  HandleBusFn handle_bus = nullptr;
  PowerFn power = nullptr;
  FieldsFn fields = nullptr;
  EnergyFn energy = nullptr;
  bool ok = false;
  Nvml() {
    void* lib = dlopen("libnvidia-ml.so.1", RTLD_LAZY | RTLD_LOCAL);
    if (!lib) lib = dlopen("libnvidia-ml.so", RTLD_LAZY | RTLD_LOCAL);
    if (!lib) return;
    init = reinterpret_cast<InitFn>(dlsym(lib, "nvmlInit_v2"));
    handle_idx = reinterpret_cast<HandleIdxFn>(dlsym(lib, "nvmlDeviceGetHandleByIndex_v2"));
    handle_bus = reinterpret_cast<HandleBusFn>(dlsym(lib, "nvmlDeviceGetHandleByPciBusId_v2"));
    power = reinterpret_cast<PowerFn>(dlsym(lib, "nvmlDeviceGetPowerUsage"));  // 1 s average on Ampere+
    fields = reinterpret_cast<FieldsFn>(dlsym(lib, "nvmlDeviceGetFieldValues"));
    energy = reinterpret_cast<EnergyFn>(dlsym(lib, "nvmlDeviceGetTotalEnergyConsumption"));  // mJ
    ok = init && (handle_bus || handle_idx) && (power || fields) && init() == 0;
  }
};
Nvml& nvml() {
  static Nvml n;
  return n;
}
double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
}  // namespace

PowerSampler::PowerSampler(int device, double period_ms) : device_(device), period_ms_(period_ms) {
  if (!nvml().ok) throw ConfigError("NVML unavailable: cannot sample GPU power");
  // CUDA ordinals and NVML indices differ under CUDA_VISIBLE_DEVICES or a
  // non-PCI enumeration order: resolve the NVML device by the CUDA device's
  // PCI bus id (libmsw_engine.so asks the CUDA runtime).
  char bus[32] = {0};
  int rc = -1;
  if (nvml().handle_bus && msw_device_pci_bus_id(device, bus, int(sizeof(bus))) == 0)
    rc = nvml().handle_bus(bus, &dev_handle_);
  if (rc != 0 && nvml().handle_idx) rc = nvml().handle_idx(unsigned(device), &dev_handle_);
  if (rc != 0) throw ConfigError("NVML: no handle for device " + std::to_string(device));
}

bool PowerSampler::read_energy_mj(unsigned long long* mj) {
  return nvml().energy && nvml().energy(dev_handle_, mj) == 0;
}

double PowerSampler::counter_joules() const {
  return have_energy_ ? double(e1_ - e0_) / 1000.0 : -1.0;
}

PowerSampler::~PowerSampler() {
  if (running_) stop();
}

void PowerSampler::sample_once() {
  // instantaneous board power (NVML_FI_DEV_POWER_INSTANT); the legacy
  // nvmlDeviceGetPowerUsage is a 1 s moving average on Ampere and newer, which
  // would smear the previous request's power into a short window
  double watts = -1.0;
  if (nvml().fields) {
    NvmlField f{};
    f.field_id = kFieldPowerInstant;
    if (nvml().fields(dev_handle_, 1, &f) == 0 && f.nvml_return == 0) {
      double mw = -1.0;  // nvmlValueType_t: 0 double, 1 uint, 2 ulong, 3 ull, 4 sll, 5 int
      switch (f.value_type) {
        case 0: mw = f.value.d; break;
        case 1: mw = double(f.value.ui); break;
        case 2: mw = double(f.value.ul); break;
        case 3: mw = double(f.value.ull); break;
        case 4: mw = double(f.value.sll); break;
        case 5: mw = double(f.value.si); break;
        default: break;
      }
      if (mw >= 0.0) watts = mw / 1000.0;
    }
  }
  if (watts < 0.0 && nvml().power) {
    unsigned mw = 0;
    if (nvml().power(dev_handle_, &mw) == 0) watts = mw / 1000.0;
  }
  if (watts < 0.0) return;
  const double t = now_ms() - t0_;
  std::lock_guard<std::mutex> lk(mu_);
  if (!trace_.samples.empty() && !(t > trace_.samples.back().timestamp_ms)) return;
  trace_.samples.push_back({t, watts});
}

void PowerSampler::start() {
  if (running_) return;
  trace_.samples.clear();
  have_energy_ = read_energy_mj(&e0_);
  t0_ = now_ms();
  sample_once();
  running_ = true;
  thread_ = std::thread([this] {
    while (running_) {
      std::this_thread::sleep_for(std::chrono::duration<double, std::milli>(period_ms_));
      sample_once();
    }
  });
}

PowerTrace PowerSampler::stop() {
  if (running_) {
    running_ = false;
    thread_.join();
  }
  sample_once();
  if (have_energy_) have_energy_ = read_energy_mj(&e1_);
  std::lock_guard<std::mutex> lk(mu_);
  return trace_;
}

}  // namespace modeswitch
