// Host controller: synthetic trace generation and the NDJSON trace format.
// Restated from reference workload.cpp:9-106 (RNG draw order is load-bearing:
// families in enum order, prompt draw then output draw, unit = (rng()>>11)*2^-53,
// no draw at zero jitter) and trace_io.cpp:12-134 (strict 7-key schema).
#include <algorithm>
#include <cmath>
#include <fstream>
#include <random>
#include <unordered_set>

#include <json.hpp>

#include "modeswitch/trace_io.hpp"
#include "modeswitch/workload.hpp"

namespace modeswitch {

// ---- workload -----------------------------------------------------------

FamilyShape family_nominal_shape(WorkloadFamily family) {
  // {prompt, output, shared_prefix, memory_pressure}, indexed by enum value.
  static constexpr FamilyShape kShapes[kFamilyCount] = {
      {128, 32, false, false},   {128, 128, false, false},
      {1024, 32, false, false},  {1024, 128, false, false},
      {1024, 128, true, false},  {2048, 64, false, true},
      {400, 16, false, false},   {250, 256, false, false},
      {200, 64, false, false},   {500, 16, false, false},
      {300, 16, false, false}};
  const int v = static_cast<int>(family);
  if (v < 0 || v >= kFamilyCount) throw DataError("unknown WorkloadFamily value");
  return kShapes[v];
}

void validate(const TraceSpec& spec) {
  if (!(spec.jitter >= 0.0 && spec.jitter < 0.5))
    throw ConfigError("trace jitter must be in [0, 0.5)");
  for (const auto& kv : spec.counts)
    if (kv.second < 0) throw ConfigError("trace counts must be nonnegative");
  if (spec.batch_pressure < 1) throw ConfigError("batch_pressure must be >= 1");
  if (!(spec.batched_fraction >= 0.0 && spec.batched_fraction <= 1.0))
    throw ConfigError("batched_fraction must be in [0, 1]");
}

namespace {

class Jitter {
 public:
  Jitter(std::uint64_t seed, double j) : rng_(seed), j_(j) {}
  int operator()(int nominal) {
    if (j_ == 0.0) return nominal;  // no RNG draw at zero jitter
    const double u = double(rng_() >> 11) * 0x1.0p-53;
    const double f = (1.0 - j_) + (2.0 * j_) * u;
    return std::max(1, int(std::llround(nominal * f)));
  }

 private:
  std::mt19937_64 rng_;
  double j_;
};

}  // namespace

std::vector<RequestDescriptor> generate_trace(const TraceSpec& spec) {
  validate(spec);
  Jitter jitter(spec.seed, spec.jitter);
  std::vector<RequestDescriptor> out;
  for (WorkloadFamily fam : all_families()) {
    const auto it = spec.counts.find(fam);
    const int n = it == spec.counts.end() ? 0 : it->second;
    if (n == 0) continue;
    const FamilyShape shape = family_nominal_shape(fam);
    const int n_batched = int(std::llround(spec.batched_fraction * n));
    const std::string prefix = std::string(to_string(fam)) + "-";
    for (int i = 0; i < n; ++i) {
      RequestDescriptor r;
      r.request_id = prefix + std::to_string(i);
      r.prompt_tokens = jitter(shape.prompt_tokens);
      r.expected_output_tokens = jitter(shape.output_tokens);
      r.shared_prefix = shape.shared_prefix;
      r.memory_pressure = shape.memory_pressure;
      r.batch_pressure = (i < n_batched) ? spec.batch_pressure : 1;
      r.workload_tag = fam;
      validate(r);
      out.push_back(std::move(r));
    }
  }
  return out;
}

std::vector<RequestDescriptor> balanced_family_trace(int n_per_family,
                                                     std::uint64_t seed,
                                                     double jitter) {
  if (n_per_family < 1)
    throw ConfigError("balanced_family_trace needs n_per_family >= 1");
  TraceSpec spec;
  spec.seed = seed;
  spec.jitter = jitter;
  for (WorkloadFamily fam : all_families()) spec.counts[fam] = n_per_family;
  return generate_trace(spec);
}

// ---- trace I/O ------------------------------------------------------------

namespace {

using json = nlohmann::json;

bool is_trace_key(const std::string& k) {
  static const std::unordered_set<std::string> keys{
      "request_id",      "prompt_tokens",   "expected_output_tokens",
      "shared_prefix",   "memory_pressure", "batch_pressure",
      "workload_tag"};
  return keys.count(k) != 0;
}

int int_field(const json& o, const char* key) {
  const auto it = o.find(key);
  if (it == o.end() || !it->is_number_integer())
    throw DataError(std::string("trace field '") + key +
                    "' missing or not an integer");
  return it->get<int>();
}

bool bool_field(const json& o, const char* key) {
  const auto it = o.find(key);
  if (it == o.end() || !it->is_boolean())
    throw DataError(std::string("trace field '") + key +
                    "' missing or not a boolean");
  return it->get<bool>();
}

}  // namespace

RequestDescriptor parse_trace_line(const std::string& line) {
  json o;
  try {
    o = json::parse(line);
  } catch (const json::exception& e) {
    throw DataError(std::string("invalid trace JSON: ") + e.what());
  }
  if (!o.is_object()) throw DataError("trace line is not a JSON object");
  for (auto it = o.begin(); it != o.end(); ++it)
    if (!is_trace_key(it.key()))
      throw DataError("unknown trace field '" + it.key() + "'");

  RequestDescriptor r;
  const auto id = o.find("request_id");
  if (id == o.end() || !id->is_string())
    throw DataError("trace field 'request_id' missing or not a string");
  r.request_id = id->get<std::string>();
  r.prompt_tokens = int_field(o, "prompt_tokens");
  r.expected_output_tokens = int_field(o, "expected_output_tokens");
  r.shared_prefix = bool_field(o, "shared_prefix");
  r.memory_pressure = bool_field(o, "memory_pressure");
  r.batch_pressure = int_field(o, "batch_pressure");
  const auto tag = o.find("workload_tag");
  if (tag == o.end()) throw DataError("trace field 'workload_tag' missing");
  if (tag->is_string()) {
    r.workload_tag = family_from_string(tag->get<std::string>());
  } else if (!tag->is_null()) {
    throw DataError("trace field 'workload_tag' must be a string or null");
  }
  validate(r);
  return r;
}

std::string format_trace_line(const RequestDescriptor& r) {
  nlohmann::ordered_json o;  // key order is the canonical wire order
  o["request_id"] = r.request_id;
  o["prompt_tokens"] = r.prompt_tokens;
  o["expected_output_tokens"] = r.expected_output_tokens;
  o["shared_prefix"] = r.shared_prefix;
  o["memory_pressure"] = r.memory_pressure;
  o["batch_pressure"] = r.batch_pressure;
  if (r.workload_tag)
    o["workload_tag"] = std::string(to_string(*r.workload_tag));
  else
    o["workload_tag"] = nullptr;
  return o.dump();
}

std::vector<RequestDescriptor> read_trace(const std::filesystem::path& path) {
  std::ifstream in(path);
  if (!in) throw DataError("cannot open trace file: " + path.string());
  std::vector<RequestDescriptor> out;
  std::unordered_set<std::string> ids;
  std::string line;
  for (size_t lineno = 1; std::getline(in, line); ++lineno) {
    if (line.empty()) continue;
    const std::string where = path.string() + ":" + std::to_string(lineno) + ": ";
    RequestDescriptor r;
    try {
      r = parse_trace_line(line);
    } catch (const DataError& e) {
      throw DataError(where + e.what());
    }
    if (!ids.insert(r.request_id).second)
      throw DataError(where + "duplicate request_id '" + r.request_id + "'");
    out.push_back(std::move(r));
  }
  return out;
}

void write_trace(const std::vector<RequestDescriptor>& trace,
                 const std::filesystem::path& path) {
  std::ofstream out(path);
  if (!out) throw DataError("cannot write trace file: " + path.string());
  for (const auto& r : trace) out << format_trace_line(r) << '\n';
  if (!out) throw DataError("failed while writing trace file: " + path.string());
}

}  // namespace modeswitch
