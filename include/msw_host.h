/* modeswitch-b200: C ABI of the host controller (libmodeswitch.so).
 *
 * Flat C entry points over the C++ controller (include/modeswitch/*.hpp) so
 * non-C++ callers (ctypes, cgo, JNI) bind it without C++ name mangling. Each
 * one replaces a reference call site:
 *   msw_route_rule        <- RulePolicy::route          (routing.cpp:186-194)
 *                            + classify/extract_features (classifier.cpp:69-113)
 *                            + resolve_family            (classifier.cpp:115-136)
 *   msw_trace_parse_line  <- parse_trace_line           (trace_io.cpp:34-76)
 *   msw_trace_format_line <- format_trace_line          (trace_io.cpp:78-92)
 *   msw_trace_generate    <- generate_trace             (workload.cpp:61-91)
 *   msw_route_cost        <- the per-decision overhead stamp (routing.cpp:188-192)
 *   msw_execute_trace     <- run_policy + simulate_request + summarize
 *                            (sim.cpp:80-235): route, EXECUTE on the B200
 *                            engine (include/msw_engine.h), aggregate
 *
 * Return codes mirror the reference CLI's exit codes (tools/modeswitch.cpp:26-30):
 *   0 ok, 2 ConfigError, 3 DataError, 1 anything else. Message via
 *   msw_host_last_error() (thread-local). No exception crosses this ABI.
 */
#ifndef MSW_HOST_H_
#define MSW_HOST_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSW_OK 0
#define MSW_ERR_OTHER 1
#define MSW_ERR_CONFIG 2
#define MSW_ERR_DATA 3

typedef struct msw_descriptor {
  const char* request_id; /* nonempty, NUL-terminated */
  int32_t prompt_tokens;
  int32_t expected_output_tokens;
  int32_t shared_prefix;   /* 0/1 */
  int32_t memory_pressure; /* 0/1 */
  int32_t batch_pressure;
  int32_t workload_tag; /* WorkloadFamily value, -1 = untagged */
} msw_descriptor;

typedef struct msw_classifier_cfg {
  int32_t long_prompt_threshold; /* 512 */
  int32_t long_output_threshold; /* 64 */
  double decode_heavy_ratio;     /* 0.5 */
  int32_t batch_threshold;       /* 2 */
} msw_classifier_cfg;

typedef struct msw_route_out {
  int32_t mode;   /* InferenceMode value */
  int32_t reason; /* RoutingReason value */
  int32_t workload_class;
  int32_t family; /* resolve_family */
  double overhead_ms;
} msw_route_out;

/* cfg may be NULL for the reference defaults. */
int msw_route_rule(const msw_descriptor* d, const msw_classifier_cfg* cfg,
                   msw_route_out* out);

/* Routes every line of an NDJSON trace held in memory; out arrays sized n_max.
 * *n_out receives the request count. ids_out (optional) receives the request
 * ids, NUL-separated, into a caller buffer of ids_cap bytes. */
int msw_route_ndjson(const char* ndjson, const msw_classifier_cfg* cfg,
                     int32_t n_max, msw_route_out* out, int32_t* n_out);

/* Parses one trace line. The id is copied into id_buf (cap bytes). */
int msw_trace_parse_line(const char* line, msw_descriptor* out, char* id_buf,
                         size_t id_cap);

/* Canonical single-line JSON; *needed = bytes incl. NUL. */
int msw_trace_format_line(const msw_descriptor* d, char* buf, size_t cap,
                          size_t* needed);

/* generate_trace(): counts[11] per family in enum order. Writes NDJSON
 * (newline-terminated lines) into buf; *needed = bytes incl. NUL. */
int msw_trace_generate(const int32_t counts[11], double jitter, uint64_t seed,
                       int32_t batch_pressure, double batched_fraction,
                       char* buf, size_t cap, size_t* needed);

/* Routes the trace `passes` times with RulePolicy and returns the mean of the
 * policy's own overhead stamps and the wall time per decision (ms). */
int msw_route_cost(const char* ndjson, int32_t passes, double* mean_stamp_ms,
                   double* wall_ms_per_decision);

/* ---- executor (include/modeswitch/executor.hpp) ---- */
struct msw_engine;

typedef struct msw_exec_opts {
  int32_t fallback_enabled;  /* FP16 emergency fallback (sim.cpp:112-124) */
  int32_t zero_overhead;
  double extra_overhead_ms;
  int32_t measure_fp16_baseline;
  uint64_t token_seed;
  int32_t prefix_len;        /* shared-prefix tokens, e.g. 768 */
  int32_t max_output_tokens; /* > 0 caps generation */
  int32_t max_prompt_tokens; /* > 0 caps prompts */
  int32_t cohort_max;        /* continuous-batching cohort size (64) */
  /* reference ConstraintSet (routing.hpp:41-45): violation accounting */
  double quality_floor_pp;   /* -1.5 */
  double energy_ratio_max;   /* 1.0 */
  double memory_ratio_max;   /* 1.10 */
  int32_t power_device;      /* >= 0: measure energy per request on this CUDA device */
  const double* quality_delta_pp; /* [12] per InferenceMode value, or NULL (all 0) */
  const char* results_csv;    /* optional: per-request SimRequestResult fields */
  const char* comparison_csv; /* optional: the reference's comparison.csv (report.cpp:83-111) */
  int32_t prefix_groups;      /* shared-prefix groups (<= 1: one group) */
} msw_exec_opts;

typedef struct msw_exec_row {
  int32_t mode;          /* routed InferenceMode */
  int32_t reason;        /* RoutingReason */
  int32_t executed_mode; /* FP16 when the fallback hit */
  int32_t family;
  int32_t prompt_tokens;
  int32_t output_tokens;
  int32_t fallback_used;
  int32_t spec_proposed;
  int32_t spec_accepted;
  int32_t prefix_hit_tokens;
  double fp16_latency_ms;
  double mode_latency_ms;
  double speedup;
  double overhead_ms;
  double prefill_ms;
  double decode_ms;
  /* reference SimRequestResult (sim.hpp:48-53), measured */
  double energy_j;       /* -1 when energy is not measured */
  double energy_ratio;
  double memory_ratio;
  double quality_delta_pp;
  int32_t constraint_violated;
} msw_exec_row;

typedef struct msw_exec_summary {
  int32_t request_count;
  int32_t fallback_count;
  double mean_speedup;
  double aggregate_latency_speedup;
  double collapsed_mean_speedup;
  double mean_overhead_ms;
  double mode_time_ms;
  int64_t generated_tokens;
  double mean_energy_ratio;
  double mean_memory_ratio;
  double mean_quality_delta_pp;
  double collapsed_mean_energy_ratio;
  double constraint_violation_rate;
  int32_t quality_gate_passed;          /* evaluate_quality_gate (sim.cpp:265-296), 1.5 pp */
  double collapsed_benchmark_delta_pp;
} msw_exec_summary;

/* Routes (RulePolicy, cfg NULL = defaults) and executes every request of an
 * NDJSON trace on the engine; rows in trace order. */
int msw_execute_trace(struct msw_engine* engine, int32_t vocab, const char* ndjson,
                      const msw_classifier_cfg* cfg, const msw_exec_opts* opts, int32_t n_max,
                      msw_exec_row* rows, int32_t* n_out, msw_exec_summary* summary);

/* The reference's decisions CSV (report.cpp:49-61) for executed rows: request
 * ids from `ndjson` (trace order), mode / reason / overhead_ms from rows[0..n). */
int msw_write_decisions_csv(const char* ndjson, const msw_exec_row* rows, int32_t n,
                            const char* path);

/* Energy (include/modeswitch/energy.hpp; reference sim.hpp:14-31, sim.cpp:10-78).
 * msw_power_start: NVML instantaneous-power polling of CUDA device `device`
 * (NVML handle resolved by PCI bus id) every period_ms in a host thread.
 * msw_power_stop: stops, optionally writes the trace as the reference's
 * "timestamp_ms,power_w" CSV, returns joules per token (tokens >= 1) by the
 * reference's trapezoid rule, the sample count and (counter_joules, optional)
 * the joules of the driver's total-energy counter over the same window, or -1
 * when unsupported; frees the sampler.
 * msw_energy_from_trace: the same integration over a CSV trace on disk. */
typedef struct msw_power_sampler msw_power_sampler;
int msw_power_start(int32_t device, double period_ms, msw_power_sampler** out);
int msw_power_stop(msw_power_sampler* s, const char* csv_path, int32_t tokens,
                   double* joules_per_token, int32_t* n_samples, double* counter_joules);
int msw_energy_from_trace(const char* csv_path, int32_t tokens, double* joules_per_token);

const char* msw_host_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* MSW_HOST_H_ */
