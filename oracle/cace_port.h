/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference replay path
 * (engine.cpp:76-239, policy.cpp:22-115), generalised to model pools the
 * reference cannot key (>16 models: model = catalog index, tie-break by
 * lex_rank).  Checked bit-exact against oracle/_ref on every reference-
 * expressible configuration (tests/test_cpu_port.py) before it is trusted for
 * the configurations only it can run (BASELINE config 5).  Never linked into
 * the product. */
#ifndef CACE_PORT_H
#define CACE_PORT_H
#include <stddef.h>
#include <stdint.h>

typedef struct {
  int32_t n_models;
  const double* load_time_s;
  const double* prefill_rate_tps;
  const double* decode_rate_tps;
  const int32_t* expected_output_tokens;
  const int32_t* lex_rank;
  const int32_t* task_class;
} port_catalog_t;

typedef struct {
  int32_t trace, variant, p1_mode, window_length, output_token_normalizer, num_accelerators,
      models_per_accelerator, reserved;
  double w1, unload_time_s;
} port_scenario_t;

typedef struct {
  uint64_t hits, misses, evictions, loads;
  double load_overhead_s;
  int32_t max_resident, status;
  uint64_t n_completion, n_reasoning;
  double sum_ttft_completion, sum_e2e_reasoning, max_ttft_completion, max_e2e_reasoning;
  uint64_t eviction_hash, outcome_hash;
} port_summary_t;

/* One run(); per-request outputs (request order) and the eviction log are
 * optional (NULL).  Returns 0 or a status code (same numbering as
 * include/cace_gpu.h), message in msg. */
int32_t port_run(const port_catalog_t* cat, const double* arrival, const int32_t* model,
                 const int32_t* prompt, const int32_t* output, int64_t n,
                 const port_scenario_t* sc, port_summary_t* summary, uint8_t* cold,
                 double* queue_wait, double* load_wait, double* prefill, double* decode,
                 double* ttft, double* e2e, int32_t* evict_model, double* evict_clock,
                 int64_t evict_cap, int64_t* n_evict, char* msg, size_t msg_cap);

/* Threaded fan-out over scenarios (traces concatenated by offsets). */
int32_t port_run_batch(const port_catalog_t* cat, const double* arrival, const int32_t* model,
                       const int32_t* prompt, const int32_t* output, const int64_t* offsets,
                       int32_t n_traces, const port_scenario_t* sc, int64_t n_scenarios,
                       int32_t threads, port_summary_t* out, double* seconds);
#endif
