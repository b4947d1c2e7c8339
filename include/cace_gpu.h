/*
 * cace_gpu.h — C ABI of the B200 trace-replay engine for CACE
 * (Context-Aware CodeLLM Eviction, arXiv 2506.18796).
 *
 * This is the drop-in boundary for the reference simulator's hot path.  Each
 * entry point names the reference interface (file:line under
 * /root/reference/proj) whose behaviour it reproduces; INTEGRATION.md shows
 * the reference-side binding.  Plain pointers and sizes only.
 *
 *   cace_replay_batch        <- SimulationReport run(const Trace&, const ModelCatalog&,
 *                               const ClusterConfig&, const Policy&)      engine.hpp:60-61
 *                               + the scenario fan-out of run_grid          experiment.hpp:54-55
 *                                 (experiment.cpp:87-122, OpenMP over cells)
 *   cace_select_victim_batch <- std::optional<std::string> select_victim(...) policy.hpp:67-71
 *   cace_eviction_score_batch<- ScoreBreakdown eviction_score(...)          policy.hpp:59-62
 *   cace_dedup_window_batch  <- LookaheadWindow dedup_window(...)           policy.hpp:56-57
 *   cace_service_times_batch <- std::pair<double,double> service_times(...) engine.hpp:54-55
 *   cace_log_selftest        <- the libm log the reference calls             policy.cpp:51
 *   cace_run_metrics_batch   <- RunMetrics compute_run_metrics(const SimulationReport&)
 *                               for every replay of a sweep                 metrics.hpp:29-31
 *   cace_metrics_select      <- LatencySummary summarize(std::vector<double>) metrics.cpp:14-33
 *   cace_trace_parse_jsonl   <- Trace parse_trace(const std::string&)        workload.hpp:71
 *   cace_trace_load_jsonl    <- Trace load_trace(const std::string& path)    workload.hpp:73
 *
 * Error behaviour: every entry returns CACE_OK (0) or one CACE_E_* code per
 * SimError site of the reference, and writes the reference's message text
 * into (msg, msg_cap).  Host wrappers rethrow SimError(msg).  Validation runs
 * on the host before launch; device-side conditions (clock < last_used,
 * deadlock) are reported per scenario in cace_summary_t.status and surfaced
 * as the call's return code for the first failing scenario.
 *
 * Threading: every call is reentrant; each call uses its own stream (or the
 * caller's, CACE_OPT stream) and its own device scratch.  Results are
 * deterministic and independent of scheduling (acceptance.cpp:452-470).
 */
#ifndef CACE_GPU_H
#define CACE_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CACE_ABI_VERSION 1

/* Return / status codes.  One per reference SimError site. */
enum {
  CACE_OK = 0,
  CACE_E_WINDOW = 1,        /* "run: window_length must be >= 1"            engine.cpp:79 */
  CACE_E_ACCELERATORS = 2,  /* "run: need at least one accelerator"         engine.cpp:80-82 */
  CACE_E_LOOKUP = 3,        /* "catalog: no model registered for (...)"     catalog.cpp:110-114 */
  CACE_E_RATES = 4,         /* "service_times: rates must be positive for " engine.cpp:17-20 */
  CACE_E_CLOCK = 5,         /* "eviction_score: clock precedes last_used_s" policy.cpp:43-46 */
  CACE_E_DEADLOCK = 6,      /* "run: deadlock — pending requests ..."       engine.cpp:235-237 */
  CACE_E_RESIDENCY = 7,     /* "run: residency bound violated"              engine.cpp:118-120 */
  CACE_E_DEDUP_LENGTH = 8,  /* "dedup_window: length must be >= 1"          policy.cpp:23 */
  CACE_E_METRICS_EMPTY = 9, /* "compute_run_metrics: empty report"           metrics.cpp:37-39 */
  CACE_E_METRICS_NO_TTFT = 10, /* "...: no completion outcomes for TTFT"     metrics.cpp:53-55 */
  CACE_E_METRICS_NO_E2E = 11,  /* "...: no reasoning outcomes for E2E"       metrics.cpp:56-58 */
  CACE_E_PARSE = 12,        /* ParseError of parse_trace (message = its text) workload.cpp:204-266 */
  CACE_E_IO = 13,           /* "trace: cannot open: <path>"                  workload.cpp:276 */
  CACE_E_INVALID = 20,      /* malformed call (null pointer, bad index, unsupported size) */
  CACE_E_CUDA = 21,         /* CUDA runtime error (message has the CUDA text) */
  CACE_E_NO_DEVICE = 22     /* no CUDA device: there is no CPU fallback */
};

/* cacesim::Variant (types.hpp:63-70) and P1Mode (policy.hpp:29-34). */
enum { CACE_LRU = 0, CACE_FULL = 1, CACE_MINUS_P1 = 2, CACE_MINUS_P2 = 3, CACE_MINUS_P3 = 4,
       CACE_MINUS_P4 = 5 };
enum { CACE_P1_PROSE = 0, CACE_P1_VERBATIM = 1 };
enum { CACE_COMPLETION = 0, CACE_REASONING = 1 };

/* Model catalog, structure-of-arrays, M models (catalog.hpp:13-25).
 * lex_rank[m] = rank of model_id under std::string operator< among the M ids
 * (the tie-break key of policy.cpp:92-98).  Host pointers. */
typedef struct {
  int32_t n_models;
  const double* load_time_s;
  const double* prefill_rate_tps;
  const double* decode_rate_tps;
  const int32_t* expected_output_tokens;
  const int32_t* lex_rank;
  const int32_t* task_class;
  const char* const* model_id; /* optional (NULL): ids for SimError messages */
} cace_catalog_t;

/* One request trace, structure-of-arrays (workload.hpp:15-24).  model[i] is
 * the catalog index catalog.lookup(language, task_class) resolves to.
 * Arrival order: the engine replays requests in (arrival_time_s, index)
 * order, the order run() pops Arrival events (engine.cpp:49-55,103-106);
 * cace_replay_batch stable-sorts when needed and reports outcomes by the
 * caller's request index. */
typedef struct {
  int64_t n_requests;
  const double* arrival_time_s;
  const int32_t* model;
  const int32_t* prompt_tokens;
  const int32_t* output_tokens;
} cace_trace_t;

/* One scenario = one run(trace, catalog, cluster, policy) (engine.hpp:60).
 * PolicyConfig (policy.hpp:39-45) + ClusterConfig (engine.hpp:13-17). */
typedef struct {
  int32_t trace; /* index into the traces array */
  int32_t variant;
  int32_t p1_mode;
  int32_t window_length;
  int32_t output_token_normalizer;
  int32_t num_accelerators;
  int32_t models_per_accelerator;
  int32_t reserved;
  double w1;
  double unload_time_s;
} cace_scenario_t;

/* Fixed-size per-scenario result.  Counters are SimCounters + loads +
 * max_resident (engine.hpp:32-52).  Latency aggregates follow
 * compute_run_metrics' split (metrics.cpp:35-62): TTFT over completion
 * requests, E2E over reasoning requests, summed in replay order.
 * Hashes (spec CACE_HASH below) fingerprint the full per-request outcome
 * stream and the eviction sequence so bit-exact parity can be checked at any
 * scale without storing 10^11 outcomes. */
typedef struct {
  uint64_t hits, misses, evictions, loads;
  double load_overhead_s;
  int32_t max_resident;
  int32_t status; /* CACE_OK or a CACE_E_* code */
  uint64_t n_completion, n_reasoning;
  double sum_ttft_completion, sum_e2e_reasoning;
  double max_ttft_completion, max_e2e_reasoning;
  uint64_t eviction_hash; /* fold over evictions: h = mix(h, bits(clock) ^ (victim_model << 32)) */
  uint64_t outcome_hash;  /* fold over requests in replay order:
                             h = mix(h, bits(ttft) ^ cold) */
} cace_summary_t;

/* CACE_HASH: h0 = 0x6a09e667f3bcc909; mix(h, x) updates the two 32-bit halves
 * independently as polynomial hashes (mod 2^32):
 *   lo(h') = lo(h) * 0x9e3779b1 + lo(x),  hi(h') = hi(h) * 0x85ebca77 + hi(x).
 * Both multipliers are odd, so mix is a bijection in h for a fixed x and any
 * single differing term changes the final value. */
#define CACE_HASH_SEED 0x6a09e667f3bcc909ULL
#define CACE_HASH_MUL_LO 0x9e3779b1u
#define CACE_HASH_MUL_HI 0x85ebca77u

/* LatencySummary (metrics.hpp:11-18) and RunMetrics (metrics.hpp:23-29). */
typedef struct {
  uint64_t count;
  double mean_s, p50_s, p95_s, p99_s, max_s;
} cace_latency_summary_t;
typedef struct {
  double cache_hit_rate;
  double load_overhead_s;
  double evictions;
  cace_latency_summary_t ttft_completion;
  cace_latency_summary_t e2e_reasoning;
  int32_t status; /* CACE_OK, the replay's status, or CACE_E_METRICS_* */
  int32_t reserved;
} cace_run_metrics_t;

/* Optional full dump for a few scenarios: per-request RequestOutcome fields
 * (engine.hpp:19-30) indexed by the caller's request index, and the
 * eviction log (victim model, clock) in eviction order.  Any pointer may be
 * NULL.  Arrays are [n_dump][n_requests of that scenario's trace] and
 * [n_dump][evict_cap]. */
typedef struct {
  int32_t n_dump;
  const int64_t* scenario_index; /* which scenarios to dump */
  uint8_t* cold_start;
  double* queue_wait_s;
  double* load_wait_s;
  double* prefill_s;
  double* decode_s;
  double* ttft_s;
  double* e2e_s;
  int64_t evict_cap;
  int32_t* evict_model;
  double* evict_clock;
  int64_t* n_evict; /* [n_dump] */
} cace_dump_t;

/* glibc log variants (see csrc/glibc_log.cuh). */
#ifndef CACE_LOG_FMA
#define CACE_LOG_FMA 0
#define CACE_LOG_SSE2 1
#endif

/* Engine options. */
enum { CACE_KERNEL_AUTO = 0, CACE_KERNEL_LANE = 1, CACE_KERNEL_WARP = 2 };
typedef struct {
  int32_t device;      /* CUDA device ordinal */
  int32_t kernel;      /* CACE_KERNEL_* (AUTO picks by capacity / pool size) */
  int32_t log_variant; /* -1 = probe this host's libm (default), else CACE_LOG_FMA/SSE2 */
  int32_t reserved;
  void* stream;        /* cudaStream_t or NULL (own stream) */
} cace_opts_t;

const char* cace_version(void);
int32_t cace_abi_version(void);
int32_t cace_device_count(void);

/* The scenario sweep: replay every scenario, write one summary each.
 * catalog/traces/scenarios/summaries/dump are HOST memory. */
int32_t cace_replay_batch(const cace_catalog_t* catalog, const cace_trace_t* traces,
                          int32_t n_traces, const cace_scenario_t* scenarios, int64_t n_scenarios,
                          cace_summary_t* summaries, const cace_dump_t* dump,
                          const cace_opts_t* opts, char* msg, size_t msg_cap);

/* The same sweep on several devices of this process (the device-scale form
 * of run_grid's OpenMP fan-out, experiment.cpp:100-115).  The traces are laid
 * out once and uploaded to every device; the scenarios are split into
 * n_devices shards with cace_shard_scenarios (every shard gets the same
 * (capacity, trace) mix, whole warps); one host thread and stream per device
 * plans and replays its shard; the 112-B summaries are gathered to
 * devices[0] over NCCL (ncclSend/ncclRecv in one group, NVLink / NVSwitch) --
 * peer copies when NCCL is not loadable or a device repeats -- and copied to
 * the caller's array in the caller's order.  *gather_kind (optional): 0 one
 * device, 1 NCCL, 2 peer copies.  Host memory in and out.  Results are
 * identical to cace_replay_batch on one device. */
int32_t cace_replay_batch_multi(const cace_catalog_t* catalog, const cace_trace_t* traces,
                                int32_t n_traces, const cace_scenario_t* scenarios,
                                int64_t n_scenarios, cace_summary_t* summaries,
                                const int32_t* devices, int32_t n_devices, const cace_opts_t* opts,
                                int32_t* gather_kind, char* msg, size_t msg_cap);
/* The shard assignment cace_replay_batch_multi uses (also for one process
 * per GPU: rank r replays the scenarios with shard_of[i] == r).  Every
 * (effective capacity, trace) group is cut into warps of 32 scenarios spread
 * evenly over the shards; scenarios run() would reject go to shard 0.  No
 * GPU needed. */
int32_t cace_shard_scenarios(const cace_scenario_t* scenarios, int64_t n, int32_t n_models,
                             int32_t n_shards, int32_t* shard_of);
/* NCCL version the multi-device gather uses (0 = not loadable). */
int32_t cace_nccl_version(void);

/* compute_run_metrics (metrics.cpp:35-62) of every scenario's replay,
 * computed on the device: the replay captures each scenario's TTFT /
 * E2E samples, one CTA per (scenario, task class) selects the nearest-rank
 * p50 / p95 / p99 and max exactly (metrics.cpp:14-33), and the counters come
 * from the replay summary.  count, percentiles, max, hit rate, load overhead
 * and evictions are bit-identical to the reference; mean_s divides the
 * replay-order sum (the reference sums the sorted samples, metrics.cpp:26), so
 * it agrees to ~1e-15 relative.  The sweep is replayed in chunks pipelined
 * with their selects over ring buffers sized to the free device memory.
 * summaries (optional, NULL) receives the replay summaries too.  Host memory. */
int32_t cace_run_metrics_batch(const cace_catalog_t* catalog, const cace_trace_t* traces,
                               int32_t n_traces, const cace_scenario_t* scenarios,
                               int64_t n_scenarios, cace_run_metrics_t* metrics,
                               cace_summary_t* summaries, const cace_opts_t* opts, char* msg,
                               size_t msg_cap);

/* The order-statistic step of compute_run_metrics alone (summarize,
 * metrics.cpp:14-33: nearest-rank p50 / p95 / p99 and the max) over caller
 * samples, through the same device select kernel the pipeline uses: segment
 * b holds ncomp[b] TTFT samples then nreq[b] - ncomp[b] E2E samples starting
 * at samples[off[b]] (latencies, >= +0).  stat[b * 8 + 4 * class + j] =
 * {p50, p95, p99, max}[j]; an empty class yields zeros (the caller reports
 * the reference's SimError).  spec: 1 speculative first digit (default
 * pipeline behaviour), 0 off, 2 every speculation forced to miss (test hook).
 * Host memory; the samples are copied (the kernel compacts its copy
 * segment by segment in place, so segments must be disjoint: overlapping
 * [off, off + nreq) ranges are rejected with CACE_E_INVALID). */
int32_t cace_metrics_select(const double* samples, const int64_t* off, const uint32_t* ncomp,
                            const uint32_t* nreq, int64_t n_segments, double* stat, int32_t spec,
                            const cace_opts_t* opts, char* msg, size_t msg_cap);

/* Trace ingestion: the reference's JSONL trace format (serialize_trace,
 * workload.cpp:181-202) parsed with parse_trace's semantics and error texts
 * (workload.cpp:204-266) on all host threads, into an opaque handle whose
 * columns are copied out as structure-of-arrays.  language / task_class are
 * the reference's enum codes (types.hpp:23-44); map them to catalog indices
 * with ModelCatalog::lookup before replay.  JSON syntax errors keep the
 * reference's "trace line N: invalid JSON: " prefix with this parser's own
 * description.  No GPU needed. */
typedef struct cace_trace_jsonl cace_trace_jsonl;
int32_t cace_trace_parse_jsonl(const char* text, size_t len, cace_trace_jsonl** out, char* msg,
                               size_t msg_cap);
int32_t cace_trace_load_jsonl(const char* path, cace_trace_jsonl** out, char* msg, size_t msg_cap);
int64_t cace_trace_jsonl_size(const cace_trace_jsonl* t);
void cace_trace_jsonl_header(const cace_trace_jsonl* t, int32_t* pattern, uint64_t* seed,
                             double* rate, double* duration, int32_t* windows);
void cace_trace_jsonl_copy(const cace_trace_jsonl* t, uint64_t* request_id, double* arrival,
                           int32_t* language, int32_t* task_class, int32_t* prompt_tokens,
                           int32_t* output_tokens);
void cace_trace_jsonl_free(cace_trace_jsonl* t);

/* Device-resident engine for repeated sweeps (bench, multi-GPU shards):
 * the catalog and traces are uploaded and pre-laid-out once; replays then
 * take DEVICE arrays of scenarios and summaries and only launch kernels. */
typedef struct cace_engine cace_engine;
int32_t cace_engine_create(const cace_catalog_t* catalog, const cace_trace_t* traces,
                           int32_t n_traces, const cace_opts_t* opts, cace_engine** out,
                           char* msg, size_t msg_cap);
void cace_engine_destroy(cace_engine* e);
/* Plan a sweep: validate the scenarios (host array) with the reference's
 * run() preconditions (engine.cpp:79-92) and group them by capacity / trace /
 * policy so each warp replays coherent scenarios.  Must precede
 * cace_engine_replay_device for the same scenario array.  Returns CACE_OK even
 * when individual scenarios are invalid: their summaries carry the status. */
int32_t cace_engine_plan(cace_engine* e, const cace_scenario_t* scenarios, int64_t n,
                         char* msg, size_t msg_cap);
/* Replay the planned sweep.  d_scenarios / d_summaries are DEVICE pointers
 * (same scenarios, same order as planned); enqueued on `stream` (NULL =
 * engine stream); asynchronous. */
int32_t cace_engine_replay_device(cace_engine* e, const cace_scenario_t* d_scenarios, int64_t n,
                                  cace_summary_t* d_summaries, void* stream, char* msg,
                                  size_t msg_cap);
/* Compose the reference's SimError text for a summary status (the message
 * run() would have thrown for that scenario).  Returns the CACE_E_* code. */
int32_t cace_engine_status_message(const cace_engine* e, int32_t status, char* msg,
                                   size_t msg_cap);
/* Number of replay-kernel launches the last replay_device call issued. */
int32_t cace_engine_last_launches(const cace_engine* e);

/* select_victim over a batch of independent ResidencySets (policy.cpp:80-115).
 * Entry k of instance b: entry_model/last_used/busy[b*max_entries + k], valid
 * for k < n_entries[b].  Window of instance b: window_models[b*max_window + j]
 * (already de-duplicated, first-occurrence order), j < n_window[b].
 * victim_out[b] = catalog index or -1 (all busy).  Host memory. */
int32_t cace_select_victim_batch(const cace_catalog_t* catalog, int64_t n_instances,
                                 int32_t max_entries, const int32_t* n_entries,
                                 const int32_t* entry_model, const double* entry_last_used,
                                 const uint8_t* entry_busy, int32_t max_window,
                                 const int32_t* n_window, const int32_t* window_models,
                                 const double* clock, const cace_scenario_t* policy,
                                 int32_t* victim_out, const cace_opts_t* opts, char* msg,
                                 size_t msg_cap);

/* eviction_score for a batch (policy.cpp:39-78): out[5*b + {0..4}] =
 * {p1_recency, p2_reload, p3_future, p4_criticality, total}. */
int32_t cace_eviction_score_batch(const cace_catalog_t* catalog, int64_t n_instances,
                                  const int32_t* model, const double* last_used,
                                  int32_t max_window, const int32_t* n_window,
                                  const int32_t* window_models, const double* clock,
                                  const cace_scenario_t* policy, double* out,
                                  const cace_opts_t* opts, char* msg, size_t msg_cap);

/* dedup_window for a batch (policy.cpp:22-37): out_models[b*max_pending + j]
 * for j < n_out[b]. */
int32_t cace_dedup_window_batch(int64_t n_instances, int32_t max_pending, const int32_t* n_pending,
                                const int32_t* pending_models, const int32_t* length,
                                int32_t* out_models, int32_t* n_out, const cace_opts_t* opts,
                                char* msg, size_t msg_cap);

/* service_times (engine.cpp:15-26) for a batch of requests. */
int32_t cace_service_times_batch(const cace_catalog_t* catalog, int64_t n, const int32_t* model,
                                 const int32_t* prompt_tokens, const int32_t* output_tokens,
                                 double* prefill_s, double* decode_s, const cace_opts_t* opts,
                                 char* msg, size_t msg_cap);

/* Device glibc-log restatement over x[0..n) (host arrays), variant as in
 * cace_opts_t.log_variant.  Used to pin P1 against the host's libm. */
int32_t cace_log_selftest(const double* x, int64_t n, int32_t log_variant, double* out,
                          const cace_opts_t* opts, char* msg, size_t msg_cap);
/* The same restatement evaluated on the host CPU (no GPU needed). */
void cace_log_host(const double* x, int64_t n, int32_t log_variant, double* out);
/* Which glibc log variant this host's libm matches (CACE_LOG_FMA / _SSE2),
 * or -1 if neither (then bit-exact P1 parity cannot be claimed). */
int32_t cace_probe_log_variant(void);

#ifdef __cplusplus
}
#endif
#endif /* CACE_GPU_H */
