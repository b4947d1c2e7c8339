// TEST INFRASTRUCTURE ONLY — never linked into, or called by, the product.
//
// C-ABI shim over the UNMODIFIED reference simulator (arXiv 2506.18796 artifact,
// /root/reference/proj/src/*.cpp), compiled out of tree by oracle/Makefile into
// oracle/_ref/libcace_ref.so.  No reference source is copied: this file only
// calls the reference's public API (engine.hpp:60 run, policy.hpp:56-71
// dedup_window/eviction_score/select_victim, workload.hpp:66 build_trace,
// catalog.hpp:45-58 ModelCatalog) and converts plain arrays to/from its types.
//
// The reference does not expose its eviction sequence, so the link step wraps
// the one external call engine.cpp:203 makes into policy.cpp
// (`-Wl,--wrap=<cacesim::select_victim>`, see Makefile): every non-empty victim
// returned to run() is appended to a thread-local recorder.  The reference code
// itself is untouched.
//
// Consumers: tests/ (parity oracle, golden-vector generation) and bench.py's
// cpu_baseline / --impl reference leg.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include <pthread.h>

#include <atomic>
#include <mutex>
#include <thread>

#include "cacesim/catalog.hpp"
#include "cacesim/engine.hpp"
#include "cacesim/metrics.hpp"
#include "cacesim/policy.hpp"
#include "cacesim/types.hpp"
#include "cacesim/workload.hpp"

using namespace cacesim;

// ---------------------------------------------------------------------------
// select_victim interposition (link-time --wrap; engine.o's undefined
// reference is redirected here, policy.o keeps the real definition).

#define SV_MANGLED \
  "_ZN7cacesim13select_victimB5cxx11ERKNS_12ResidencySetERKNS_15LookaheadWindowERKNS_12ModelCatalogEdRKNS_12PolicyConfigE"

std::optional<std::string> real_select_victim(const ResidencySet&, const LookaheadWindow&,
                                              const ModelCatalog&, double,
                                              const PolicyConfig&) __asm__("__real_" SV_MANGLED);

namespace {
struct EvictionRecorder {
  std::vector<std::string> victims;
  std::vector<double> clocks;
  bool active = false;
};
// One recorder per calling thread, found through POSIX thread-specific data.
// (Compiler TLS — thread_local, libgomp — faults when ctypes dlopen()s this
// library with this toolchain, so there is no OpenMP here: the CPU fan-out
// below uses std::thread with experiment.cpp:105's dynamic scheduling.)
pthread_key_t g_key;
pthread_once_t g_key_once = PTHREAD_ONCE_INIT;
EvictionRecorder g_idle;  // never active; returned for unregistered threads
void make_key() { pthread_key_create(&g_key, nullptr); }
inline EvictionRecorder& rec() {
  pthread_once(&g_key_once, make_key);
  void* p = pthread_getspecific(g_key);
  return p ? *static_cast<EvictionRecorder*>(p) : g_idle;
}
struct RecorderScope {  // binds a recorder to the calling thread
  EvictionRecorder r;
  RecorderScope() {
    pthread_once(&g_key_once, make_key);
    pthread_setspecific(g_key, &r);
  }
  ~RecorderScope() { pthread_setspecific(g_key, nullptr); }
};
}  // namespace

std::optional<std::string> wrapped_select_victim(const ResidencySet& r, const LookaheadWindow& w,
                                                 const ModelCatalog& c, double clock,
                                                 const PolicyConfig& cfg) __asm__("__wrap_" SV_MANGLED);
std::optional<std::string> wrapped_select_victim(const ResidencySet& r, const LookaheadWindow& w,
                                                 const ModelCatalog& c, double clock,
                                                 const PolicyConfig& cfg) {
  auto v = real_select_victim(r, w, c, clock, cfg);
  EvictionRecorder& g_rec = rec();
  if (g_rec.active && v) {
    g_rec.victims.push_back(*v);
    g_rec.clocks.push_back(clock);
  }
  return v;
}

// ---------------------------------------------------------------------------

extern "C" {

struct ref_scenario_t {
  int32_t trace;
  int32_t variant;  // cacesim::Variant numbering (types.hpp:63-70)
  int32_t p1_mode;  // cacesim::P1Mode numbering (policy.hpp:29-34)
  int32_t window_length;
  int32_t output_token_normalizer;
  int32_t num_accelerators;
  int32_t models_per_accelerator;
  int32_t pad_;
  double w1;
  double unload_time_s;
};

struct ref_counters_t {
  uint64_t hits, misses, evictions, loads;
  double load_overhead_s;
  int64_t max_resident;
};

// Per-scenario summary; field meaning identical to cace_summary_t in
// include/cace_gpu.h (restated here, the oracle does not include product code).
struct ref_summary_t {
  uint64_t hits, misses, evictions, loads;
  double load_overhead_s;
  int32_t max_resident;
  int32_t status;
  uint64_t n_completion, n_reasoning;
  double sum_ttft_completion, sum_e2e_reasoning;
  double max_ttft_completion, max_e2e_reasoning;
  uint64_t eviction_hash, outcome_hash;
};

}  // extern "C"

namespace {

void put_msg(char* msg, size_t cap, const std::string& s) {
  if (!msg || cap == 0) return;
  size_t k = std::min(cap - 1, s.size());
  std::memcpy(msg, s.data(), k);
  msg[k] = 0;
}

// Summary hash: the spec documented at include/cace_gpu.h (CACE_HASH_*).
inline uint64_t mix(uint64_t h, uint64_t x) {
  /* CACE_HASH, include/cace_gpu.h */
  const uint32_t lo = (uint32_t)h * 0x9e3779b1u + (uint32_t)x;
  const uint32_t hi = (uint32_t)(h >> 32) * 0x85ebca77u + (uint32_t)(x >> 32);
  return ((uint64_t)hi << 32) | lo;
}
inline uint64_t bits(double d) {
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
}
constexpr uint64_t kHashSeed = 0x6a09e667f3bcc909ULL;

PolicyConfig to_policy(const ref_scenario_t& s) {
  PolicyConfig pc;
  pc.variant = static_cast<Variant>(s.variant);
  pc.p1_mode = static_cast<P1Mode>(s.p1_mode);
  pc.window_length = s.window_length;
  pc.output_token_normalizer = s.output_token_normalizer;
  pc.w1 = s.w1;
  return pc;
}

ClusterConfig to_cluster(const ref_scenario_t& s) {
  ClusterConfig cc;
  cc.num_accelerators = s.num_accelerators;
  cc.models_per_accelerator = s.models_per_accelerator;
  cc.unload_time_s = s.unload_time_s;
  return cc;
}

Trace make_trace(const ModelCatalog& cat, const double* arrival, const int32_t* model_idx,
                 const int32_t* prompt, const int32_t* output, int64_t n) {
  Trace t;
  t.requests.resize(static_cast<size_t>(n));
  const auto& models = cat.models();
  for (int64_t i = 0; i < n; ++i) {
    Request& r = t.requests[static_cast<size_t>(i)];
    const ModelDescriptor& m = models.at(static_cast<size_t>(model_idx[i]));
    r.request_id = static_cast<uint64_t>(i);
    r.arrival_time_s = arrival[i];
    r.language = m.language;
    r.task_class = m.task_class;
    r.prompt_tokens = prompt[i];
    r.output_tokens = output[i];
  }
  return t;
}

int model_index(const ModelCatalog& cat, const std::string& id) {
  const auto& models = cat.models();
  for (size_t i = 0; i < models.size(); ++i)
    if (models[i].model_id == id) return static_cast<int>(i);
  return -1;
}

// Summary over a report, outcomes visited in arrival order (stable by index),
// matching the device engine's service order.
void summarize_report(const SimulationReport& rep, const Trace& t, const ModelCatalog& cat,
                      const std::vector<std::string>& victims, const std::vector<double>& clocks,
                      ref_summary_t* s) {
  std::memset(s, 0, sizeof(*s));
  s->hits = rep.counters.hits;
  s->misses = rep.counters.misses;
  s->evictions = rep.counters.evictions;
  s->loads = rep.loads;
  s->load_overhead_s = rep.counters.load_overhead_s;
  s->max_resident = rep.max_resident;
  const size_t n = rep.outcomes.size();
  std::vector<size_t> order(n);
  for (size_t i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    return t.requests[a].arrival_time_s < t.requests[b].arrival_time_s;
  });
  uint64_t h = kHashSeed;
  for (size_t k : order) {
    const RequestOutcome& o = rep.outcomes[k];
    if (o.task_class == TaskClass::Completion) {
      s->n_completion++;
      s->sum_ttft_completion += o.ttft_s;
      if (o.ttft_s > s->max_ttft_completion) s->max_ttft_completion = o.ttft_s;
    } else {
      s->n_reasoning++;
      s->sum_e2e_reasoning += o.e2e_s;
      if (o.e2e_s > s->max_e2e_reasoning) s->max_e2e_reasoning = o.e2e_s;
    }
    h = mix(h, bits(o.ttft_s) ^ (o.cold_start ? 1ULL : 0ULL));
  }
  s->outcome_hash = h;
  uint64_t he = kHashSeed;
  for (size_t k = 0; k < victims.size(); ++k) {
    he = mix(he, bits(clocks[k]) ^ (static_cast<uint64_t>(model_index(cat, victims[k])) << 32));
  }
  s->eviction_hash = he;
}

}  // namespace

extern "C" {

const char* ref_version(void) { return "cacesim-reference (arXiv 2506.18796 artifact), oracle shim v1"; }

void* ref_catalog_default(void) { return new ModelCatalog(ModelCatalog::build_default()); }

void* ref_catalog_from_json(const char* json, char* msg, size_t cap) {
  try {
    return new ModelCatalog(ModelCatalog::load(std::string(json)));
  } catch (const std::exception& e) {
    put_msg(msg, cap, e.what());
    return nullptr;
  }
}

void ref_catalog_free(void* cat) { delete static_cast<ModelCatalog*>(cat); }

int64_t ref_catalog_json(void* cat, char* buf, size_t cap) {
  std::string s = static_cast<ModelCatalog*>(cat)->save();
  put_msg(buf, cap, s);
  return static_cast<int64_t>(s.size());
}

int32_t ref_catalog_size(void* cat) {
  return static_cast<int32_t>(static_cast<ModelCatalog*>(cat)->models().size());
}

int32_t ref_catalog_max_tokens(void* cat) {
  return static_cast<ModelCatalog*>(cat)->max_expected_output_tokens();
}

// Reference trace generator (workload.cpp:127-179) with default TokenParams.
int32_t ref_build_trace(void* catp, int32_t pattern, double rate, double duration, uint64_t seed,
                        int32_t windows, int64_t cap, double* arrival, int32_t* model_idx,
                        int32_t* prompt, int32_t* output, int64_t* n_out, char* msg, size_t mcap) {
  try {
    const ModelCatalog& cat = *static_cast<ModelCatalog*>(catp);
    Trace t = build_trace(static_cast<PatternName>(pattern), rate, duration, seed, cat,
                          TokenParams{}, windows);
    *n_out = static_cast<int64_t>(t.requests.size());
    for (size_t i = 0; i < t.requests.size() && static_cast<int64_t>(i) < cap; ++i) {
      const Request& r = t.requests[i];
      arrival[i] = r.arrival_time_s;
      model_idx[i] = model_index(cat, cat.lookup(r.language, r.task_class).model_id);
      prompt[i] = r.prompt_tokens;
      output[i] = r.output_tokens;
    }
    return 0;
  } catch (const SimError& e) {
    put_msg(msg, mcap, e.what());
    return 1;
  } catch (const std::exception& e) {
    put_msg(msg, mcap, e.what());
    return 2;
  }
}

// One replay through the reference run() (engine.cpp:76-239).  Outcome arrays
// are indexed by request position (the reference's outcome order); any may be
// NULL.  Victims are catalog indices in eviction order.
int32_t ref_run(void* catp, const double* arrival, const int32_t* model_idx, const int32_t* prompt,
                const int32_t* output, int64_t n, const ref_scenario_t* sc, ref_counters_t* counters,
                uint8_t* cold, double* queue_wait, double* load_wait, double* prefill,
                double* decode, double* ttft, double* e2e, int32_t* evict_model,
                double* evict_clock, int64_t evict_cap, int64_t* n_evict, char* msg, size_t mcap) {
  RecorderScope scope;
  EvictionRecorder& g_rec = scope.r;
  g_rec.victims.clear();
  g_rec.clocks.clear();
  try {
    const ModelCatalog& cat = *static_cast<ModelCatalog*>(catp);
    Trace t = make_trace(cat, arrival, model_idx, prompt, output, n);
    Policy pol = make_policy(to_policy(*sc));
    g_rec.active = true;
    SimulationReport rep = run(t, cat, to_cluster(*sc), pol);
    g_rec.active = false;
    counters->hits = rep.counters.hits;
    counters->misses = rep.counters.misses;
    counters->evictions = rep.counters.evictions;
    counters->loads = rep.loads;
    counters->load_overhead_s = rep.counters.load_overhead_s;
    counters->max_resident = rep.max_resident;
    for (int64_t i = 0; i < n; ++i) {
      const RequestOutcome& o = rep.outcomes[static_cast<size_t>(i)];
      if (cold) cold[i] = o.cold_start ? 1 : 0;
      if (queue_wait) queue_wait[i] = o.queue_wait_s;
      if (load_wait) load_wait[i] = o.load_wait_s;
      if (prefill) prefill[i] = o.prefill_s;
      if (decode) decode[i] = o.decode_s;
      if (ttft) ttft[i] = o.ttft_s;
      if (e2e) e2e[i] = o.e2e_s;
    }
    *n_evict = static_cast<int64_t>(g_rec.victims.size());
    for (size_t k = 0; k < g_rec.victims.size() && static_cast<int64_t>(k) < evict_cap; ++k) {
      if (evict_model) evict_model[k] = model_index(cat, g_rec.victims[k]);
      if (evict_clock) evict_clock[k] = g_rec.clocks[k];
    }
    return 0;
  } catch (const SimError& e) {
    g_rec.active = false;
    put_msg(msg, mcap, e.what());
    return 1;
  } catch (const std::exception& e) {
    g_rec.active = false;
    put_msg(msg, mcap, e.what());
    return 2;
  }
}

// Reference parse_trace (workload.cpp:204-266): columns of the parsed
// Trace (up to cap requests) + header; language / task_class as enum codes.
int32_t ref_parse_trace(const char* text, int64_t len, int64_t cap, uint64_t* request_id,
                        double* arrival, int32_t* language, int32_t* task_class, int32_t* prompt,
                        int32_t* output, int64_t* n_out, int32_t* pattern, uint64_t* seed,
                        double* rate, double* duration, int32_t* windows, char* msg, size_t mcap) {
  try {
    Trace t = parse_trace(std::string(text, static_cast<size_t>(len)));
    *n_out = static_cast<int64_t>(t.requests.size());
    *pattern = static_cast<int32_t>(t.pattern);
    *seed = t.seed;
    *rate = t.arrival_rate_per_s;
    *duration = t.window_duration_s;
    *windows = t.windows;
    for (size_t i = 0; i < t.requests.size() && static_cast<int64_t>(i) < cap; ++i) {
      const Request& r = t.requests[i];
      request_id[i] = r.request_id;
      arrival[i] = r.arrival_time_s;
      language[i] = static_cast<int32_t>(r.language);
      task_class[i] = static_cast<int32_t>(r.task_class);
      prompt[i] = r.prompt_tokens;
      output[i] = r.output_tokens;
    }
    return 0;
  } catch (const SimError& e) {
    put_msg(msg, mcap, e.what());
    return 1;
  } catch (const std::exception& e) {
    put_msg(msg, mcap, e.what());
    return 2;
  }
}

// Reference serialize_trace (workload.cpp:181-202) of the trace build_trace
// generates: writes up to cap bytes, returns the full length.
int64_t ref_serialize_built_trace(int32_t pattern, double rate, double duration, uint64_t seed,
                                  int32_t windows, char* out, int64_t cap) {
  const ModelCatalog cat = ModelCatalog::build_default();
  Trace t = build_trace(static_cast<PatternName>(pattern), rate, duration, seed, cat, TokenParams{},
                        windows);
  const std::string s = serialize_trace(t);
  if (out && cap > 0) std::memcpy(out, s.data(), std::min<size_t>(s.size(), static_cast<size_t>(cap)));
  return static_cast<int64_t>(s.size());
}

// Reference compute_run_metrics (metrics.cpp:35-62) of one run():
// out = {hit_rate, load_overhead_s, evictions, ttft{mean,p50,p95,p99,max},
// e2e{mean,p50,p95,p99,max}}, counts = {ttft count, e2e count}.
int32_t ref_run_metrics(void* catp, const double* arrival, const int32_t* model_idx,
                        const int32_t* prompt, const int32_t* output, int64_t n,
                        const ref_scenario_t* sc, double* out, uint64_t* counts, char* msg,
                        size_t mcap) {
  try {
    const ModelCatalog& cat = *static_cast<ModelCatalog*>(catp);
    Trace t = make_trace(cat, arrival, model_idx, prompt, output, n);
    Policy pol = make_policy(to_policy(*sc));
    SimulationReport rep = run(t, cat, to_cluster(*sc), pol);
    RunMetrics m = compute_run_metrics(rep);
    out[0] = m.cache_hit_rate;
    out[1] = m.load_overhead_s;
    out[2] = m.evictions;
    const LatencySummary* ls[2] = {&m.ttft_completion, &m.e2e_reasoning};
    for (int c = 0; c < 2; ++c) {
      counts[c] = ls[c]->count;
      out[3 + 5 * c + 0] = ls[c]->mean_s;
      out[3 + 5 * c + 1] = ls[c]->p50_s;
      out[3 + 5 * c + 2] = ls[c]->p95_s;
      out[3 + 5 * c + 3] = ls[c]->p99_s;
      out[3 + 5 * c + 4] = ls[c]->max_s;
    }
    return 0;
  } catch (const SimError& e) {
    put_msg(msg, mcap, e.what());
    return 1;
  } catch (const std::exception& e) {
    put_msg(msg, mcap, e.what());
    return 2;
  }
}

// Reference dedup_window (policy.cpp:22-37) over catalog indices.
int32_t ref_dedup_window(void* catp, const int32_t* pending_model, int32_t n_pending,
                         int32_t length, int32_t* out_models, int32_t* n_out, char* msg,
                         size_t mcap) {
  try {
    const ModelCatalog& cat = *static_cast<ModelCatalog*>(catp);
    std::vector<std::string> ids;
    for (int32_t i = 0; i < n_pending; ++i)
      ids.push_back(cat.models().at(static_cast<size_t>(pending_model[i])).model_id);
    LookaheadWindow w = dedup_window(ids, length);
    *n_out = static_cast<int32_t>(w.model_ids.size());
    for (size_t k = 0; k < w.model_ids.size(); ++k) out_models[k] = model_index(cat, w.model_ids[k]);
    return 0;
  } catch (const SimError& e) {
    put_msg(msg, mcap, e.what());
    return 1;
  }
}

// Reference eviction_score (policy.cpp:39-78).  window_models is the already
// de-duplicated window (first-occurrence order).  out = {p1,p2,p3,p4,total}.
int32_t ref_eviction_score(void* catp, int32_t model, double last_used, const int32_t* window_models,
                           int32_t n_window, int32_t window_length, double clock,
                           const ref_scenario_t* sc, double* out, char* msg, size_t mcap) {
  try {
    const ModelCatalog& cat = *static_cast<ModelCatalog*>(catp);
    const ModelDescriptor& d = cat.models().at(static_cast<size_t>(model));
    LookaheadWindow w;
    w.length = window_length;
    for (int32_t k = 0; k < n_window; ++k)
      w.model_ids.push_back(cat.models().at(static_cast<size_t>(window_models[k])).model_id);
    ResidencyEntry e{d.model_id, last_used, false};
    ScoreBreakdown s = eviction_score(e, d, w, clock, to_policy(*sc));
    out[0] = s.p1_recency;
    out[1] = s.p2_reload;
    out[2] = s.p3_future;
    out[3] = s.p4_criticality;
    out[4] = s.total;
    return 0;
  } catch (const SimError& e) {
    put_msg(msg, mcap, e.what());
    return 1;
  }
}

// Reference select_victim (policy.cpp:80-115).  Returns the victim's catalog
// index in *victim, or -1 when every resident is busy.
int32_t ref_select_victim(void* catp, const int32_t* entry_model, const double* entry_last_used,
                          const uint8_t* entry_busy, int32_t n_entries,
                          const int32_t* window_models, int32_t n_window, int32_t window_length,
                          double clock, const ref_scenario_t* sc, int32_t* victim, char* msg,
                          size_t mcap) {
  try {
    const ModelCatalog& cat = *static_cast<ModelCatalog*>(catp);
    ResidencySet set;
    for (int32_t k = 0; k < n_entries; ++k)
      set.entries.push_back(ResidencyEntry{
          cat.models().at(static_cast<size_t>(entry_model[k])).model_id, entry_last_used[k],
          entry_busy[k] != 0});
    LookaheadWindow w;
    w.length = window_length;
    for (int32_t k = 0; k < n_window; ++k)
      w.model_ids.push_back(cat.models().at(static_cast<size_t>(window_models[k])).model_id);
    auto v = real_select_victim(set, w, cat, clock, to_policy(*sc));
    *victim = v ? model_index(cat, *v) : -1;
    return 0;
  } catch (const SimError& e) {
    put_msg(msg, mcap, e.what());
    return 1;
  }
}

// CPU batch: the reference's own fan-out pattern (experiment.cpp:105,
// `#pragma omp parallel for schedule(dynamic)`, here std::thread + an atomic
// work counter) over scenarios, each a full
// reference run().  Traces are concatenated; trace k occupies
// [offsets[k], offsets[k+1]).  Only the parallel region is timed.
int32_t ref_run_batch(void* catp, const double* arrival, const int32_t* model_idx,
                      const int32_t* prompt, const int32_t* output, const int64_t* offsets,
                      int32_t n_traces, const ref_scenario_t* scenarios, int64_t n_scenarios,
                      int32_t threads, ref_summary_t* summaries, double* seconds, char* msg,
                      size_t mcap) {
  const ModelCatalog& cat = *static_cast<ModelCatalog*>(catp);
  std::vector<Trace> traces;
  try {
    for (int32_t k = 0; k < n_traces; ++k) {
      int64_t b = offsets[k], e = offsets[k + 1];
      traces.push_back(make_trace(cat, arrival + b, model_idx + b, prompt + b, output + b, e - b));
    }
  } catch (const std::exception& e) {
    put_msg(msg, mcap, e.what());
    return 2;
  }
  int nthr = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
  if (nthr < 1) nthr = 1;
  std::string error;
  std::mutex err_mu;
  std::atomic<int64_t> next{0};
  auto worker = [&]() {
    RecorderScope scope;
    EvictionRecorder& g_rec = scope.r;
    for (;;) {
      const int64_t i = next.fetch_add(1, std::memory_order_relaxed);  // schedule(dynamic)
      if (i >= n_scenarios) break;
      const ref_scenario_t& sc = scenarios[i];
      try {
        g_rec.victims.clear();
        g_rec.clocks.clear();
        g_rec.active = true;
        const Trace& t = traces.at(static_cast<size_t>(sc.trace));
        SimulationReport rep = run(t, cat, to_cluster(sc), make_policy(to_policy(sc)));
        g_rec.active = false;
        summarize_report(rep, t, cat, g_rec.victims, g_rec.clocks, &summaries[i]);
      } catch (const std::exception& e) {
        g_rec.active = false;
        std::memset(&summaries[i], 0, sizeof(ref_summary_t));
        summaries[i].status = 1;
        std::lock_guard<std::mutex> lk(err_mu);
        if (error.empty()) error = e.what();
      }
    }
  };
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int k = 1; k < nthr; ++k) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  auto t1 = std::chrono::steady_clock::now();
  if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
  if (!error.empty()) {
    put_msg(msg, mcap, error);
    return 1;
  }
  return 0;
}

// CPU baseline timing: the same fan-out running the reference run() only --
// no eviction recorder bound (the --wrap shim just forwards to
// select_victim) and no summary; reports are discarded.  This is what
// bench_grid.cpp:18-25 times (run_grid wall time around run()).
int32_t ref_time_batch(void* catp, const double* arrival, const int32_t* model_idx, const int32_t* prompt,
                       const int32_t* output, const int64_t* offsets, int32_t n_traces,
                       const ref_scenario_t* scenarios, int64_t n_scenarios, int32_t threads, double* seconds,
                       char* msg, size_t mcap) {
  const ModelCatalog& cat = *static_cast<ModelCatalog*>(catp);
  std::vector<Trace> traces;
  try {
    for (int32_t k = 0; k < n_traces; ++k) {
      int64_t b = offsets[k], e = offsets[k + 1];
      traces.push_back(make_trace(cat, arrival + b, model_idx + b, prompt + b, output + b, e - b));
    }
  } catch (const std::exception& e) {
    put_msg(msg, mcap, e.what());
    return 2;
  }
  int nthr = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
  if (nthr < 1) nthr = 1;
  std::string error;
  std::mutex err_mu;
  std::atomic<int64_t> next{0};
  std::atomic<uint64_t> sink{0};
  auto worker = [&]() {
    for (;;) {
      const int64_t i = next.fetch_add(1, std::memory_order_relaxed);  // schedule(dynamic)
      if (i >= n_scenarios) break;
      const ref_scenario_t& sc = scenarios[i];
      try {
        SimulationReport rep = run(traces.at(static_cast<size_t>(sc.trace)), cat, to_cluster(sc),
                                   make_policy(to_policy(sc)));
        sink.fetch_add(rep.counters.evictions, std::memory_order_relaxed);
      } catch (const std::exception& e) {
        std::lock_guard<std::mutex> lk(err_mu);
        if (error.empty()) error = e.what();
      }
    }
  };
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int k = 1; k < nthr; ++k) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  auto t1 = std::chrono::steady_clock::now();
  if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
  if (!error.empty()) {
    put_msg(msg, mcap, error);
    return 1;
  }
  return 0;
}

int32_t ref_max_threads(void) { return static_cast<int32_t>(std::thread::hardware_concurrency()); }

// libm log as the reference calls it (policy.cpp:51), for device-log pinning.
void ref_libm_log(const double* x, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = std::log(x[i]);
}

}  // extern "C"
