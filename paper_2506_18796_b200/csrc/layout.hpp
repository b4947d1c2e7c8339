// Host-side preparation shared by the C ABI (capi.cu) and the test-only host
// emulation build: catalog validation, the replay-order trace layout
// (ReqRec records, next-same-model links, per-model first occurrences) and the
// reference run() preconditions per scenario.
#pragma once
#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cace_gpu.h"
#include "replay_types.h"

namespace cace {

struct Invalid {
  int32_t code;
  std::string what;
};

inline std::string model_name(const std::vector<std::string>& ids, int m) {
  if (m >= 0 && m < (int)ids.size() && !ids[m].empty()) return ids[m];
  return "model#" + std::to_string(m);
}

constexpr int kMaxLaneC = 16;  // capacities the lane kernel is instantiated for
constexpr int kMaxWarpC = 64;  // warp kernel: <= 2 slots per lane

// Host copy of the catalog columns the replay reads (catalog.hpp:13-25).
struct HostCatalog {
  int M = 0;
  std::vector<double> lt, pr, dr, tok, p2;
  std::vector<int32_t> lex, cls;
  std::vector<std::string> ids;

  void load(const cace_catalog_t* c) {
    if (!c || c->n_models < 1 || c->n_models > 16383 || !c->load_time_s || !c->prefill_rate_tps ||
        !c->decode_rate_tps || !c->expected_output_tokens || !c->lex_rank || !c->task_class)
      throw Invalid{CACE_E_INVALID, "cace: malformed catalog"};
    M = c->n_models;
    for (int m = 0; m < M; ++m) {
      // catalog.cpp:49 rejects load_time_s <= 0; infinite times/rates would
      // make the event clock non-monotone, which the engine does not model.
      if (!(c->load_time_s[m] > 0) || !std::isfinite(c->load_time_s[m]))
        throw Invalid{CACE_E_INVALID, "catalog: load_time_s must be positive and finite"};
      if (std::isinf(c->prefill_rate_tps[m]) || std::isinf(c->decode_rate_tps[m]) ||
          std::isnan(c->prefill_rate_tps[m]) || std::isnan(c->decode_rate_tps[m]))
        throw Invalid{CACE_E_INVALID, "catalog: prefill/decode rates must be finite"};
      if (c->lex_rank[m] < 0 || c->lex_rank[m] >= M)
        throw Invalid{CACE_E_INVALID, "cace: lex_rank out of range"};
    }
    lt.assign(c->load_time_s, c->load_time_s + M);
    pr.assign(c->prefill_rate_tps, c->prefill_rate_tps + M);
    dr.assign(c->decode_rate_tps, c->decode_rate_tps + M);
    tok.resize(M);
    p2.resize(M);
    for (int m = 0; m < M; ++m) {
      tok[m] = (double)c->expected_output_tokens[m];
      p2[m] = 1.0 / (1.0 + lt[m] / 100.0);  // policy.cpp:55
    }
    lex.assign(c->lex_rank, c->lex_rank + M);
    cls.assign(c->task_class, c->task_class + M);
    ids.assign(M, std::string());
    if (c->model_id)
      for (int m = 0; m < M; ++m)
        if (c->model_id[m]) ids[m] = c->model_id[m];
  }
  bool bad_rates(int m) const { return pr[m] <= 0 || dr[m] <= 0; }  // engine.cpp:17
};

// std::allocator that default-initialises (no zero fill of the large
// record array: every element is written by build_layout).
template <class T>
struct DefaultInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = DefaultInitAlloc<U>;
  };
  DefaultInitAlloc() = default;
  template <class U>
  DefaultInitAlloc(const DefaultInitAlloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept {
    ::new ((void*)p) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new ((void*)p) U(std::forward<A>(a)...);
  }
};

// Replay-order layout of all traces, concatenated.
struct HostLayout {
  int T = 0;
  int M = 0;                       // catalog size the layout was built for
  std::vector<int64_t> off;        // [T+1]
  std::vector<ReqRec, DefaultInitAlloc<ReqRec>> rec;  // [N] sorted by (arrival, index)
  ReqRec* ext_rec = nullptr;  // if set (>= N records): records are written here instead of `rec`
  ReqRec* records() { return ext_rec ? ext_rec : rec.data(); }
  std::vector<uint32_t> perm;      // [N] sorted position -> caller's request index
  std::vector<uint32_t> first0;    // [T][M] first sorted index of each model (n if absent)
  std::vector<int32_t> bad_model;  // [T] model of the first request with bad rates, or -1
  std::vector<uint32_t> ncomp;     // [T] completion-class requests
};

inline int64_t layout_requests(const cace_trace_t* traces, int32_t n_traces) {
  int64_t N = 0;
  for (int t = 0; t < n_traces; ++t) N += std::max<int64_t>(0, traces[t].n_requests);
  return N;
}

inline void build_layout(const HostCatalog& cat, const cace_trace_t* traces, int32_t n_traces,
                         HostLayout& L) {
  const int M = cat.M;
  if (n_traces < 0 || (n_traces > 0 && !traces)) throw Invalid{CACE_E_INVALID, "cace: bad traces"};
  L.T = n_traces;
  L.M = M;
  L.off.assign(n_traces + 1, 0);
  for (int t = 0; t < n_traces; ++t) {
    // replay index k < 2^30: the kernels pack (event kind, push seq) into one
    // 32-bit cursor word (replay_lane.cuh)
    if (traces[t].n_requests < 0 || traces[t].n_requests >= (1LL << 30))
      throw Invalid{CACE_E_INVALID, "cace: trace too long (more than 2^30 - 1 requests)"};
    L.off[t + 1] = L.off[t] + traces[t].n_requests;
  }
  const int64_t N = L.off[n_traces];
  L.rec.clear();
  if (!L.ext_rec) L.rec.resize(N);
  ReqRec* const rec = L.records();
  L.perm.resize(N);
  L.first0.assign((size_t)n_traces * M, 0);
  L.bad_model.assign(n_traces, -1);
  L.ncomp.assign(n_traces, 0);
  // Traces are independent: lay them out on several host threads; the error
  // reported is the one of the lowest-numbered failing trace (as a serial
  // pass would report).
  std::vector<double> worst_t(n_traces, 0.0);
  std::vector<int> err_t(n_traces, 0);
  std::vector<Invalid> err_v(n_traces);
  auto one = [&](int t, std::vector<uint32_t>& last) {
    const cace_trace_t& tr = traces[t];
    const int64_t n = tr.n_requests, b = L.off[t];
    if (n > 0 && (!tr.arrival_time_s || !tr.model || !tr.prompt_tokens || !tr.output_tokens))
      throw Invalid{CACE_E_INVALID, "cace: trace arrays missing"};
    // run() resolves every request's model first (engine.cpp:87-92).
    for (int64_t i = 0; i < n; ++i) {
      const int m = tr.model[i];
      if (m < 0 || m >= M)
        throw Invalid{CACE_E_LOOKUP,
                      "catalog: no model registered for model index " + std::to_string(m)};
      if (!std::isfinite(tr.arrival_time_s[i]))
        throw Invalid{CACE_E_INVALID, "cace: non-finite arrival_time_s"};
      // parse_trace rejects negative arrivals (workload.cpp:245-248); the
      // kernels' sign-encoded slot times rely on a non-negative clock.
      if (tr.arrival_time_s[i] < 0)
        throw Invalid{CACE_E_INVALID, "cace: negative arrival_time_s"};
      if (tr.prompt_tokens[i] < 0)  // a negative prefill would run the event clock backwards
        throw Invalid{CACE_E_INVALID, "cace: negative prompt_tokens"};
      if (!(std::fabs(tr.arrival_time_s[i]) < 1e20))  // keeps every event time < 1e30
        throw Invalid{CACE_E_INVALID, "cace: |arrival_time_s| must be < 1e20"};
    }
    // Replay order = Arrival pop order (time, seq = index) (engine.cpp:49-55).
    std::vector<uint32_t> ord(n);
    std::iota(ord.begin(), ord.end(), 0u);
    bool sorted = true;
    for (int64_t i = 1; i < n && sorted; ++i)
      sorted = !(tr.arrival_time_s[i] < tr.arrival_time_s[i - 1]);
    if (!sorted)
      std::stable_sort(ord.begin(), ord.end(), [&](uint32_t x, uint32_t y) {
        return tr.arrival_time_s[x] < tr.arrival_time_s[y];
      });
    for (int m = 0; m < M; ++m) last[m] = (uint32_t)n;
    double worst = 0.0;
    uint32_t ncomp = 0;
    int bad = -1;
    for (int64_t k = n - 1; k >= 0; --k) {
      const uint32_t i = ord[k];
      const int m = tr.model[i];
      ReqRec& r = rec[b + k];
      r.arrival = tr.arrival_time_s[i];
      // service_times (engine.cpp:15-26)
      r.prefill = (double)tr.prompt_tokens[i] / cat.pr[m];
      r.decode = (double)std::max(tr.output_tokens[i], 1) / cat.dr[m];
      r.nxt = last[m];
      r.nxa = last[m] < (uint32_t)n ? rec[b + last[m]].arrival : INFINITY;
      r.mc = (uint32_t)m | ((uint32_t)(cat.cls[m] == CACE_REASONING) << 16);
      // same-class requests after k (turned into the class-local index below)
      r.ci = cat.cls[m] == CACE_REASONING ? (uint32_t)(n - 1 - k) - ncomp : ncomp;
      r.prv = 0xffffffffu;
      if (last[m] < (uint32_t)n) rec[b + last[m]].prv = (uint32_t)k;
      worst = std::max(worst, r.prefill + r.decode);
      last[m] = (uint32_t)k;
      L.perm[b + k] = i;
      ncomp += cat.cls[m] == CACE_REASONING ? 0u : 1u;
      if (cat.bad_rates(m)) bad = m;  // ends as the first in replay order
    }
    // class-local index (position among the same-class requests)
    const uint32_t nreas = (uint32_t)n - ncomp;
    for (int64_t k = 0; k < n; ++k) {
      ReqRec& r = rec[b + k];
      const bool reas = (r.mc >> 16) != 0;
      r.ci = (reas ? nreas : ncomp) - 1 - r.ci;
    }
    // per-trace results written once (no false sharing between threads)
    worst_t[t] = worst;
    L.ncomp[t] = ncomp;
    L.bad_model[t] = bad;
    for (int m = 0; m < M; ++m) L.first0[(size_t)t * M + m] = last[m];
  };
  const int nth = (int)std::min<int64_t>(
      {(int64_t)std::max(1u, std::thread::hardware_concurrency()), (int64_t)n_traces, (int64_t)32,
       std::max<int64_t>(1, N / 65536)});
  auto worker = [&](int w) {
    std::vector<uint32_t> last(M);
    for (int t = w; t < n_traces; t += nth) {
      try {
        one(t, last);
      } catch (const Invalid& x) {
        err_t[t] = 1;
        err_v[t] = x;
      }
    }
  };
  if (nth <= 1) {
    worker(0);
  } else {
    std::vector<std::thread> pool;
    for (int w = 0; w < nth; ++w) pool.emplace_back(worker, w);
    for (auto& th : pool) th.join();
  }
  for (int t = 0; t < n_traces; ++t)
    if (err_t[t]) throw err_v[t];
  // Event times stay < 1e30 (the kernels' fp32 screening relies on it): the
  // clock advances by at most one load (+ unload) and one service per request.
  double worst = 0.0;
  for (int m = 0; m < M; ++m) worst = std::max(worst, cat.lt[m]);
  for (int t = 0; t < n_traces; ++t) worst = std::max(worst, worst_t[t]);
  if (!(worst * (double)(N + 1) < 1e28))
    throw Invalid{CACE_E_INVALID, "cace: load/service times too large (event clock would exceed 1e28 s)"};
}

// Slots a replay can ever use: capacity = num_accelerators x
// models_per_accelerator (engine.cpp:83-84), clamped to the pool size M.  With
// capacity >= M a non-resident head always finds a free slot (at most M - 1
// other models are resident), so nothing is ever evicted and the replay -- every
// outcome, counter and max_resident -- is identical to capacity = M.
inline int64_t effective_capacity(const cace_scenario_t& sc, int M) {
  const int64_t cap = (int64_t)sc.num_accelerators * sc.models_per_accelerator;
  return cap < (int64_t)M ? cap : (int64_t)M;
}

// Reference run() preconditions (engine.cpp:79-92, 17-20) for one scenario:
// the SimError it would raise (code | model << 8), CACE_OK, or CACE_E_INVALID
// for inputs outside the engine's domain.
inline int32_t precheck(const HostLayout& L, const cace_scenario_t& sc) {
  if (sc.trace < 0 || sc.trace >= L.T) return CACE_E_INVALID;
  if (sc.variant < CACE_LRU || sc.variant > CACE_MINUS_P4) return CACE_E_INVALID;
  if (sc.window_length < 1) return CACE_E_WINDOW;
  if (sc.num_accelerators < 1) return CACE_E_ACCELERATORS;
  // A negative unload delay can schedule a LoadComplete before the current
  // event (time running backwards); the engine requires a monotone clock.
  if (!(sc.unload_time_s >= 0.0 && sc.unload_time_s < 1e15))
    return CACE_E_INVALID | (1 << 8);
  const int64_t n = L.off[sc.trace + 1] - L.off[sc.trace];
  if (n == 0) return CACE_OK;
  if (L.bad_model[sc.trace] >= 0) return CACE_E_RATES | (L.bad_model[sc.trace] << 8);
  const int64_t cap = (int64_t)sc.num_accelerators * sc.models_per_accelerator;
  if (cap < 1) return CACE_E_DEADLOCK;  // nothing can ever load (engine.cpp:235-237)
  if (effective_capacity(sc, L.M) > kMaxWarpC) return CACE_E_INVALID | (2 << 8);
  return CACE_OK;
}

inline std::string status_text(const HostCatalog& cat, int32_t status) {
  const int code = status & 0xff;
  const int m = status >> 8;
  switch (code) {
    case CACE_OK: return "";
    case CACE_E_WINDOW: return "run: window_length must be >= 1";
    case CACE_E_ACCELERATORS: return "run: need at least one accelerator";
    case CACE_E_RATES: return "service_times: rates must be positive for " + model_name(cat.ids, m);
    case CACE_E_CLOCK:
      return "eviction_score: clock precedes last_used_s for " + model_name(cat.ids, m);
    case CACE_E_DEADLOCK:
      return "run: deadlock \xe2\x80\x94 pending requests with no schedulable event";
    case CACE_E_RESIDENCY: return "run: residency bound violated";
    case CACE_E_METRICS_EMPTY: return "compute_run_metrics: empty report";
    case CACE_E_METRICS_NO_TTFT: return "compute_run_metrics: no completion outcomes for TTFT";
    case CACE_E_METRICS_NO_E2E: return "compute_run_metrics: no reasoning outcomes for E2E";
    default:
      if (code == CACE_E_INVALID && m == 1) return "cace: unload_time_s must be in [0, 1e15)";
      if (code == CACE_E_INVALID && m == 2) return "cace: capacity > 64 is not supported";
      return "cace: invalid scenario (bad trace index or variant)";
  }
}

}  // namespace cace
