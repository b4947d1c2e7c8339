// Policy-level kernels: one thread per independent instance.  These back the
// unit-parity entry points of include/cace_gpu.h (select_victim,
// eviction_score, dedup_window, service_times, log) and restate
// policy.cpp:22-115 / engine.cpp:15-26 for arbitrary inputs.
#pragma once
#include <stdint.h>

#include "../../include/cace_gpu.h"
#include "glibc_log.cuh"
#include "replay_lane.cuh"

namespace cace {

__global__ void fill_status_kernel(const int64_t* idx, const int32_t* code, int64_t n,
                                   cace_summary_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  cace_summary_t o;
  o.hits = o.misses = o.evictions = o.loads = 0;
  o.load_overhead_s = 0.0;
  o.max_resident = 0;
  o.status = code[i];
  o.n_completion = o.n_reasoning = 0;
  o.sum_ttft_completion = o.sum_e2e_reasoning = 0.0;
  o.max_ttft_completion = o.max_e2e_reasoning = 0.0;
  o.eviction_hash = CACE_HASH_SEED;
  o.outcome_hash = CACE_HASH_SEED;
  out[idx[i]] = o;
}

// eviction_score (policy.cpp:39-78) for one entry.  p3 from an explicit
// de-duplicated window list.  Returns false if clock < last_used (throws).
__device__ __forceinline__ bool score_entry(const DevCatalog& cat, int m, double last_used,
                                            const int32_t* win, int nwin, int wlen, double clock,
                                            const cace_scenario_t& pol, const double* tab,
                                            const double* tab2, int logv, double* parts) {
  if (clock < last_used) return false;
  const double d = clock - last_used;
  const double t = d < 1.0 ? 1.0 : d;
  const double p1v = 1.0 / (1.0 + cace_glibc_log(t, logv, tab, tab2));
  double p1 = pol.p1_mode == CACE_P1_VERBATIM ? p1v : 1.0 - p1v;
  double p2 = __ldg(cat.p2 + m);
  double p3 = 1.0;
  for (int k = 0; k < nwin; ++k)
    if (win[k] == m) {
      p3 = (double)k / (double)wlen;
      break;
    }
  double p4 = pol.w1 * (__ldg(cat.tokens + m) / (double)pol.output_token_normalizer);
  switch (pol.variant) {
    case CACE_MINUS_P1: p1 = 0.0; break;
    case CACE_MINUS_P2: p2 = 0.0; break;
    case CACE_MINUS_P3: p3 = 0.0; break;
    case CACE_MINUS_P4: p4 = 0.0; break;
    default: break;
  }
  parts[0] = p1;
  parts[1] = p2;
  parts[2] = p3;
  parts[3] = p4;
  parts[4] = ((p1 + p2) + p3) + p4;
  return true;
}

__global__ void eviction_score_kernel(DevCatalog cat, int64_t n, const int32_t* model,
                                      const double* last_used, int max_window,
                                      const int32_t* n_window, const int32_t* window_models,
                                      const double* clock, const cace_scenario_t* pol,
                                      const double* tab, const double* tab2, int logv,
                                      double* out, int32_t* status) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n) return;
  const cace_scenario_t p = pol[b];
  double parts[5] = {0, 0, 0, 0, 0};
  const bool ok = score_entry(cat, model[b], last_used[b], window_models + b * max_window,
                              n_window[b], p.window_length, clock[b], p, tab, tab2, logv, parts);
  for (int k = 0; k < 5; ++k) out[5 * b + k] = parts[k];
  status[b] = ok ? CACE_OK : CACE_E_CLOCK;
}

// select_victim (policy.cpp:80-115): idle entries sorted by (last_used,
// model_id); LRU -> front; CACE -> first strict max of total in that order.
__global__ void select_victim_kernel(DevCatalog cat, int64_t n, int max_entries,
                                     const int32_t* n_entries, const int32_t* entry_model,
                                     const double* entry_lu, const uint8_t* entry_busy,
                                     int max_window, const int32_t* n_window,
                                     const int32_t* window_models, const double* clock,
                                     const cace_scenario_t* pol, const double* tab,
                                     const double* tab2, int logv, int32_t* victim,
                                     int32_t* status) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n) return;
  const cace_scenario_t p = pol[b];
  const int ne = n_entries[b];
  const int32_t* em = entry_model + b * max_entries;
  const double* lu = entry_lu + b * max_entries;
  const uint8_t* busy = entry_busy + b * max_entries;
  status[b] = CACE_OK;
  // Selection sort by (last_used, lex) over idle entries — ne is tiny.
  int order[64];
  int k = 0;
  for (int e = 0; e < ne && k < 64; ++e)
    if (!busy[e]) order[k++] = e;
  for (int i = 0; i < k; ++i)
    for (int j = i + 1; j < k; ++j) {
      const int a = order[i], c = order[j];
      const bool less = lu[c] < lu[a] || (!(lu[a] < lu[c]) && __ldg(cat.lex + em[c]) < __ldg(cat.lex + em[a]));
      if (less) {
        order[i] = c;
        order[j] = a;
      }
    }
  if (k == 0) {
    victim[b] = -1;
    return;
  }
  if (p.variant == CACE_LRU) {
    victim[b] = em[order[0]];
    return;
  }
  int best = -1;
  double bt = 0.0;
  for (int i = 0; i < k; ++i) {
    const int e = order[i];
    double parts[5];
    if (!score_entry(cat, em[e], lu[e], window_models + b * max_window, n_window[b],
                     p.window_length, clock[b], p, tab, tab2, logv, parts)) {
      status[b] = CACE_E_CLOCK | (em[e] << 8);
      victim[b] = -1;
      return;
    }
    if (best < 0 || parts[4] > bt) {
      best = e;
      bt = parts[4];
    }
  }
  victim[b] = em[best];
}

// dedup_window (policy.cpp:22-37): first occurrences of pending[0..min(n,len)).
__global__ void dedup_window_kernel(int64_t n, int max_pending, const int32_t* n_pending,
                                    const int32_t* pending, const int32_t* length, int32_t* out,
                                    int32_t* n_out) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n) return;
  const int np = n_pending[b];
  const int lim = np < length[b] ? np : length[b];
  const int32_t* pm = pending + b * max_pending;
  int32_t* o = out + b * max_pending;
  int k = 0;
  for (int i = 0; i < lim; ++i) {
    bool seen = false;
    for (int j = 0; j < k && !seen; ++j) seen = o[j] == pm[i];
    if (!seen) o[k++] = pm[i];
  }
  n_out[b] = k;
}

// service_times (engine.cpp:15-26).
__global__ void service_times_kernel(int64_t n, const int32_t* model, const int32_t* prompt,
                                     const int32_t* output, const double* prefill_rate,
                                     const double* decode_rate, double* pf, double* dc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int m = model[i];
  pf[i] = (double)prompt[i] / prefill_rate[m];
  const int o = output[i] > 1 ? output[i] : 1;
  dc[i] = (double)o / decode_rate[m];
}

__global__ void log_kernel(int64_t n, const double* x, int variant, const double* tab,
                           const double* tab2, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = cace_glibc_log(x[i], variant, tab, tab2);
}

}  // namespace cace
