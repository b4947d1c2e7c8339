// Warp-per-scenario trace-replay kernel (sm_100a) for large model pools and
// capacities (BASELINE config 5: 256 CodeLLMs, capacity ~32, window 1024).
//
// Same request-synchronous event algebra as replay_lane.cuh (see its file
// comment for why request k can be processed in one step), but one WARP
// replays one scenario: lane l owns slots l, l+32, ... (SPL slots per lane),
// so every per-slot scan of the lane kernel becomes one predicate per lane
// plus a ballot or a shuffle reduction:
//   * classification: ballot(slot model == head model);
//   * bulk completion updates: each lane updates its own slots;
//   * all-busy case: warp arg-min of (done, seq) over busy slots;
//   * eviction decision: every idle candidate's exact fp64 eviction_score
//     (policy.cpp:39-78, glibc-log P1) is computed by its owner lane in
//     parallel, then "first strict max in (last_used, model_id) order"
//     (policy.cpp:92-113) is a warp reduction (no fp32 screening needed).
// The lookahead window: first[m] and the arrival time of that request live in
// shared memory per warp.  For windows of <= 1024 requests the ranks come
// from a sliding 1024-bit map of "first pending occurrence" positions (lane l
// holds positions k + 32 l .. k + 32 l + 31; one funnel shift per request),
// so rank(m) = popcount of the map below first[m] is a warp prefix sum at
// decision time and nothing per model is touched per request.  Longer
// windows keep explicit ranks advanced cooperatively (lanes stride over
// models, ballot/popc).
// Scenario-level state (cursor, counters, fingerprints) is warp-uniform:
// every lane computes it identically; lane 0 writes the summary.
#pragma once
#include <math.h>
#include <stdint.h>

#include "../../include/cace_gpu.h"
#include "glibc_log.cuh"
#include "replay_lane.cuh"
#include "replay_types.h"

namespace cace {

constexpr int WARP_BLOCK = 128;  // 4 scenarios per block
// catalog columns at the start of the warp kernel's shared memory (8-aligned)
inline __host__ __device__ size_t warp_smem_cat(int M) { return ((size_t)M * (3 * 8 + 4) + 7) & ~(size_t)7; }

// Order-preserving unsigned key of a non-NaN double (-0.0 folded onto +0.0,
// which compare equal in the reference's doubles).
__device__ __forceinline__ uint64_t okey(double d) {
  const uint64_t u = (uint64_t)__double_as_longlong(d + 0.0);
  return (u >> 63) ? ~u : (u | (1ull << 63));
}

// Warp-wide max of a 64-bit key with two 32-bit redux.sync reductions.
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t k) {
  const uint32_t hi = __reduce_max_sync(kFull, (uint32_t)(k >> 32));
  const uint32_t lo = __reduce_max_sync(kFull, (uint32_t)(k >> 32) == hi ? (uint32_t)k : 0u);
  return ((uint64_t)hi << 32) | lo;
}

// (d, q) < (d2, q2) lexicographically
__device__ __forceinline__ bool key_lt(double d, uint32_t q, double d2, uint32_t q2) {
  return d < d2 || (d == d2 && q < q2);
}

template <int SPL, bool DUMP>
__global__ void __launch_bounds__(WARP_BLOCK) replay_warp_kernel(ReplayParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int M = P.cat.M;
  double* s_lt = reinterpret_cast<double*>(smem);
  double* s_p2 = s_lt + M;
  double* s_tok = s_p2 + M;
  int* s_lex = reinterpret_cast<int*>(s_tok + M);
  double* wfa = reinterpret_cast<double*>(smem + warp_smem_cat(M));  // [4][M] arrival of first[m]
  double* wp4 = wfa + (size_t)(WARP_BLOCK / 32) * M;                  // [4][M] exact p4 of model m
  uint32_t* wfirst = reinterpret_cast<uint32_t*>(wp4 + (size_t)(WARP_BLOCK / 32) * M);  // [4][M]
  uint32_t* wrank = wfirst + (size_t)(WARP_BLOCK / 32) * M;   // [4][M]
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    s_lt[m] = P.cat.load_time[m];
    s_p2[m] = P.cat.p2[m];
    s_tok[m] = P.cat.tokens[m];
    s_lex[m] = P.cat.lex[m];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t gi = P.seg_begin + (int64_t)blockIdx.x * (WARP_BLOCK / 32) + warp;
  if (gi >= P.seg_end) return;  // whole warp
  const int64_t sidx = (int64_t)((uint64_t)P.order[gi] & (kShadowBit - 1));
  const cace_scenario_t sc = P.scen[sidx];
  const int64_t base = P.trace_off[sc.trace];
  const uint32_t n = (uint32_t)(P.trace_off[sc.trace + 1] - base);
  const ReqRec* tr = P.rec + base;
  const int C = (int)min((int64_t)sc.num_accelerators * sc.models_per_accelerator, (int64_t)M);  // effective_capacity
  const int variant = sc.variant;
  const bool is_lru = variant == CACE_LRU;
  const bool need_win = !is_lru && variant != CACE_MINUS_P3;
  const bool verbatim = sc.p1_mode == CACE_P1_VERBATIM;
  const uint32_t w = (uint32_t)sc.window_length;
  const double wd = (double)sc.window_length;
  const double norm = (double)sc.output_token_normalizer;
  uint32_t* first = wfirst + (size_t)warp * M;
  uint32_t* rank = wrank + (size_t)warp * M;
  double* fa = wfa + (size_t)warp * M;
  double* p4t = wp4 + (size_t)warp * M;
  // exact p4 of every model (policy.cpp:66-67), once per scenario
  for (int m = lane; m < M; m += 32) p4t[m] = variant == CACE_MINUS_P4 ? 0.0 : sc.w1 * (s_tok[m] / norm);
  __syncwarp();  // the table is read by every lane's decisions
  const bool bitmap = need_win && w <= 1024;  // rank from the first-occurrence map
  uint32_t fo = 0;  // this lane's 32 positions of the map

  int dslot = -1;
  int64_t doff = 0, dn_ev = 0;
  if (DUMP) {
    dslot = P.dump.slot[sidx];
    if (dslot >= 0) doff = P.dump.dump_off[dslot];
  }
  if (need_win) {
    const uint32_t* f0 = P.first0 + (int64_t)sc.trace * M;
    for (int m = lane; m < M; m += 32) {
      first[m] = __ldg(f0 + m);
      fa[m] = first[m] < n ? __ldg(&tr[first[m]].arrival) : INFINITY;
    }
    __syncwarp();
    if (bitmap) {
      // positions [0, 1024): first occurrences in the trace
      for (int b = 0; b < 32; ++b) {
        const uint32_t pos = 32u * lane + b;
        if (pos < n && __ldg(&tr[pos].prv) == 0xffffffffu) fo |= 1u << b;
      }
    } else {
      for (int m = lane; m < M; m += 32) {
        const uint32_t fm = first[m];
        uint32_t c = 0;
        for (int q = 0; q < M; ++q) c += first[q] < fm ? 1u : 0u;
        rank[m] = c;
      }
    }
    __syncwarp();
  }

  // Slots owned by this lane: global slot id g = lane + 32 j.
  int smodel[SPL], slex[SPL];
  bool sbusy[SPL], svalid[SPL];
  double stime[SPL];  // busy: ServiceComplete time; idle: last_used (same value once applied)
  uint32_t sseq[SPL];
#pragma unroll
  for (int j = 0; j < SPL; ++j) {
    smodel[j] = -1;
    slex[j] = 0;
    sbusy[j] = false;
    svalid[j] = lane + 32 * j < C;
    stime[j] = 0.0;
    sseq[j] = 0;
  }
  int occ = 0;
  uint32_t seqc = 0;
  Cursor cur{-INFINITY, 2, 0};
  uint32_t hits = 0, evictions = 0, loads = 0, nc = 0, nr = 0;
  double lo_sum = 0.0, sttft = 0.0, se2e = 0.0, mttft = 0.0, me2e = 0.0;
  uint64_t ho = CACE_HASH_SEED, he = CACE_HASH_SEED;

  double na = 0.0, npf = 0.0, ndc = 0.0;
  uint32_t nnxt = 0, nmc = 0;
  if (n > 0) load_rec(tr, na, npf, ndc, nnxt, nmc);
  uint32_t eprv_next = (bitmap && 1024 < n) ? __ldg(&tr[1024].prv) : 0u;
  for (uint32_t k = 0; k < n; ++k) {
    const double a = na, pf = npf, dc = ndc;
    const uint32_t nxt = nnxt, mc = nmc;
    if (k + 1 < n) load_rec(tr + k + 1, na, npf, ndc, nnxt, nmc);
    // window maintenance inputs, needed only at the end of the iteration;
    // the entering position's prv (1024 requests ahead: an L2/DRAM load) is
    // fetched one iteration early
    double nxa = 0.0;
    const uint32_t eprv = eprv_next;
    if (need_win) {
      nxa = __ldg(&tr[k].nxa);
      if (bitmap && k + 1025 < n) eprv_next = __ldg(&tr[k + 1025].prv);
    }
    const int m = (int)(mc & 0xffffu);

    if (!(a < cur.t)) {  // head's Arrival into an empty queue
#pragma unroll
      for (int j = 0; j < SPL; ++j)
        if (sbusy[j] && stime[j] <= a) {
          sbusy[j] = false;
        }
      cur = Cursor{a, 2, k};
    }
    // classify: which (lane, j) holds the head's model
    int hs = -1;  // global slot id
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
      const unsigned b = __ballot_sync(kFull, smodel[j] == m);
      if (b) hs = (__ffs(b) - 1) + 32 * j;
    }
    double lw = 0.0;
    const bool hit = hs >= 0;
    if (hit) {
      ++hits;
      const int ol = hs & 31, oj = hs >> 5;
      bool hb = false;
      double td = 0.0;
      uint32_t tq = 0;
#pragma unroll
      for (int j = 0; j < SPL; ++j) {
        const bool b = __shfl_sync(kFull, sbusy[j], ol);
        const double d = __shfl_sync(kFull, stime[j], ol);
        const uint32_t q = __shfl_sync(kFull, sseq[j], ol);
        if (j == oj) {
          hb = b;
          td = d;
          tq = q;
        }
      }
      if (hb) {  // blocked until the model's own ServiceComplete
        cur = Cursor{td, 1, tq};
#pragma unroll
        for (int j = 0; j < SPL; ++j)
          if (sbusy[j] && sc_le(stime[j], sseq[j], cur)) {
            sbusy[j] = false;
          }
      }
    } else {
      int v;  // victim / target global slot id
      double ud = 0.0;
      if (occ < C) {
        v = occ++;
      } else {
        int nidle = 0, one = -1;
#pragma unroll
        for (int j = 0; j < SPL; ++j) {
          const unsigned b = __ballot_sync(kFull, svalid[j] && !sbusy[j]);
          nidle += __popc(b);
          if (b) one = (__ffs(b) - 1) + 32 * j;
        }
        if (nidle == 0) {
          // all busy: min-key ServiceComplete (warp arg-min over (done, seq))
          double bd = INFINITY;
          uint32_t bq = 0xffffffffu;
          int bg = -1;
#pragma unroll
          for (int j = 0; j < SPL; ++j)
            if (svalid[j] && key_lt(stime[j], sseq[j], bd, bq)) {
              bd = stime[j];
              bq = sseq[j];
              bg = lane + 32 * j;
            }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            const double od = __shfl_xor_sync(kFull, bd, off);
            const uint32_t oq = __shfl_xor_sync(kFull, bq, off);
            const int og = __shfl_xor_sync(kFull, bg, off);
            if (key_lt(od, oq, bd, bq)) {
              bd = od;
              bq = oq;
              bg = og;
            }
          }
          v = bg;
#pragma unroll
          for (int j = 0; j < SPL; ++j)
            if (lane + 32 * j == v) sbusy[j] = false;
          cur = Cursor{bd, 1, bq};
        } else if (nidle == 1) {
          v = one;
        } else {
          // ---- eviction decision: each lane scores its idle slots ----
          const double now = cur.t;
          // window position of each own slot's model (policy.cpp:57-64):
          // rank when its first pending request is in [k, min(k + w,
          // arrived)), else -1 (collective: the map prefix is warp-wide)
          int wrk[SPL];
          uint32_t excl = 0;
          if (bitmap) {
            const uint32_t pc = __popc(fo);
            uint32_t incl = pc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t y = __shfl_up_sync(kFull, incl, o);
              if (lane >= o) incl += y;
            }
            excl = incl - pc;
          }
#pragma unroll
          for (int j = 0; j < SPL; ++j) {
            wrk[j] = -1;
            const bool cand = need_win && svalid[j] && !sbusy[j];
            const int ms = cand ? smodel[j] : 0;
            const uint32_t fm = cand ? first[ms] : k;
            const bool iw = cand && fm - k < w && fa[ms] < now;
            if (bitmap) {
              const uint32_t d = iw ? fm - k : 0u;  // < 1024
              const uint32_t wl = __shfl_sync(kFull, fo, (int)(d >> 5));
              const uint32_t el = __shfl_sync(kFull, excl, (int)(d >> 5));
              if (iw) wrk[j] = (int)(el + __popc(wl & ((1u << (d & 31u)) - 1u)));
            } else if (iw) {
              wrk[j] = (int)rank[ms];
            }
          }
          // Per lane: the best own candidate by (total desc, last_used asc,
          // lex asc) over non-NaN totals, its own sorted-first by
          // (last_used, lex), and whether any own total is NaN.
          double bt = 0.0, blu = 0.0, flu = 0.0;
          int blex = 0, bj = -1, flex = 0, fj = -1;
          bool has_nan = false;
          bool tnan[SPL];
#pragma unroll
          for (int j = 0; j < SPL; ++j) {
            tnan[j] = false;
            if (!(svalid[j] && !sbusy[j])) continue;
            if (fj < 0 || stime[j] < flu || (stime[j] == flu && slex[j] < flex)) {
              flu = stime[j];
              flex = slex[j];
              fj = j;
            }
            if (is_lru) continue;
            const int ms = smodel[j];
            double p1 = 0.0;
            if (variant != CACE_MINUS_P1) {
              const double d = now - stime[j];
              const double t = d < 1.0 ? 1.0 : d;
              const double lg = t == 1.0 ? 0.0 : cace_glibc_log(t, P.log_variant, P.log_tab, P.log_tab2);
              const double p1v = 1.0 / (1.0 + lg);
              p1 = verbatim ? p1v : 1.0 - p1v;
            }
            const double p2 = variant == CACE_MINUS_P2 ? 0.0 : s_p2[ms];
            double p3 = 0.0;
            if (variant != CACE_MINUS_P3) {
              p3 = 1.0;
              if (wrk[j] >= 0) p3 = (double)wrk[j] / wd;
            }
            const double p4 = p4t[ms];
            const double T = ((p1 + p2) + p3) + p4;
            tnan[j] = T != T;
            has_nan |= tnan[j];
            if (T == T && (bj < 0 || T > bt ||
                           (T == bt && (stime[j] < blu || (stime[j] == blu && slex[j] < blex))))) {
              bt = T;
              blu = stime[j];
              blex = slex[j];
              bj = j;
            }
          }
          // Sorted-first across the warp: min (last_used, lex) via redux.
          auto sorted_first = [&]() {
            const uint64_t kl = fj >= 0 ? ~okey(flu) : 0ull;  // max of ~key = min of key
            const uint64_t mx = warp_max_u64(kl);
            const bool tie = fj >= 0 && kl == mx;
            const uint32_t lx = __reduce_min_sync(kFull, tie ? (uint32_t)flex : 0xffffffffu);
            const unsigned who = __ballot_sync(kFull, tie && (uint32_t)flex == lx);
            const int ol = __ffs(who) - 1;
            return ol + 32 * __shfl_sync(kFull, fj, ol);
          };
          if (is_lru) {
            v = sorted_first();
          } else {
            // first strict max in sorted order (policy.cpp:102-113) = max
            // non-NaN total, ties to the smaller (last_used, lex) ...
            const uint64_t kt = bj >= 0 ? okey(bt) : 0ull;
            const uint64_t mt = warp_max_u64(kt);
            unsigned tied = __ballot_sync(kFull, bj >= 0 && kt == mt);
            if (tied & (tied - 1u)) {  // exact tie across lanes (rare)
              const bool in = (tied >> lane) & 1u;
              const uint64_t kl = in ? ~okey(blu) : 0ull;
              const uint64_t mx = warp_max_u64(kl);
              const bool t2 = in && kl == mx;
              const uint32_t lx = __reduce_min_sync(kFull, t2 ? (uint32_t)blex : 0xffffffffu);
              tied = __ballot_sync(kFull, t2 && (uint32_t)blex == lx);
            }
            const int ol = __ffs(tied) - 1;
            v = ol + 32 * __shfl_sync(kFull, bj, ol);
            // ... unless the sorted-first entry's total is NaN: it keeps the slot.
            if (__any_sync(kFull, has_nan)) {
              const int f = sorted_first();
              bool fn = false;
#pragma unroll
              for (int j = 0; j < SPL; ++j)
                if (lane + 32 * j == f) fn = tnan[j];
              if (__any_sync(kFull, fn)) v = f;
            }
          }
        }
        // evict v (engine.cpp:205-206)
        int vm = 0;
#pragma unroll
        for (int j = 0; j < SPL; ++j) {
          const int mm = __shfl_sync(kFull, smodel[j], v & 31);
          if ((v >> 5) == j) vm = mm;
        }
        ++evictions;
        he = hmix(he, dbits(cur.t) ^ ((uint64_t)vm << 32));
        if (DUMP && dslot >= 0 && lane == 0) {
          if (dn_ev < P.dump.evict_cap) {
            if (P.dump.evict_model) P.dump.evict_model[dslot * P.dump.evict_cap + dn_ev] = vm;
            if (P.dump.evict_clock) P.dump.evict_clock[dslot * P.dump.evict_cap + dn_ev] = cur.t;
          }
        }
        ++dn_ev;
        ud = sc.unload_time_s;
      }
      // start_load (engine.cpp:123-132) then wait for LoadComplete (r, 0, .)
      const double lt = s_lt[m];
      const double r = (cur.t + ud) + lt;
      lw = r - cur.t;
      lo_sum += lt;
      ++loads;
#pragma unroll
      for (int j = 0; j < SPL; ++j) {
        if (lane + 32 * j == v) {
          smodel[j] = m;
          slex[j] = s_lex[m];
          sbusy[j] = false;
        }
        if (sbusy[j] && stime[j] < r) {
          sbusy[j] = false;
        }
      }
      cur = Cursor{r, 0, 0};
      hs = v;
    }

    // start_service at now = cur.t (engine.cpp:134-153)
    const double now = cur.t;
    const double qd = now - a;
    const double ttft = qd + pf;
    const double e2e = ttft + dc;
    const double done = (now + pf) + dc;
#pragma unroll
    for (int j = 0; j < SPL; ++j)
      if (lane + 32 * j == hs) {
        sbusy[j] = true;
        stime[j] = done;
        sseq[j] = seqc;
      }
    ++seqc;
    if ((mc >> 16) == CACE_COMPLETION) {
      ++nc;
      sttft += ttft;
      mttft = ttft > mttft ? ttft : mttft;
    } else {
      ++nr;
      se2e += e2e;
      me2e = e2e > me2e ? e2e : me2e;
    }
    ho = hmix(ho, dbits(ttft) ^ (hit ? 0ull : 1ull));
    if (DUMP && dslot >= 0 && lane == 0) {
      const int64_t o = doff + P.perm[base + k];
      if (P.dump.cold) P.dump.cold[o] = hit ? 0 : 1;
      if (P.dump.queue_wait) P.dump.queue_wait[o] = qd - lw;
      if (P.dump.load_wait) P.dump.load_wait[o] = lw;
      if (P.dump.prefill) P.dump.prefill[o] = pf;
      if (P.dump.decode) P.dump.decode[o] = dc;
      if (P.dump.ttft) P.dump.ttft[o] = ttft;
      if (P.dump.e2e) P.dump.e2e[o] = e2e;
      if (P.dump.samples) {  // metrics samples, as in the lane kernel
        const bool comp = (mc >> 16) == CACE_COMPLETION;
        P.dump.samples[doff + (comp ? nc - 1 : P.trace_ncomp[sc.trace] + nr - 1)] = comp ? ttft : e2e;
      }
    }
    if (bitmap) {
      // the window slides to k + 1: position k leaves, k + 1024 enters (a
      // first occurrence iff its model's previous request is <= k), and the
      // head's model's next request becomes its first pending occurrence
      const uint32_t nw = __shfl_down_sync(kFull, fo, 1);
      fo = __funnelshift_r(fo, lane == 31 ? 0u : nw, 1);
      if (lane == 31 && k + 1024 < n && eprv + 1u <= k + 1u) fo |= 1u << 31;
      const uint32_t dj = nxt - (k + 1);
      if (nxt < n && dj < 1024u && (int)(dj >> 5) == lane) fo |= 1u << (dj & 31u);
      __syncwarp();
      if (lane == 0) {
        first[m] = nxt;
        fa[m] = nxa;
      }
      __syncwarp();
    } else if (need_win) {  // window advance: lanes stride over the models
      __syncwarp();
      uint32_t cnt = 0;
      for (int b0 = 0; b0 < M; b0 += 32) {
        const int jm = b0 + lane;
        const bool before = jm < M && jm != m && first[jm] < nxt;
        cnt += __popc(__ballot_sync(kFull, before));
        if (before) rank[jm] -= 1;
      }
      __syncwarp();
      if (lane == 0) {
        first[m] = nxt;
        rank[m] = cnt;
        fa[m] = nxa;
      }
      __syncwarp();
    }
  }

  if (lane != 0) return;
  cace_summary_t o;
  o.hits = hits;
  o.misses = n - hits;
  o.evictions = evictions;
  o.loads = loads;
  o.load_overhead_s = lo_sum;
  o.max_resident = occ;
  o.status = CACE_OK;
  o.n_completion = nc;
  o.n_reasoning = nr;
  o.sum_ttft_completion = sttft;
  o.sum_e2e_reasoning = se2e;
  o.max_ttft_completion = mttft;
  o.max_e2e_reasoning = me2e;
  o.eviction_hash = he;
  o.outcome_hash = ho;
  P.out[sidx] = o;
  if (DUMP && dslot >= 0 && P.dump.n_evict) P.dump.n_evict[dslot] = dn_ev;
}

inline size_t warp_smem_bytes(int M) {
  return warp_smem_cat(M) + (size_t)(WARP_BLOCK / 32) * M * (8 + 8 + 4 + 4);
}

}  // namespace cace
