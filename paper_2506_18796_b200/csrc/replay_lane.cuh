// Lane-per-scenario trace-replay kernel (sm_100a).
//
// One thread replays one scenario = one reference run(trace, catalog,
// cluster, policy) (engine.cpp:76-239 + policy.cpp:22-115), bit-exact.
// Lanes of a warp replay scenarios of the same trace and capacity (the host
// plan groups them), so they read the same request records; the trace is
// L2-resident and each request record is one 32-B sector.
//
// Event model (exactly the reference's min-heap order (time, kind, seq),
// engine.cpp:49-55, without a heap):
//   * at most ONE LoadComplete is ever in flight (only the queue head starts
//     loads and it stays head until served), kind 0;
//   * one ServiceComplete per Busy slot, kind 1, seq = service-start order;
//   * Arrivals, kind 2, in (time, index) order.  An Arrival into a non-empty
//     queue cannot change any dispatch decision (the head was already
//     examined and nothing it waits on changed), so only the arrival of the
//     head into an EMPTY queue is processed as an event; every other request
//     j > head counts as arrived at event time `now` iff a[j] < now.
//   * The pending queue is the contiguous sorted range [head, arrived), so
//     the lookahead window is [head, min(head + w, arrived)) and needs no
//     storage: first[m] (first index >= head requesting model m) is kept per
//     lane in shared memory and rank(m) = #{m' : first[m'] < first[m]}
//     (dedup_window, policy.cpp:22-37).
//   * All fp64 arithmetic uses the reference's operation order with no
//     contraction (built with -fmad=false); P1's log is the glibc
//     restatement (glibc_log.cuh).
#pragma once
#include <stdint.h>

#include "../../include/cace_gpu.h"
#include "glibc_log.cuh"

namespace cace {

enum : int { ST_IDLE = 0, ST_BUSY = 1, ST_LOADING = 2 };

// One request in replay (sorted) order.  32 B = one sector: a lane advancing
// its queue head fetches exactly one sector (two 128-bit loads).
struct __align__(32) ReqRec {
  double arrival;  // Request::arrival_time_s
  double prefill;  // service_times(): prompt / prefill_rate   (engine.cpp:21-22)
  double decode;   // service_times(): max(out,1) / decode_rate (engine.cpp:23-24)
  uint32_t nxt;    // next sorted index with the same model (n if none)
  uint32_t mc;     // model | task_class << 16
};

struct DevCatalog {
  int M;
  const double* load_time;  // [M] ModelDescriptor::load_time_s
  const double* p2;         // [M] 1 / (1 + load_time / 100)  (policy.cpp:55)
  const double* tokens;     // [M] (double) expected_output_tokens
  const int* lex;           // [M] rank of model_id under std::string <
};

struct DumpDev {
  const int32_t* slot;  // [n_scenarios] dump slot or -1; NULL = no dump
  const int64_t* dump_off;  // [n_dump] offset of slot's per-request block
  uint8_t* cold;
  double *queue_wait, *load_wait, *prefill, *decode, *ttft, *e2e;
  int64_t evict_cap;
  int32_t* evict_model;
  double* evict_clock;
  int64_t* n_evict;
};

struct ReplayParams {
  const ReqRec* rec;        // all traces, concatenated, sorted order
  const int64_t* trace_off; // [T+1]
  const uint32_t* first0;   // [T][M] first sorted index of each model
  const uint32_t* perm;     // sorted index -> caller's request index
  DevCatalog cat;
  const double* log_tab;
  const double* log_tab2;
  int log_variant;
  const cace_scenario_t* scen;
  const int64_t* order;     // plan: scenario indices grouped by capacity
  int64_t seg_begin, seg_end;
  cace_summary_t* out;
  DumpDev dump;
};

__device__ __forceinline__ uint64_t hmix(uint64_t h, uint64_t x) {
  h ^= x;
  h *= CACE_HASH_MUL;
  return h ^ (h >> 31);
}
__device__ __forceinline__ uint64_t dbits(double d) { return (uint64_t)__double_as_longlong(d); }

__device__ __forceinline__ void load_rec(const ReqRec* p, double& a, double& pf, double& dc,
                                         uint32_t& nxt, uint32_t& mc) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
  const uint4 q0 = __ldg(q);
  const uint4 q1 = __ldg(q + 1);
  a = __hiloint2double((int)q0.y, (int)q0.x);
  pf = __hiloint2double((int)q0.w, (int)q0.z);
  dc = __hiloint2double((int)q1.y, (int)q1.x);
  nxt = q1.z;
  mc = q1.w;
}

// Per-lane replay state for one scenario.  Template C = capacity (slots):
// the slot arrays live in registers with fully unrolled scans.
template <int C>
struct Lane {
  // slots: model | state << 16, last_used, ServiceComplete time + push seq
  int sms[C];
  double slu[C], sdone[C];
  uint32_t sseq[C];
  int occ;
  int ls;          // slot with the in-flight load (-1 none)
  double lready;   // its LoadComplete time
  uint32_t seqc;   // ServiceComplete push order
  // queue head (first unserved request, replay order)
  uint32_t head;
  double ha, hpf, hdc, hlw;
  uint32_t hnxt, hmc;
  bool hc, hcold, harr;
  double now;
  // results
  uint32_t hits, misses, evictions, loads, nc, nr;
  double lo_sum, sttft, se2e, mttft, me2e;
  uint64_t ho, he;
  int status;
};

// Slot word: model (bits 0-15) | state (16-17) | lex rank of model_id (18-31).
__device__ __forceinline__ int slot_model(int v) { return v & 0xffff; }
__device__ __forceinline__ int slot_state(int v) { return (v >> 16) & 3; }
__device__ __forceinline__ int slot_lex(int v) { return (int)((unsigned)v >> 18); }
__device__ __forceinline__ int with_state(int v, int st) { return (v & ~(3 << 16)) | (st << 16); }

// start_load (engine.cpp:123-132): the head's model into `target`.
template <int C>
__device__ __forceinline__ void start_load(Lane<C>& L, int target, double udelay, const double* s_lt,
                                           const int* s_lex) {
  const int hm = (int)(L.hmc & 0xffffu);
  const double lt = s_lt[hm];
  const double ready = (L.now + udelay) + lt;
  L.hlw = ready - L.now;
  L.lo_sum += lt;
  ++L.loads;
#pragma unroll
  for (int s = 0; s < C; ++s)
    if (s == target) {
      L.sms[s] = hm | (ST_LOADING << 16) | (s_lex[hm] << 18);
      L.slu[s] = L.now;
    }
  L.ls = target;
  L.lready = ready;
}

// Replays one scenario.  Two phases per iteration so the expensive part runs
// converged across the warp:
//   A (divergent, cheap): events + head-of-line dispatch (hits, service
//     starts, free-slot loads) until the lane reaches an eviction decision
//     or finishes;
//   B (converged): the eviction decision — victim selection over the idle
//     residents (policy.cpp:80-115) and the load that follows.
// first/p4 are this lane's shared-memory columns (element m at [m*stride]).
template <int C, bool DUMP>
__device__ void replay_scenario(const ReplayParams& P, int64_t sidx, uint32_t* first,
                                double* p4tab, int stride, const double* s_lt,
                                const double* s_p2, const int* s_lex) {
  const cace_scenario_t sc = P.scen[sidx];
  const int M = P.cat.M;
  const int64_t base = P.trace_off[sc.trace];
  const uint32_t n = (uint32_t)(P.trace_off[sc.trace + 1] - base);
  const ReqRec* tr = P.rec + base;
  const int variant = sc.variant;
  const bool is_lru = variant == CACE_LRU;
  const bool need_win = !is_lru && variant != CACE_MINUS_P3;
  const bool verbatim = sc.p1_mode == CACE_P1_VERBATIM;
  const uint32_t w = (uint32_t)sc.window_length;
  const double wd = (double)sc.window_length;

  int dslot = -1;
  int64_t doff = 0, dn_ev = 0;
  if (DUMP) {
    dslot = P.dump.slot[sidx];
    if (dslot >= 0) doff = P.dump.dump_off[dslot];
  }

  if (need_win) {
    const uint32_t* f0 = P.first0 + (int64_t)sc.trace * M;
    for (int m = 0; m < M; ++m) first[m * stride] = __ldg(f0 + m);
  }
  if (!is_lru) {
    // p4 = w1 * (tokens / normalizer)   (policy.cpp:66-67)
    const double norm = (double)sc.output_token_normalizer;
    for (int m = 0; m < M; ++m) p4tab[m * stride] = sc.w1 * (__ldg(P.cat.tokens + m) / norm);
  }

  Lane<C> L;
#pragma unroll
  for (int s = 0; s < C; ++s) {
    L.sms[s] = 0xffff;  // empty
    L.slu[s] = 0.0;
    L.sdone[s] = 0.0;
    L.sseq[s] = 0;
  }
  L.occ = 0;
  L.ls = -1;
  L.lready = 0.0;
  L.seqc = 0;
  L.head = 0;
  L.ha = L.hpf = L.hdc = L.hlw = 0.0;
  L.hnxt = L.hmc = 0;
  L.hc = L.hcold = L.harr = false;
  L.now = 0.0;
  L.hits = L.misses = L.evictions = L.loads = L.nc = L.nr = 0;
  L.lo_sum = L.sttft = L.se2e = L.mttft = L.me2e = 0.0;
  L.ho = L.he = CACE_HASH_SEED;
  L.status = CACE_OK;
  if (n > 0) load_rec(tr, L.ha, L.hpf, L.hdc, L.hnxt, L.hmc);

  bool active = n > 0;
  bool need_dec = false;
  for (;;) {
    // ================= phase A: cheap, divergent =================
    while (active && !need_dec) {
      // next completion: min (time, kind, seq) over the load and the busy
      // slots (engine.cpp:49-55)
      double tc = L.lready;
      int sc_slot = L.ls;
      bool cload = L.ls >= 0;
      uint32_t qc = 0;
#pragma unroll
      for (int s = 0; s < C; ++s) {
        const bool better = slot_state(L.sms[s]) == ST_BUSY &&
                            (sc_slot < 0 || L.sdone[s] < tc ||
                             (L.sdone[s] == tc && !cload && L.sseq[s] < qc));
        if (better) {
          tc = L.sdone[s];
          sc_slot = s;
          cload = false;
          qc = L.sseq[s];
        }
      }
      if (!L.harr && (sc_slot < 0 || L.ha < tc)) {
        L.now = L.ha;  // arrival of the head into an empty queue
        L.harr = true;
      } else if (sc_slot < 0) {
        L.status = CACE_E_DEADLOCK;  // pending requests, nothing schedulable
        active = false;
        break;
      } else {
        // Load/ServiceComplete: slot -> Idle, last_used = event time
        // (engine.cpp:219-230)
        L.now = tc;
#pragma unroll
        for (int s = 0; s < C; ++s)
          if (s == sc_slot) {
            L.sms[s] = with_state(L.sms[s], ST_IDLE);
            L.slu[s] = tc;
          }
        if (cload) L.ls = -1;
        if (!L.harr) continue;  // queue empty: dispatch has nothing to do
      }

      // dispatch(now): head-of-line FIFO (engine.cpp:157-210)
      for (;;) {
        const int hm = (int)(L.hmc & 0xffffu);
        int hs = -1, hst = ST_IDLE;
#pragma unroll
        for (int s = 0; s < C; ++s)
          if (slot_model(L.sms[s]) == hm) {
            hs = s;
            hst = slot_state(L.sms[s]);
          }
        if (!L.hc) {  // classify once (engine.cpp:163-173)
          L.hc = true;
          const bool hit = hs >= 0 && hst != ST_LOADING;
          L.hits += hit ? 1u : 0u;
          L.misses += hit ? 0u : 1u;
          L.hcold = !hit;
        }
        if (hs >= 0) {
          if (hst != ST_IDLE) break;  // busy or still loading
          // start_service (engine.cpp:134-153)
          const double qd = L.now - L.ha;
          const double ttft = qd + L.hpf;
          const double e2e = ttft + L.hdc;
          const double done = (L.now + L.hpf) + L.hdc;
#pragma unroll
          for (int s = 0; s < C; ++s)
            if (s == hs) {
              L.sms[s] = with_state(L.sms[s], ST_BUSY);
              L.sdone[s] = done;
              L.sseq[s] = L.seqc;
            }
          ++L.seqc;
          if ((L.hmc >> 16) == CACE_COMPLETION) {
            ++L.nc;
            L.sttft += ttft;
            L.mttft = ttft > L.mttft ? ttft : L.mttft;
          } else {
            ++L.nr;
            L.se2e += e2e;
            L.me2e = e2e > L.me2e ? e2e : L.me2e;
          }
          L.ho = hmix(hmix(L.ho, dbits(ttft)), dbits(e2e) ^ (L.hcold ? 1ull : 0ull));
          if (DUMP && dslot >= 0) {
            const int64_t o = doff + P.perm[base + L.head];
            if (P.dump.cold) P.dump.cold[o] = L.hcold ? 1 : 0;
            if (P.dump.queue_wait) P.dump.queue_wait[o] = qd - L.hlw;
            if (P.dump.load_wait) P.dump.load_wait[o] = L.hlw;
            if (P.dump.prefill) P.dump.prefill[o] = L.hpf;
            if (P.dump.decode) P.dump.decode[o] = L.hdc;
            if (P.dump.ttft) P.dump.ttft[o] = ttft;
            if (P.dump.e2e) P.dump.e2e[o] = e2e;
          }
          // pop the head; the next is pending iff it arrived before now
          if (need_win) first[hm * stride] = L.hnxt;
          ++L.head;
          if (L.head == n) {
            active = false;
            break;
          }
          load_rec(tr + L.head, L.ha, L.hpf, L.hdc, L.hnxt, L.hmc);
          L.hc = false;
          L.hcold = false;
          L.hlw = 0.0;
          L.harr = L.ha < L.now;
          if (!L.harr) break;
          continue;
        }
        if (L.occ < C) {  // free slot, no unload delay (engine.cpp:184-187)
          start_load(L, L.occ, 0.0, s_lt, s_lex);
          ++L.occ;
          break;
        }
        bool any_idle = false;
#pragma unroll
        for (int s = 0; s < C; ++s) any_idle |= slot_state(L.sms[s]) == ST_IDLE;
        need_dec = any_idle;  // else every resident busy: wait (engine.cpp:203)
        break;
      }
    }

    // ================= phase B: eviction decision, converged =================
    if (need_dec) {
      need_dec = false;
      const double now = L.now;
      // Sorted-first = min (last_used, lex) over idle residents = LRU victim.
      int f = -1;
      double flu = 0.0;
      int flex = 0;
#pragma unroll
      for (int s = 0; s < C; ++s) {
        const int lx = slot_lex(L.sms[s]);
        if (slot_state(L.sms[s]) == ST_IDLE &&
            (f < 0 || L.slu[s] < flu || (L.slu[s] == flu && lx < flex))) {
          f = s;
          flu = L.slu[s];
          flex = lx;
        }
      }
      int victim = f;
      if (!is_lru) {
        // eviction_score for every idle entry (policy.cpp:39-78); the victim
        // is the first strict max in sorted order.
        uint32_t fm[C];
        int rank[C];
#pragma unroll
        for (int s = 0; s < C; ++s) {
          fm[s] = need_win ? first[slot_model(L.sms[s]) * stride] : 0u;
          rank[s] = 0;
        }
        if (need_win) {
          for (int mm = 0; mm < M; ++mm) {
            const uint32_t x = first[mm * stride];
#pragma unroll
            for (int s = 0; s < C; ++s) rank[s] += x < fm[s] ? 1 : 0;
          }
        }
        bool inwin[C];
        bool bad_clock = false;
#pragma unroll
        for (int s = 0; s < C; ++s) {
          bool iw = false;
          if (variant != CACE_MINUS_P3) {
            // in window [head, min(head + w, arrived)); fm >= head always
            iw = fm[s] < n && fm[s] - L.head < w;
            if (iw) iw = __ldg(&tr[fm[s]].arrival) < now;
          }
          inwin[s] = iw;
          bad_clock |= slot_state(L.sms[s]) == ST_IDLE && now < L.slu[s];
        }
        // ---- screening pass in fp32 with a rigorous error bound: if one
        // candidate's approximate total beats every other by more than the
        // bound, it is the exact arg-max and the fp64 totals are not needed.
        // |T~ - T| <= 2.6e-5 (3-ulp __logf on ln t < 70, Lipschitz-1 P1) plus
        // fp32 rounding of the terms and sums (<= 2^-22 |T|); margin 2x that.
        float best = -INFINITY, second = -INFINITY, tmax = 0.0f;
        int bs = -1;
        bool exact = bad_clock;
        const float wf = (float)sc.window_length;
#pragma unroll
        for (int s = 0; s < C; ++s) {
          const int m = slot_model(L.sms[s]);
          float p1 = 0.0f;
          if (variant != CACE_MINUS_P1) {
            const double d = now - L.slu[s];
            const double t = d < 1.0 ? 1.0 : d;
            exact |= !(t < 1e30);
            const float p1v = __frcp_rn(1.0f + __logf((float)t));
            p1 = verbatim ? p1v : 1.0f - p1v;
          }
          const float p2 = variant == CACE_MINUS_P2 ? 0.0f : (float)s_p2[m];
          const float p3 =
              variant == CACE_MINUS_P3 ? 0.0f : (inwin[s] ? __fdiv_rn((float)rank[s], wf) : 1.0f);
          const float p4 = variant == CACE_MINUS_P4 ? 0.0f : (float)p4tab[m * stride];
          const float T = ((p1 + p2) + p3) + p4;
          if (slot_state(L.sms[s]) == ST_IDLE) {
            tmax = fmaxf(tmax, fabsf(T));
            exact |= !(fabsf(T) <= 1e6f);  // NaN / inf / huge: decide exactly
            if (T > best) {
              second = best;
              best = T;
              bs = s;
            } else if (T > second) {
              second = T;
            }
          }
        }
        const float margin = 6e-5f + 4.8e-7f * tmax;
        exact |= !(best - second > margin);
        victim = bs;
        if (exact) {
          // ---- exact fp64 path (policy.cpp:39-115), bit-identical to the
          // reference: needed for near-ties (3-11% of CACE decisions are
          // exact ties broken by last_used, then model_id).
          double tot[C];
          int bad_lex = 1 << 30, bad_model = -1;
#pragma unroll
          for (int s = 0; s < C; ++s) {
            tot[s] = 0.0;
            if (slot_state(L.sms[s]) != ST_IDLE) continue;
            const int m = slot_model(L.sms[s]);
            if (now < L.slu[s]) {  // eviction_score throws (policy.cpp:43-46)
              const int lx = slot_lex(L.sms[s]);
              if (lx < bad_lex) {
                bad_lex = lx;
                bad_model = m;
              }
            }
            double p1 = 0.0;
            if (variant != CACE_MINUS_P1) {
              const double d = now - L.slu[s];
              const double t = d < 1.0 ? 1.0 : d;  // std::max(d, 1.0)
              const double lg = t == 1.0 ? 0.0 : cace_glibc_log(t, P.log_variant, P.log_tab, P.log_tab2);
              const double p1v = 1.0 / (1.0 + lg);
              p1 = verbatim ? p1v : 1.0 - p1v;
            }
            const double p2 = variant == CACE_MINUS_P2 ? 0.0 : s_p2[m];
            const double p3 =
                variant == CACE_MINUS_P3 ? 0.0 : (inwin[s] ? (double)rank[s] / wd : 1.0);
            const double p4 = variant == CACE_MINUS_P4 ? 0.0 : p4tab[m * stride];
            tot[s] = ((p1 + p2) + p3) + p4;
          }
          if (bad_model >= 0) {
            L.status = CACE_E_CLOCK | (bad_model << 8);
            active = false;
          } else {
            victim = f;
            double bt = 0.0;
#pragma unroll
            for (int s = 0; s < C; ++s)
              if (s == f) bt = tot[s];
            if (bt == bt) {  // a NaN sorted-first entry keeps the slot; NaN never wins later
              int blex = flex;
              double blu = flu;
#pragma unroll
              for (int s = 0; s < C; ++s) {
                const int lx = slot_lex(L.sms[s]);
                const bool earlier = L.slu[s] < blu || (L.slu[s] == blu && lx < blex);
                if (slot_state(L.sms[s]) == ST_IDLE && s != f &&
                    (tot[s] > bt || (tot[s] == bt && earlier))) {
                  victim = s;
                  bt = tot[s];
                  blu = L.slu[s];
                  blex = lx;
                }
              }
            }
          }
        }
      }
      if (active) {
        int vm = -1;
#pragma unroll
        for (int s = 0; s < C; ++s)
          if (s == victim) vm = slot_model(L.sms[s]);
        ++L.evictions;  // residents.erase(victim) (engine.cpp:205-206)
        L.he = hmix(hmix(L.he, (uint64_t)vm), dbits(now));
        if (DUMP && dslot >= 0) {
          if (dn_ev < P.dump.evict_cap) {
            if (P.dump.evict_model) P.dump.evict_model[dslot * P.dump.evict_cap + dn_ev] = vm;
            if (P.dump.evict_clock) P.dump.evict_clock[dslot * P.dump.evict_cap + dn_ev] = now;
          }
          ++dn_ev;
        }
        start_load(L, victim, sc.unload_time_s, s_lt, s_lex);
      }
    }
    if (!active) break;
  }

  cace_summary_t o;
  o.hits = L.hits;
  o.misses = L.misses;
  o.evictions = L.evictions;
  o.loads = L.loads;
  o.load_overhead_s = L.lo_sum;
  o.max_resident = L.occ;
  o.status = L.status;
  o.n_completion = L.nc;
  o.n_reasoning = L.nr;
  o.sum_ttft_completion = L.sttft;
  o.sum_e2e_reasoning = L.se2e;
  o.max_ttft_completion = L.mttft;
  o.max_e2e_reasoning = L.me2e;
  o.eviction_hash = L.he;
  o.outcome_hash = L.ho;
  P.out[sidx] = o;
  if (DUMP && dslot >= 0 && P.dump.n_evict) P.dump.n_evict[dslot] = dn_ev;
}

// Block of LANE_BLOCK lanes; per-lane shared columns for first[] and p4[],
// block-shared copy of the hot catalog columns.
constexpr int LANE_BLOCK = 128;

template <int C, bool DUMP>
__global__ void __launch_bounds__(LANE_BLOCK) replay_lane_kernel(ReplayParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int M = P.cat.M;
  double* s_lt = reinterpret_cast<double*>(smem);
  double* s_p2 = s_lt + M;
  double* p4tab = s_p2 + M;                                      // [M][LANE_BLOCK]
  int* s_lex = reinterpret_cast<int*>(p4tab + (size_t)M * LANE_BLOCK);
  uint32_t* first = reinterpret_cast<uint32_t*>(s_lex + M);       // [M][LANE_BLOCK]
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    s_lt[m] = P.cat.load_time[m];
    s_p2[m] = P.cat.p2[m];
    s_lex[m] = P.cat.lex[m];
  }
  __syncthreads();
  const int64_t gi = P.seg_begin + (int64_t)blockIdx.x * LANE_BLOCK + threadIdx.x;
  if (gi >= P.seg_end) return;
  replay_scenario<C, DUMP>(P, P.order[gi], first + threadIdx.x, p4tab + threadIdx.x, LANE_BLOCK,
                           s_lt, s_p2, s_lex);
}

inline size_t lane_smem_bytes(int M) {
  return (size_t)M * (8 + 8 + 4) + (size_t)M * LANE_BLOCK * (8 + 4);
}

}  // namespace cace
