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

// Replays one scenario.  first/p4 are this lane's shared-memory columns
// (element m at [m * stride]).  Template C = capacity (slots), so the slot
// arrays live in registers with fully unrolled scans.
template <int C>
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
  const double unload = sc.unload_time_s;

  // Dump slot (rare; only for full-report scenarios).
  int dslot = -1;
  if (P.dump.slot) dslot = P.dump.slot[sidx];
  const int64_t doff = dslot >= 0 ? P.dump.dump_off[dslot] : 0;
  int64_t dn_ev = 0;

  if (need_win) {
    const uint32_t* f0 = P.first0 + (int64_t)sc.trace * M;
    for (int m = 0; m < M; ++m) first[m * stride] = __ldg(f0 + m);
  }
  if (!is_lru) {
    // p4 = w1 * (tokens / normalizer)   (policy.cpp:66-67)
    const double norm = (double)sc.output_token_normalizer;
    for (int m = 0; m < M; ++m) p4tab[m * stride] = sc.w1 * (__ldg(P.cat.tokens + m) / norm);
  }

  // Slot state (registers).
  int sm[C];
  int sst[C];
  double slu[C], sdone[C];
  uint32_t sseq[C];
#pragma unroll
  for (int s = 0; s < C; ++s) {
    sm[s] = -1;
    sst[s] = ST_IDLE;
    slu[s] = 0.0;
    sdone[s] = 0.0;
    sseq[s] = 0;
  }
  int occ = 0;
  int ls = -1;          // slot with the in-flight load
  double lready = 0.0;  // its LoadComplete time
  uint32_t seqc = 0;    // ServiceComplete push order

  uint64_t hits = 0, misses = 0, evictions = 0, loads = 0;
  double lo_sum = 0.0;
  uint64_t nc = 0, nr = 0;
  double sttft = 0.0, se2e = 0.0, mttft = 0.0, me2e = 0.0;
  uint64_t ho = CACE_HASH_SEED, he = CACE_HASH_SEED;
  int status = CACE_OK;

  // Queue head.
  uint32_t head = 0;
  double ha = 0.0, hpf = 0.0, hdc = 0.0, hlw = 0.0;
  uint32_t hnxt = 0, hmc = 0;
  bool hc = false, hcold = false, harr = false;
  if (n > 0) load_rec(tr, ha, hpf, hdc, hnxt, hmc);

  while (head < n) {
    // ---- next completion event: min (time, kind, seq) over the load and
    // the busy slots (engine.cpp:49-55).
    double tc = 0.0;
    int sc_slot = -1;
    bool cload = false;
    uint32_t qc = 0;
    if (ls >= 0) {
      tc = lready;
      sc_slot = ls;
      cload = true;
    }
#pragma unroll
    for (int s = 0; s < C; ++s) {
      const bool busy = sst[s] == ST_BUSY;
      const bool better =
          busy && (sc_slot < 0 || sdone[s] < tc || (sdone[s] == tc && !cload && sseq[s] < qc));
      if (better) {
        tc = sdone[s];
        sc_slot = s;
        cload = false;
        qc = sseq[s];
      }
    }
    double now;
    if (!harr && (sc_slot < 0 || ha < tc)) {
      // Arrival of the head into an empty queue.
      now = ha;
      harr = true;
    } else if (sc_slot < 0) {
      status = CACE_E_DEADLOCK;  // pending requests, nothing schedulable
      break;
    } else {
      // LoadComplete / ServiceComplete: slot -> Idle, last_used = event time
      // (engine.cpp:219-230).
      now = tc;
#pragma unroll
      for (int s = 0; s < C; ++s)
        if (s == sc_slot) {
          sst[s] = ST_IDLE;
          slu[s] = now;
        }
      if (cload) ls = -1;
      if (!harr) continue;  // queue empty: dispatch has nothing to do
    }

    // ---- dispatch(now): head-of-line FIFO (engine.cpp:157-210).
    for (;;) {
      const int hm = (int)(hmc & 0xffffu);
      int hs = -1;
#pragma unroll
      for (int s = 0; s < C; ++s)
        if (sm[s] == hm) hs = s;
      int hst = ST_IDLE;
#pragma unroll
      for (int s = 0; s < C; ++s)
        if (s == hs) hst = sst[s];
      if (!hc) {  // classify once (engine.cpp:163-173)
        hc = true;
        const bool hit = hs >= 0 && hst != ST_LOADING;
        hits += hit ? 1 : 0;
        misses += hit ? 0 : 1;
        hcold = !hit;
      }
      if (hs >= 0) {
        if (hst != ST_IDLE) break;  // busy or still loading
        // start_service (engine.cpp:134-153)
        const double qd = now - ha;
        const double ttft = qd + hpf;
        const double e2e = ttft + hdc;
        const double done = (now + hpf) + hdc;
#pragma unroll
        for (int s = 0; s < C; ++s)
          if (s == hs) {
            sst[s] = ST_BUSY;
            sdone[s] = done;
            sseq[s] = seqc;
          }
        ++seqc;
        if ((hmc >> 16) == CACE_COMPLETION) {
          ++nc;
          sttft += ttft;
          mttft = ttft > mttft ? ttft : mttft;
        } else {
          ++nr;
          se2e += e2e;
          me2e = e2e > me2e ? e2e : me2e;
        }
        ho = hmix(hmix(ho, dbits(ttft)), dbits(e2e) ^ (hcold ? 1ull : 0ull));
        if (dslot >= 0) {
          const int64_t o = doff + P.perm[base + head];
          if (P.dump.cold) P.dump.cold[o] = hcold ? 1 : 0;
          if (P.dump.queue_wait) P.dump.queue_wait[o] = qd - hlw;
          if (P.dump.load_wait) P.dump.load_wait[o] = hlw;
          if (P.dump.prefill) P.dump.prefill[o] = hpf;
          if (P.dump.decode) P.dump.decode[o] = hdc;
          if (P.dump.ttft) P.dump.ttft[o] = ttft;
          if (P.dump.e2e) P.dump.e2e[o] = e2e;
        }
        // pop the head; the next one is pending iff it arrived before now.
        if (need_win) first[hm * stride] = hnxt;
        ++head;
        if (head == n) break;
        load_rec(tr + head, ha, hpf, hdc, hnxt, hmc);
        hc = false;
        hcold = false;
        hlw = 0.0;
        harr = ha < now;
        if (!harr) break;
        continue;
      }

      int target;
      double udelay;
      if (occ < C) {  // free slot: load without unload delay (engine.cpp:184-187)
        target = occ;
        ++occ;
        udelay = 0.0;
      } else {
        // ---- victim selection among idle residents (policy.cpp:80-115).
        // Sorted-first = min (last_used, lex) over idle = the LRU victim.
        int f = -1;
        double flu = 0.0;
        int flex = 0;
#pragma unroll
        for (int s = 0; s < C; ++s) {
          if (sst[s] != ST_IDLE) continue;
          const int lx = s_lex[sm[s]];
          if (f < 0 || slu[s] < flu || (slu[s] == flu && lx < flex)) {
            f = s;
            flu = slu[s];
            flex = lx;
          }
        }
        if (f < 0) break;  // every resident busy: wait (engine.cpp:203)
        int victim = f;
        if (!is_lru) {
          // Score every idle entry; "first strict max in sorted order".
          double tot[C];
          int bad_lex = 1 << 30, bad_model = -1;
#pragma unroll
          for (int s = 0; s < C; ++s) {
            tot[s] = 0.0;
            if (sst[s] != ST_IDLE) continue;
            const int m = sm[s];
            if (now < slu[s]) {  // eviction_score throws (policy.cpp:43-46)
              const int lx = s_lex[m];
              if (lx < bad_lex) {
                bad_lex = lx;
                bad_model = m;
              }
            }
            double p1 = 0.0;
            if (variant != CACE_MINUS_P1) {
              const double d = now - slu[s];
              const double t = d < 1.0 ? 1.0 : d;  // std::max(d, 1.0)
              const double L = cace_glibc_log(t, P.log_variant, P.log_tab, P.log_tab2);
              const double p1v = 1.0 / (1.0 + L);
              p1 = verbatim ? p1v : 1.0 - p1v;
            }
            const double p2 = variant == CACE_MINUS_P2 ? 0.0 : s_p2[m];
            double p3 = 0.0;
            if (variant != CACE_MINUS_P3) {
              const uint32_t fm = first[m * stride];
              // in window [head, min(head + w, arrived)): fm >= head always
              bool inwin = fm < n && fm - head < w;
              if (inwin) inwin = __ldg(&tr[fm].arrival) < now;
              if (inwin) {
                int rank = 0;
                for (int mm = 0; mm < M; ++mm) rank += first[mm * stride] < fm ? 1 : 0;
                p3 = (double)rank / wd;
              } else {
                p3 = 1.0;
              }
            }
            const double p4 = variant == CACE_MINUS_P4 ? 0.0 : p4tab[m * stride];
            tot[s] = ((p1 + p2) + p3) + p4;
          }
          if (bad_model >= 0) {
            status = CACE_E_CLOCK | (bad_model << 8);
            break;
          }
          double bt = 0.0;
#pragma unroll
          for (int s = 0; s < C; ++s)
            if (s == f) bt = tot[s];
          if (bt == bt) {  // sorted-first NaN keeps it; NaN never wins later
            int blex = flex;
            double blu = flu;
#pragma unroll
            for (int s = 0; s < C; ++s) {
              if (sst[s] != ST_IDLE || s == f) continue;
              const double ts = tot[s];
              const int lx = s_lex[sm[s]];
              const bool earlier = slu[s] < blu || (slu[s] == blu && lx < blex);
              if (ts > bt || (ts == bt && earlier)) {
                victim = s;
                bt = ts;
                blu = slu[s];
                blex = lx;
              }
            }
          }
        }
        int vm = -1;
#pragma unroll
        for (int s = 0; s < C; ++s)
          if (s == victim) vm = sm[s];
        ++evictions;  // residents.erase(victim) (engine.cpp:205-206)
        he = hmix(hmix(he, (uint64_t)vm), dbits(now));
        if (dslot >= 0) {
          if (dn_ev < P.dump.evict_cap) {
            if (P.dump.evict_model) P.dump.evict_model[dslot * P.dump.evict_cap + dn_ev] = vm;
            if (P.dump.evict_clock) P.dump.evict_clock[dslot * P.dump.evict_cap + dn_ev] = now;
          }
          ++dn_ev;
        }
        target = victim;
        udelay = unload;
      }
      // start_load (engine.cpp:123-132)
      const double lt = s_lt[hm];
      const double ready = (now + udelay) + lt;
      hlw = ready - now;
      lo_sum += lt;
      ++loads;
#pragma unroll
      for (int s = 0; s < C; ++s)
        if (s == target) {
          sm[s] = hm;
          sst[s] = ST_LOADING;
          slu[s] = now;
        }
      ls = target;
      lready = ready;
      break;
    }
    if (status != CACE_OK) break;
  }

  cace_summary_t o;
  o.hits = hits;
  o.misses = misses;
  o.evictions = evictions;
  o.loads = loads;
  o.load_overhead_s = lo_sum;
  o.max_resident = occ;
  o.status = status;
  o.n_completion = nc;
  o.n_reasoning = nr;
  o.sum_ttft_completion = sttft;
  o.sum_e2e_reasoning = se2e;
  o.max_ttft_completion = mttft;
  o.max_e2e_reasoning = me2e;
  o.eviction_hash = he;
  o.outcome_hash = ho;
  P.out[sidx] = o;
  if (dslot >= 0 && P.dump.n_evict) P.dump.n_evict[dslot] = dn_ev;
}

// Block of LANE_BLOCK lanes; per-lane shared columns for first[] and p4[],
// block-shared copy of the hot catalog columns.
constexpr int LANE_BLOCK = 128;

template <int C>
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
  replay_scenario<C>(P, P.order[gi], first + threadIdx.x, p4tab + threadIdx.x, LANE_BLOCK, s_lt,
                     s_p2, s_lex);
}

inline size_t lane_smem_bytes(int M) {
  return (size_t)M * (8 + 8 + 4) + (size_t)M * LANE_BLOCK * (8 + 4);
}

}  // namespace cace
