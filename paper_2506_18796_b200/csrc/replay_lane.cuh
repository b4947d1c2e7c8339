// Lane-per-scenario, request-synchronous trace-replay kernel (sm_100a).
//
// One thread replays one scenario = one reference run(trace, catalog,
// cluster, policy) (engine.cpp:76-239 + policy.cpp:22-115), bit-exact.  The
// host plan makes every warp trace-uniform (capacity/trace groups padded to
// whole warps with shadow lanes), and the replay loop is organised so that
// iteration k of EVERY lane processes request k of the trace — the request
// record is a warp-uniform broadcast read and the lanes never drift apart.
//
// Why request k can be processed in one step (the reference's min-heap order
// (time, kind, seq) of engine.cpp:49-55; kind 0 LoadComplete, 1
// ServiceComplete, 2 Arrival).  Between two service starts the reference's
// event loop can only do the following (engine.cpp:157-230,
// policy.cpp:80-115):
//   * queue empty -> the head's Arrival (a_k, 2, k) is the next relevant
//     event; each ServiceComplete with a smaller key just idles its slot
//     (last_used = its time) — dispatch with an empty queue does nothing;
//   * head resident & Idle -> served in the current dispatch (a hit);
//   * head resident & Busy -> blocked until its own ServiceComplete; earlier
//     completions only idle other slots (the head blocks the FIFO);
//   * head not resident -> a free slot (load without unload delay), or an
//     eviction decision at the current event if any slot is Idle (forced
//     when exactly one), or, if every slot is Busy, at the next
//     ServiceComplete, whose slot is then the only Idle one (forced victim);
//     then blocked until its LoadComplete (r, 0, .), before which
//     completions only idle slots.  At most one load is ever in flight.
//   * An Arrival into a non-empty queue never changes a decision; request
//     j > head is pending at event time `now` iff a_j < now.
// So completions are applied in bulk against the event cursor, the pending
// queue is the contiguous range [k, arrived), and only a decision with >= 2
// idle candidates evaluates eviction_score.
//
// Slot state is one register per slot, SIGN-ENCODED: stime >= 0 is an Idle
// slot with last_used_s = stime; stime < 0 is a Busy slot whose
// ServiceComplete is at -stime (a completion sets last_used to its own event
// time, engine.cpp:224-229, so applying it is |stime|).  Event times are
// >= 0 (arrivals are validated non-negative, as parse_trace requires,
// workload.cpp:245) and service completions are > 0, so the sign is free.
//
// Lookahead window (dedup_window, policy.cpp:22-37): p3 of a resident model
// m needs first[m] (first replay index >= k requesting m), rank(m) =
// #{m' : first[m'] < first[m]} and whether first[m] has arrived.  These
// depend only on the trace and k, so they are warp-wide: lane j owns models
// j, j+32 in registers, advances them with one warp reduction per request and
// publishes {first, rank, arrival of first} to a per-warp shared-memory table
// that deciding lanes read per candidate.
//
// The trace is staged per warp in shared memory by TMA bulk copies (one
// cp.async.bulk of 32 records per chunk, double-buffered, mbarrier-completed),
// so the per-request record read is a broadcast shared load and no registers
// carry a prefetched record.
//
// All fp64 arithmetic uses the reference's operation order with no
// contraction (built with -fmad=false); P1's log is the glibc restatement
// (glibc_log.cuh).  Decisions are first screened in fp32 with a rigorous
// error margin; near-ties fall back to the exact fp64 scores of the
// candidates within the margin (exact ties of identical inputs short-cut to
// the reference's tie order).
#pragma once
#include <math.h>
#include <stdint.h>

#include "../../include/cace_gpu.h"
#include "glibc_log.cuh"
#include "replay_types.h"

// Instrumentation hook of the test-only host emulation (per-request decision
// statistics, tools/decision_stats.py); compiled out of the product.
#ifndef CACE_STAT
#define CACE_STAT(kind, k)
#endif

namespace cace {

// Summary fingerprint (spec CACE_HASH in include/cace_gpu.h).
__device__ __forceinline__ uint64_t hmix(uint64_t h, uint64_t x) {
  const uint32_t lo = (uint32_t)h * CACE_HASH_MUL_LO + (uint32_t)x;
  const uint32_t hi = (uint32_t)(h >> 32) * CACE_HASH_MUL_HI + (uint32_t)(x >> 32);
  return ((uint64_t)hi << 32) | lo;
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

// Slot word: model (bits 0-15) | lex rank of model_id (bits 18-31).
__device__ __forceinline__ int slot_model(int v) { return v & 0xffff; }
__device__ __forceinline__ int slot_lex(int v) { return (int)((unsigned)v >> 18); }
// Event key (time, kind, seq) of engine.cpp:49-55 (warp kernel).
struct Cursor {
  double t;
  int kind;
  uint32_t seq;
};

// key(ServiceComplete of a slot) <= cursor
__device__ __forceinline__ bool sc_le(double d, uint32_t q, const Cursor& c) {
  return d < c.t || (d == c.t && (c.kind > 1 || (c.kind == 1 && q <= c.seq)));
}

constexpr unsigned kFull = 0xffffffffu;
constexpr float kLn2f = 0.693147180559945309f;

#ifdef CACE_HOST_EMULATION
__device__ __forceinline__ float fast_lg2(float x) { return log2f(x); }
__device__ __forceinline__ float fast_rcp(float x) { return 1.0f / x; }
#else
__device__ __forceinline__ float fast_lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fast_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
#endif

// Exact fp64 P1 of eviction_score (policy.cpp:50-53) with the glibc log.
// Out of line: one copy serves every unrolled candidate of the rare exact
// path, and its temporaries do not add to the replay loop's register peak.
#ifdef CACE_EXACT_INLINE
__device__ __forceinline__
#else
__device__ __noinline__
#endif
double exact_p1(double now, double last_used, bool verbatim, int log_variant,
                                        const double* tab, const double* tab2) {
  const double d = now - last_used;
  const double t = d < 1.0 ? 1.0 : d;  // std::max(d, 1.0)
  const double lg = t == 1.0 ? 0.0 : cace_glibc_log(t, log_variant, tab, tab2);
  const double p1v = 1.0 / (1.0 + lg);
  return verbatim ? p1v : 1.0 - p1v;
}

// Per-warp window table entry: first pending index of the model, its rank
// among the models' first occurrences (as a float: an exact small integer),
// and that request's arrival time (+inf when the model has no pending
// request left).
struct alignas(16) WinEnt {
  uint32_t f;
  float r;
  double fa;
};

// Warp-wide lookahead window (see the file comment).  MW registers per lane:
// lane j owns models j + 32q, q < MW.
template <int MW>
struct Window {
#ifdef CACE_HOST_EMULATION
  uint32_t f[32 * MW], r[32 * MW];
  double fa[32 * MW];
  int M;
  void init(const uint32_t* f0, int M_, const ReqRec* tr, uint32_t n, WinEnt*) {
    M = M_;
    for (int m = 0; m < M; ++m) {
      f[m] = f0[m];
      fa[m] = f0[m] < n ? tr[f0[m]].arrival : INFINITY;
    }
    for (int m = 0; m < M; ++m) {
      uint32_t c = 0;
      for (int q = 0; q < M; ++q) c += f0[q] < f0[m] ? 1u : 0u;
      r[m] = c;
    }
  }
  WinEnt gather(int ms) const { return WinEnt{f[ms], (float)r[ms], fa[ms]}; }
  WinEnt gather128(int ms) const { return gather(ms); }
  int pmk = 0;
  uint32_t pnx = 0;
  void prepare(int mk, uint32_t nx) {
    pmk = mk;
    pnx = nx;
  }
  void commit(double nxa) { advance(pmk, pnx, nxa); }
  void advance(int mk, uint32_t nx, double nxa) {
    uint32_t cnt = 0;
    for (int j = 0; j < M; ++j)
      if (j != mk && f[j] < nx) {
        r[j] -= 1;
        ++cnt;
      }
    f[mk] = nx;
    r[mk] = cnt;
    fa[mk] = nxa;
  }
#else
  // ranks are kept as floats (exact small integers; the table stores them as
  // floats) so committing them needs no conversion
  uint32_t f[MW];
  float r[MW];
  int M;
  WinEnt* tab;
  __device__ __forceinline__ void init(const uint32_t* f0, int M_, const ReqRec* tr, uint32_t n,
                                       WinEnt* tab_) {
    M = M_;
    tab = tab_;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < MW; ++q) {
      const int m = lane + 32 * q;
      f[q] = m < M ? __ldg(f0 + m) : 0xffffffffu;
      uint32_t c = 0;
      for (int mm = 0; mm < M; ++mm) c += __ldg(f0 + mm) < f[q] ? 1u : 0u;
      r[q] = (float)c;
      if (m < M) tab[m] = WinEnt{f[q], (float)c, f[q] < n ? __ldg(&tr[f[q]].arrival) : INFINITY};
    }
    __syncwarp();
  }
  // Per lane (no collective): model ms's entry.
  __device__ __forceinline__ WinEnt gather(int ms) const { return tab[ms]; }
  // The same entry through one 128-bit load: +3% on the wide-pool kernel
  // (config 5), -5% on the latency instantiation (config 3), so only the
  // wide mode uses it (profiles/r2/ab_window_load_r2am.txt).
  __device__ __forceinline__ WinEnt gather128(int ms) const {
    const uint4 q = *reinterpret_cast<const uint4*>(tab + ms);
    return WinEnt{q.x, __uint_as_float(q.y), __hiloint2double((int)q.w, (int)q.z)};
  }
  // Collective: prepare computes the state after the head (model mk) is
  // served -- mk's first becomes nx -- without touching what the iteration's
  // decisions read; commit installs it.  (Issuing prepare at the top of the
  // iteration to overlap the ballot latency measured slower; the replay loop
  // calls them back to back at the end.)  mk's new rank = the number of other
  // models whose first pending request precedes nx: each lane counts its own
  // models, one warp reduction sums them.
  uint32_t nf[MW];
  float nr[MW];
  int pmk;
  __device__ __forceinline__ void prepare(int mk, uint32_t nx) {
    const int lane = threadIdx.x & 31;
    pmk = mk;
    uint32_t lc = 0;
#pragma unroll
    for (int q = 0; q < MW; ++q) {
      const int m = lane + 32 * q;
      const bool before = m < M && m != mk && f[q] < nx;
      lc += before ? 1u : 0u;
      nf[q] = f[q];
      nr[q] = before ? r[q] - 1.0f : r[q];
    }
    const float cnt = (float)__reduce_add_sync(kFull, lc);
#pragma unroll
    for (int q = 0; q < MW; ++q)
      if (lane + 32 * q == mk) {
        nf[q] = nx;
        nr[q] = cnt;
      }
  }
  __device__ __forceinline__ void commit(double nxa) {
    const int lane = threadIdx.x & 31;
    __syncwarp();  // every lane's reads of the table for this request precede the writes
#pragma unroll
    for (int q = 0; q < MW; ++q) {
      const int m = lane + 32 * q;
      f[q] = nf[q];
      r[q] = nr[q];
      if (m == pmk) tab[m].fa = nxa;
      if (m < M) *reinterpret_cast<uint2*>(&tab[m]) = make_uint2(f[q], __float_as_uint(r[q]));
    }
    __syncwarp();
  }
#endif
};

// Trace records of the warp's trace in replay order.  Device: per-warp
// shared-memory double buffer of 2 x 32 records, filled one chunk ahead.
// Default: ONE bulk copy per chunk (cp.async.bulk on the TMA engine; SASS
// UBLKCP) issued by lane 0 and completed on a per-buffer mbarrier
// (expect_tx / complete_tx) that the warp waits on with try_wait.parity.
// CACE_REC_LDGSTS selects round 1's per-lane cp.async staging (LDGSTS,
// 3 x 16 B per lane) for A/B measurements.
struct RecStream {
#ifdef CACE_HOST_EMULATION
  const ReqRec* g;
  void init(const ReqRec* g_, uint32_t, ReqRec*, uint64_t*) { g = g_; }
  void fini() {}
  const ReqRec* chunk(uint32_t c) { return g + (size_t)c * 32; }
#elif defined(CACE_REC_LDGSTS)
  const ReqRec* g;
  uint32_t n;
  ReqRec* buf;
  __device__ __forceinline__ void issue(uint32_t c) {
    const uint32_t i = c * 32 + (threadIdx.x & 31);
    if (i < n) {
      const char* src = reinterpret_cast<const char*>(g + i);
      const uint32_t dst =
          (uint32_t)__cvta_generic_to_shared(buf + ((c & 1) * 32 + (threadIdx.x & 31)));
#pragma unroll
      for (int b = 0; b < (int)sizeof(ReqRec); b += 16)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst + b), "l"(src + b)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  __device__ __forceinline__ void init(const ReqRec* g_, uint32_t n_, ReqRec* buf_, uint64_t*) {
    g = g_;
    n = n_;
    buf = buf_;
    issue(0);
  }
  __device__ __forceinline__ void fini() { __syncwarp(); }
  // Collective: records [32c, 32c + 32) once chunk c has landed; prefetches
  // chunk c + 1 into the other half.
  __device__ __forceinline__ const ReqRec* chunk(uint32_t c) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    issue(c + 1);
    return buf + (c & 1) * 32;
  }
#else
  const ReqRec* g;
  uint32_t n;
  ReqRec* buf;
  uint32_t bar;  // shared address of the two mbarriers (8 B each)
  __device__ __forceinline__ void issue(uint32_t c) {
    if ((threadIdx.x & 31) == 0 && c * 32 < n) {
      const uint32_t bytes = min(32u, n - c * 32) * (uint32_t)sizeof(ReqRec);  // multiple of 16
      const uint32_t b = bar + (c & 1) * 8;
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(buf + (c & 1) * 32);
      // the warp's generic-proxy reads of this half (chunk c - 2) precede the
      // async-proxy write
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dst), "l"(g + (size_t)c * 32), "r"(bytes), "r"(b)
                   : "memory");
    }
  }
  __device__ __forceinline__ void init(const ReqRec* g_, uint32_t n_, ReqRec* buf_, uint64_t* bar_) {
    g = g_;
    n = n_;
    buf = buf_;
    bar = (uint32_t)__cvta_generic_to_shared(bar_);
    if ((threadIdx.x & 31) == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar + 8) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    issue(0);
  }
  // Collective, after the last chunk: no copy is in flight; the barriers are
  // invalidated so the memory can be re-initialised for the warp's next replay.
  __device__ __forceinline__ void fini() {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bar + 8) : "memory");
    }
    __syncwarp();
  }
  // Collective: records [32c, 32c + 32) once chunk c has landed (phase c / 2
  // of its half's mbarrier); prefetches chunk c + 1 into the other half.
  __device__ __forceinline__ const ReqRec* chunk(uint32_t c) {
    const uint32_t b = bar + (c & 1) * 8, par = (c >> 1) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(b), "r"(par)
          : "memory");
    __syncwarp();
    issue(c + 1);
    return buf + (c & 1) * 32;
  }
#endif
};

// Block-shared catalog columns.
struct CatShared {
  const double* lt;   // load_time_s
  const double* p2;   // 1 / (1 + load_time / 100)
  const double* tok;  // (double) expected_output_tokens
  const float* p2f;   // fp32 copies for screening
  const float* tokf;
  const int* lex;     // rank of model_id under std::string <
};

// One resident slot: completion time of its last service (= last_used_s once
// that ServiceComplete has popped), the service's push seq, and the slot word
// (model | lex rank << 18).  16 B: one 128-bit shared load per slot.
struct alignas(16) SlotEnt {
  double done;
  uint32_t seq;
  int word;
};

// Per-lane shared-memory columns (element i at [i * stride]) and the lane's
// warp-shared tables.
struct LaneSmem {
  float* p4f;        // [M] p2 + p4 = p2 + w1 * (tokens / normalizer), fp32 (screening)
  double* p4d;       // [M] p4 = w1 * (tokens / normalizer), exact fp64 (policy.cpp:66-67) (NULL: wide)
  SlotEnt* slot;     // [C] resident slots
  float* prm;        // [4] screen constants: 1/w, p1 scale, p1 offset, margin (+inf: no screen)
  double* ud;        // [1] unload_time_s (read on evictions)
  float* wprm;       // [2] wide pools: p2 scale (0 / 1), w1 / normalizer (fp32; 0 when p4 is ablated)
  uint8_t* slot_of;  // [M] slot + 1 holding model m, 0 = not resident
  int stride;
  ReqRec* rec;       // warp: record double buffer [64]
  WinEnt* win;       // warp: window table [M]
  double* samp;      // warp: metrics sample tile [2 classes][kSampT][32 lanes] (DUMP only)
  uint64_t* rbar;    // warp: the record buffers' two mbarriers
};

// Event cursor (time, kind, seq) of engine.cpp:49-55 as (ct, cw) with
// cw = kind << 30 | seq (replay indices are < 2^30, layout.hpp).  A slot's
// ServiceComplete (done, 1, seq) has popped -- the slot is Idle with
// last_used_s = done -- iff its key is <= the cursor.
constexpr uint32_t kKindSC = 1u << 30;
constexpr uint32_t kKindArr = 2u << 30;
// Compared as 96-bit unsigned keys (bits(done), kKindSC | seq) <=
// (bits(ct), cw): every clock value is a non-negative finite double
// (layout.hpp rejects negative arrivals; done = (now + pf) + dc is never -0)
// whose bit pattern orders like the value, and the cursor's sign bit is
// cleared so an arrival at -0.0 compares equal to +0.0.  One integer
// subtract-with-borrow chain instead of two fp64 compares.
// The wide-pool kernel keeps the two fp64 compares (INTKEY = false): there
// the integer chain measured 6% slower on config 5 (profiles/r2/ab_wide_key_r2ba.txt).
template <bool INTKEY = true>
__device__ __forceinline__ bool sc_popped(double done, uint32_t seq, double ct, uint32_t cw) {
  if constexpr (!INTKEY) return done < ct || (done == ct && (kKindSC | seq) <= cw);
  const uint64_t db = (uint64_t)__double_as_longlong(done);
  const uint64_t cb = (uint64_t)__double_as_longlong(ct) & 0x7fffffffffffffffull;
#ifdef CACE_HOST_EMULATION
  return db < cb || (db == cb && (kKindSC | seq) <= cw);
#else
  uint32_t b;
  asm("{\n\t.reg .u32 t;\n\t"
      "sub.cc.u32 t, %1, %2;\n\t"
      "subc.cc.u32 t, %3, %4;\n\t"
      "subc.cc.u32 t, %5, %6;\n\t"
      "subc.u32 %0, 0, 0;\n\t}"
      : "=r"(b)
      : "r"(cw), "r"(kKindSC | seq), "r"((uint32_t)cb), "r"((uint32_t)db), "r"((uint32_t)(cb >> 32)),
        "r"((uint32_t)(db >> 32)));
  return b == 0u;
#endif
}

// Metrics samples leave through a per-warp shared tile: the lanes of a warp
// replay the same trace in lockstep, so request k has the same class-local
// index ci in every lane; kSampT consecutive samples per lane are gathered and
// written as kSampT * 8 contiguous bytes per scenario (32 / kSampT scenarios
// per store instruction) instead of 32 scattered 8-B stores per request.
constexpr int kSampT = 4;

#ifndef CACE_HOST_EMULATION
// Warp-collective: lane q's tile column [0, cnt) -> mine(q)[base + 0 .. cnt).
// The warp's 32 destination pointers (null: write nothing) and the trace's
// completion count sit after the tile, so they hold no registers.
__device__ __forceinline__ double* const* samp_ptrs(double* tile) {
  return reinterpret_cast<double* const*>(tile + 2 * kSampT * 32);
}
__device__ __forceinline__ uint32_t samp_ncomp(double* tile) {
  return *reinterpret_cast<const uint32_t*>(tile + 2 * kSampT * 32 + 32);
}
__device__ __forceinline__ void flush_samples(const double* tile, double* const* ptrs, int64_t base, int cnt) {
  const int lane = threadIdx.x & 31;
  const int j = lane % kSampT;
#pragma unroll
  for (int i = 0; i < kSampT; ++i) {
    const int q = lane / kSampT + (32 / kSampT) * i;
    const double v = tile[j * 32 + q];
    double* pq = ptrs[q];
    if (pq && j < cnt) pq[base + j] = v;
  }
}
#endif

// Replays one scenario (see the file comment).  shadow lanes (warp padding)
// replay a copy of a real scenario for lockstep and write nothing.
// XR: the exact fallback as rolled loops over the idle slots re-reading the
// shared slot table (compact code, few live registers) or unrolled over the
// slot entries already in registers.
// WIDE (pools > 64 models or capacities > 16): C is the unroll bound and the
// capacity is cap_rt (<= C); no per-lane p2 + p4 tables -- the fp32 screen
// forms p2 + p4 from the block's catalog columns and two per-lane scalars,
// the exact path recomputes p4 = w1 * (tokens / normalizer).
// MC > 0: the pool size is the compile-time constant MC (== P.cat.M), so the
// shared-memory layout folds into immediate offsets (the 8-model pool of
// BASELINE configs 1-4); 0: the runtime P.cat.M.
// RTC: the capacity is cap_rt (<= C, a runtime value) in the one-lane mode
// too -- one instantiation serves every capacity up to C (the mixed-capacity
// launch of shallow sweeps).
template <int C, int MW, int DM, bool XR = true, bool WIDE = false, int G = 1, int MC = 0, bool RTC = false>
__device__ void replay_scenario(const ReplayParams& P, int64_t sidx, bool shadow, bool warp_win,
                                const CatShared& K, const LaneSmem& S, int cap_rt = C) {
  static_assert(G == 1 || WIDE, "lane groups are a wide-pool mode");
  const int cap = (WIDE || RTC) ? cap_rt : C;
#ifdef CACE_HOST_EMULATION
  const int lig = 0;
  const unsigned gmask = 1u;
#else
  const int lig = (int)(threadIdx.x & (G - 1));  // lane within the scenario's group
  const unsigned gmask = G == 32 ? kFull : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
#endif
  const cace_scenario_t sc = P.scen[sidx];
  const int M = MC > 0 ? MC : P.cat.M;
  const int64_t base = P.trace_off[sc.trace];
  const uint32_t n = (uint32_t)(P.trace_off[sc.trace + 1] - base);
  const ReqRec* tr = P.rec + base;
  const int variant = sc.variant;
  const bool is_lru = variant == CACE_LRU;
  const bool need_win = !is_lru && variant != CACE_MINUS_P3;
  const bool verbatim = sc.p1_mode == CACE_P1_VERBATIM;
  const uint32_t w = (uint32_t)sc.window_length;
  const double norm = (double)sc.output_token_normalizer;

  const int st = S.stride;
  // fp32 screening is valid while every p2 + p4 is finite and moderate; the
  // event clock is finite (validated on the host) and t < 1e30 below.
  // tbound >= |total| of every candidate (p1, p3 in [0, 1]) sets the margin.
  bool screen_ok = true;
  float tbound = 2.0f;
  const bool writer = !WIDE || lig == 0;  // wide pools: one writer per group's shared columns
  for (int mm = 0; mm < M; ++mm) {
    if (writer) S.slot_of[mm * st] = 0;
    // p2 + p4 of model mm (policy.cpp:55, 66-67): exact p4 for the fp64
    // path, fp32 p2 + p4 for screening; ablated terms are 0 exactly as the
    // reference zeroes them
    if (!is_lru) {
      const double p2 = variant == CACE_MINUS_P2 ? 0.0 : K.p2[mm];
      const double p4 = variant == CACE_MINUS_P4 ? 0.0 : sc.w1 * (K.tok[mm] / norm);
      if (!WIDE) {
        S.p4d[mm * st] = p4;
        S.p4f[mm * st] = (float)(p2 + p4);
      }
      const double b = WIDE ? fabs(p2) + fabs(p4) : fabs(p2 + p4);
      screen_ok = screen_ok && b <= 1e5;  // false for NaN / inf
      if (screen_ok) tbound = fmaxf(tbound, 2.0f + (float)b);
    }
  }
  if (WIDE && writer) {
    // fp32 p2 + p4 = fma(p4s, tokens, p2s * p2): the roundings of p2, w1 /
    // normalizer and the fma add <= 2^-22 (|p2| + |p4|) to the screen's
    // error, covered by the doubled coefficient of the margin below
    S.wprm[0] = variant == CACE_MINUS_P2 ? 0.0f : 1.0f;
    S.wprm[st] = variant == CACE_MINUS_P4 ? 0.0f : (float)(sc.w1 / norm);
  }
  // screen constants live in shared memory: read only by deciding lanes, so
  // they hold no registers across the replay loop
  // (fp32 p1 = p1s * p1v + p1o: verbatim p1v, prose 1 - p1v, ablated 0)
  if (writer) {
    S.ud[0] = sc.unload_time_s;  // read on evictions only
    S.prm[0] = 1.0f / (float)sc.window_length;
    S.prm[st] = variant == CACE_MINUS_P1 ? 0.0f : (verbatim ? 1.0f : -1.0f);
    S.prm[2 * st] = variant == CACE_MINUS_P1 || verbatim ? 0.0f : 1.0f;
    S.prm[3 * st] = screen_ok ? 6e-5f + (WIDE ? 2e-6f : 1e-6f) * (tbound + 4.0f) : INFINITY;
  }
#ifndef CACE_HOST_EMULATION
  if (WIDE) __syncwarp();  // the leaders' column set-up precedes every lane's reads
#endif

  int dslot = -1;
  int64_t doff = 0, dn_ev = 0;
  bool dump_outcomes = false;
  double* samples = nullptr;  // this scenario's metrics samples
  uint32_t ncomp_t = 0;
  if (DM != 0 && !shadow && lig == 0) {  // one lane of a group writes
    dslot = P.dump.slot[sidx];
    if (dslot >= 0) doff = P.dump.dump_off[dslot];
    if (DM == 1)
      dump_outcomes = P.dump.cold || P.dump.queue_wait || P.dump.load_wait || P.dump.prefill ||
                      P.dump.decode || P.dump.ttft || P.dump.e2e;
    if (dslot >= 0 && P.dump.samples) samples = P.dump.samples + doff;
  }
  if (DM != 0) ncomp_t = P.trace_ncomp[sc.trace];
#ifndef CACE_HOST_EMULATION
  if (DM == 2 || (DM == 1 && P.dump.samples)) {  // the sample tile's pointer table (shadows too: flushes are collective)
    reinterpret_cast<double**>(S.samp + 2 * kSampT * 32)[threadIdx.x & 31] = samples;
    if ((threadIdx.x & 31) == 0) *reinterpret_cast<uint32_t*>(S.samp + 2 * kSampT * 32 + 32) = ncomp_t;
    __syncwarp();
  }
#endif
  RecStream rs;
  rs.init(tr, n, S.rec, S.rbar);
  Window<MW> win;
  if (C > 1 && warp_win) win.init(P.first0 + (int64_t)sc.trace * M, M, tr, n, S.win);

  // Slots [0, occ) are resident (shared slot table); there is no eager
  // per-slot state machine: a slot is Busy until its ServiceComplete key
  // passes the cursor (sc_popped), and then Idle with last_used_s = done
  // (a completion sets last_used to its own event time, engine.cpp:219-230;
  // the only Loading slot is the head's own, which is served the moment its
  // LoadComplete pops).
  int occ = 0;
  double ct = -INFINITY;  // cursor time
  uint32_t cw = kKindArr;  // cursor kind << 30 | seq

  // loads == misses == n - hits; evictions == loads - final occupancy.
  uint32_t hits = 0;
  double sttft = 0.0, se2e = 0.0, mttft = 0.0, me2e = 0.0;
  uint64_t ho = CACE_HASH_SEED;
  double lo_sum = 0.0;
  uint64_t he = CACE_HASH_SEED;

  for (uint32_t c = 0, k = 0; k < n; ++c) {
  const ReqRec* const cb = rs.chunk(c);
  const uint32_t kend = n - k < 32 ? n : k + 32;
  for (const ReqRec* rp = cb; k < kend; ++k, ++rp) {
    const ReqRec& R = *rp;
    const double a = R.arrival, pf = R.prefill, dc = R.decode;
    const uint32_t mc = R.mc;
    const int m = (int)(mc & 0xffffu);

    // Head not yet pending: the next relevant event is its Arrival (a, 2, k);
    // completions with a smaller key only idle their slots (engine.cpp:219-230).
    if (!(a < ct)) {
      ct = a;
      cw = kKindArr | k;
    }

    // classify (engine.cpp:163-173): resident (never Loading here) -> hit
    int hs = (int)S.slot_of[m * st] - 1;
    double lw = 0.0;
    const bool hit = hs >= 0;
    if (hit) {
      ++hits;
      CACE_STAT(0, k);
      // Busy: blocked until the model's own ServiceComplete (td, 1, tq)
      // (engine.cpp:175-181); every earlier completion just idles its slot.
      const SlotEnt te = S.slot[hs * st];  // one 16-B load
      const double td = te.done;
      const uint32_t tq = te.seq;
      if (!sc_popped<!WIDE>(td, tq, ct, cw)) {
        ct = td;
        cw = kKindSC | tq;
      }
    } else {
      int v;
      double ud = 0.0;
      if (occ < cap) {  // free slot, no unload delay (engine.cpp:184-187)
        v = occ++;
        if (WIDE) __syncwarp(gmask);  // the group's reads of slot_of precede the leader's writes
      } else {
        CACE_STAT(1, k);
        if constexpr (!WIDE) {
        // Full: the Idle residents are the eviction candidates
        // (engine.cpp:189-208, policy.cpp:85-89).
        double sd[C];
        uint32_t sq[C];
        int sw[C];
        unsigned idm = 0;
#pragma unroll
        for (int s = 0; s < C; ++s) {
          if ((WIDE || RTC) && s >= cap) break;
          const SlotEnt e = S.slot[s * st];
          sd[s] = e.done;
          sq[s] = e.seq;
          sw[s] = e.word;
          idm |= sc_popped<!WIDE>(e.done, e.seq, ct, cw) ? (1u << s) : 0u;
        }
        if (idm == 0) {
          // every resident busy: nothing to evict now (select_victim ->
          // nullopt); the next event is the min-key ServiceComplete, whose
          // slot is then the only Idle one (forced victim).
          int s1 = 0;
          double t1 = sd[0];
          uint32_t q1 = sq[0];
#pragma unroll
          for (int s = 1; s < C; ++s) {
            if ((WIDE || RTC) && s >= cap) break;
            if (sd[s] < t1 || (sd[s] == t1 && sq[s] < q1)) {
              s1 = s;
              t1 = sd[s];
              q1 = sq[s];
            }
          }
          ct = t1;
          cw = kKindSC | q1;
          v = s1;
          CACE_STAT(2, k);
        } else if ((idm & (idm - 1u)) == 0) {
          v = __ffs(idm) - 1;  // exactly one candidate
          CACE_STAT(3, k);
        } else {
          // ---- eviction decision among >= 2 idle residents ----------
          const double now = ct;
          CACE_STAT(4, k);
          if (is_lru) {
            // sorted-first = min (last_used, lex) over idle (policy.cpp:92-100)
            int f = -1;
            double flu = 0.0;
            int flex = 0;
#pragma unroll
            for (int s = 0; s < C; ++s) {
              if ((WIDE || RTC) && s >= cap) break;
              const int lx = slot_lex(sw[s]);
              if ((idm >> s) & 1u)
                if (f < 0 || sd[s] < flu || (sd[s] == flu && lx < flex)) {
                  f = s;
                  flu = sd[s];
                  flex = lx;
                }
            }
            v = f;
          } else {
            // p3 (policy.cpp:57-64): rank / w when the model's first pending
            // request lies in the window [k, min(k + w, arrived)), else 1.
            // Idle residents are not the head's model, so first > k.
            // fp32 screening with a rigorous bound: if one candidate's
            // approximate total beats every other by more than the bound it
            // is the exact arg-max.  |dL| <= 2.3e-5 (lg2.approx, ln t < 70)
            // propagates with Lipschitz constant 1 through 1/(1+L); the
            // approximate reciprocal, rank*(1/w), p4 = w1*tok*(1/norm), the
            // term conversions and three fp32 sums add <= 2^-21 (|T| + 4).
            // The margin is twice the worst case.
            const float rcpw = S.prm[0], p1s = S.prm[st], p1o = S.prm[2 * st];
            const float p2s = WIDE ? S.wprm[0] : 0.0f, p4s = WIDE ? S.wprm[st] : 0.0f;
            float best = -INFINITY, second = -INFINITY;
            int bs = 0;
            float Ts[C];  // screened totals (the exact pass skips the hopeless ones)
            const uint32_t wend = k + w;
#pragma unroll
            for (int s = 0; s < C; ++s) {
              Ts[s] = -INFINITY;
              if ((WIDE || RTC) && s >= cap) break;
              const int ms = slot_model(sw[s]);
              const float t = fmaxf((float)(now - sd[s]), 1.0f);  // max(d, 1) in fp32
              const float p1v = fast_rcp(fmaf(fast_lg2(t), kLn2f, 1.0f));
              const float p1 = fmaf(p1s, p1v, p1o);
              float p3 = 0.0f;
              if (need_win) {
                const WinEnt e = win.gather(ms);
                p3 = (e.f < wend && e.fa < now) ? e.r * rcpw : 1.0f;
              }
              float T = (p1 + p3) + (WIDE ? fmaf(p4s, K.tokf[ms], p2s * K.p2f[ms])
                                          : S.p4f[ms * st]);  // p2 + p4 pre-summed
              T = ((idm >> s) & 1u) ? T : -INFINITY;
              Ts[s] = T;
              bs = T > best ? s : bs;
              second = fmaxf(second, fminf(best, T));
              best = fmaxf(best, T);
            }
            v = bs;
            const float margin = S.prm[3 * st];
            if (!(best - second > margin)) {
              CACE_STAT(5, k);
              // Only candidates whose screened total is within the margin of
              // the best can be the exact arg-max: every screened total is
              // within margin / 2 of its exact value, so T_s < best - margin
              // means exact_s < exact_best.  (No pruning when the screen is
              // off -- infinite margin, possibly non-finite totals.)
              // Measured: +4% on deep sweeps (per-capacity, rolled exact
              // path); -2..-5% in the latency (unrolled) and mixed-capacity
              // instantiations, which keep the full candidate set.
              constexpr bool kPrune = XR && !RTC;  // mixed-capacity: -15% with it (ab_rtc_prune_r2ao)
              unsigned idx = idm;
              if (kPrune) {
                const float thr = margin < INFINITY ? best - margin : -INFINITY;
                unsigned near = 0;
#pragma unroll
                for (int s = 0; s < C; ++s)
                  if (!(Ts[s] < thr)) near |= 1u << s;
                idx &= near;
              }
              // Exact fp64 eviction_score (policy.cpp:39-78) and "first
              // strict max in (last_used, model_id) order"
              // (policy.cpp:92-113), bit-identical to the reference; taken on
              // near-ties (3-11% of CACE decisions are exact ties).
              // One pass: the best non-NaN total, ties to the earlier entry in
              // (last_used, lex) order; a NaN sorted-first entry keeps the
              // slot (no later total compares greater than NaN).
              int f = -1;
              double flu = 0.0;
              int flex = 0;
              bool f_nan = false;
              double bt = 0.0, blu = 0.0;
              int blex = 0, bv = -1;
              // candidates that went idle at the same event share last_used
              // and hence p1 (same-time completions are common): one log each
              double c_lu = -1.0, c_p1 = 0.0;
              auto cand = [&](int s, double lu, int wd) {
                const int ms = slot_model(wd);
                const int lx = slot_lex(wd);
                if (f < 0 || lu < flu || (lu == flu && lx < flex)) {  // sorted-first so far
                  f = s;
                  flu = lu;
                  flex = lx;
                }
                // (rolled instantiations; the latency one measured 3% slower with it)
                if (variant != CACE_MINUS_P1 && (!XR || lu != c_lu)) {
                  c_lu = lu;
                  c_p1 = exact_p1(now, lu, verbatim, P.log_variant, P.log_tab, P.log_tab2);
                }
                const double p1 = variant == CACE_MINUS_P1 ? 0.0 : c_p1;
                const double p2 = variant == CACE_MINUS_P2 ? 0.0 : K.p2[ms];
                double p3 = 0.0;
                if (variant != CACE_MINUS_P3) {
                  const WinEnt e = win.gather(ms);
                  p3 = (e.f - k < w && e.fa < now) ? (double)e.r / (double)w : 1.0;
                }
                const double p4 = !WIDE ? S.p4d[ms * st]
                                        : (variant == CACE_MINUS_P4 ? 0.0 : sc.w1 * (K.tok[ms] / norm));
                const double T = ((p1 + p2) + p3) + p4;
                if (T == T && (bv < 0 || T > bt || (T == bt && (lu < blu || (lu == blu && lx < blex))))) {
                  bt = T;
                  blu = lu;
                  blex = lx;
                  bv = s;
                }
                return T != T;
              };
              unsigned nanm = 0;
              if constexpr (XR) {
                // Exact-tie shortcut: when every remaining candidate has the
                // same last_used (so the same p1), p3 = 1 (first pending
                // request outside the window or not arrived) and the same p2
                // and p4, all exact totals are bitwise equal and the reference
                // keeps the first in (last_used, model_id) order: the least
                // lex rank.  (Same-class models of a pool share load time and
                // expected tokens; same-time completions share last_used.)
                bool tie = kPrune;
                double lu0 = 0.0, p20 = 0.0, p40 = 0.0;
                int tlex = 0x7fffffff, ts = -1;
#pragma unroll 1
                for (unsigned q = idx; tie && q; q &= q - 1u) {
                  const int s = __ffs(q) - 1;
                  const double lu = S.slot[s * st].done;
                  const int wd = S.slot[s * st].word;
                  const int ms = slot_model(wd);
                  const double p2 = variant == CACE_MINUS_P2 ? 0.0 : K.p2[ms];
                  const double p4 = S.p4d[ms * st];
                  bool p3one = true;
                  if (variant != CACE_MINUS_P3) {
                    const WinEnt e = win.gather(ms);
                    p3one = !(e.f - k < w && e.fa < now);
                  }
                  if (ts < 0) {
                    lu0 = lu;
                    p20 = p2;
                    p40 = p4;
                  }
                  tie = p3one && lu == lu0 && p2 == p20 && p4 == p40;
                  if (slot_lex(wd) < tlex) {
                    tlex = slot_lex(wd);
                    ts = s;
                  }
                }
                if (tie) {
                  f = ts;  // sorted-first; no NaN with the screen on
                  bv = ts;
                } else {
#pragma unroll 1
                  for (unsigned q = idx; q; q &= q - 1u) {
                    const int s = __ffs(q) - 1;
                    if (cand(s, S.slot[s * st].done, S.slot[s * st].word)) nanm |= 1u << s;
                  }
                }
              } else {
#pragma unroll
                for (int s = 0; s < C; ++s)
                  if ((idx >> s) & 1u)
                    if (cand(s, sd[s], sw[s])) nanm |= 1u << s;
              }
              f_nan = (nanm >> f) & 1u;
              v = f_nan ? f : bv;
            }
          }
        }
        } else {
          // ---- wide pools: the scenario's G lanes split its slots (lane
          // lig owns slots lig + G j) and combine partial results with
          // shuffles inside the group ----
          constexpr int J = C / G;
          double ld[J];
          uint32_t lq[J];
          int lwd[J];
          unsigned idm = 0;
#pragma unroll
          for (int j = 0; j < J; ++j) {
            const int s = lig + G * j;
            ld[j] = INFINITY;
            lq[j] = 0xffffffffu;
            lwd[j] = 0;
            if (s < cap) {
              const SlotEnt e = S.slot[s * st];
              ld[j] = e.done;
              lq[j] = e.seq;
              lwd[j] = e.word;
              idm |= sc_popped<!WIDE>(e.done, e.seq, ct, cw) ? (1u << s) : 0u;
            }
          }
#pragma unroll
          for (int o = 1; o < G; o <<= 1) idm |= __shfl_xor_sync(gmask, idm, o);
          if (idm == 0) {
            // every resident busy: the min-key ServiceComplete's slot
            double t1 = INFINITY;
            uint32_t q1 = 0xffffffffu;
            int s1 = 0;
#pragma unroll
            for (int j = 0; j < J; ++j)
              if (ld[j] < t1 || (ld[j] == t1 && lq[j] < q1)) {
                t1 = ld[j];
                q1 = lq[j];
                s1 = lig + G * j;
              }
#pragma unroll
            for (int o = 1; o < G; o <<= 1) {
              const double ot = __shfl_xor_sync(gmask, t1, o);
              const uint32_t oq = __shfl_xor_sync(gmask, q1, o);
              const int os = __shfl_xor_sync(gmask, s1, o);
              if (ot < t1 || (ot == t1 && oq < q1)) {
                t1 = ot;
                q1 = oq;
                s1 = os;
              }
            }
            ct = t1;
            cw = kKindSC | q1;
            v = s1;
          } else if ((idm & (idm - 1u)) == 0) {
            v = __ffs(idm) - 1;  // exactly one candidate
          } else {
            const double now = ct;
            if (is_lru) {
              // sorted-first = min (last_used, lex) over idle (policy.cpp:92-100)
              double flu = INFINITY;
              int flex = 0x7fffffff, f = 0;
#pragma unroll
              for (int j = 0; j < J; ++j) {
                const int s = lig + G * j;
                const int lx = slot_lex(lwd[j]);
                if ((idm >> s) & 1u)
                  if (ld[j] < flu || (ld[j] == flu && lx < flex)) {
                    flu = ld[j];
                    flex = lx;
                    f = s;
                  }
              }
#pragma unroll
              for (int o = 1; o < G; o <<= 1) {
                const double ou = __shfl_xor_sync(gmask, flu, o);
                const int ox = __shfl_xor_sync(gmask, flex, o);
                const int of = __shfl_xor_sync(gmask, f, o);
                if (ou < flu || (ou == flu && ox < flex)) {
                  flu = ou;
                  flex = ox;
                  f = of;
                }
              }
              v = f;
            } else {
              // fp32 screen over the lane's own idle slots, then the group's
              // (best, second, arg-best); the margin test is as in the
              // one-lane path (an fp32 tie leaves best - second = 0)
              const float rcpw = S.prm[0], p1s = S.prm[st], p1o = S.prm[2 * st];
              const float p2s = S.wprm[0], p4s = S.wprm[st];
              float best = -INFINITY, second = -INFINITY;
              int bs = 0x7fffffff;
              float Tj[J];  // the lane's screened totals (exact-pass pruning)
              const uint32_t wend = k + w;
#pragma unroll
              for (int j = 0; j < J; ++j) {
                const int s = lig + G * j;
                Tj[j] = -INFINITY;
                if (!((idm >> s) & 1u)) continue;
                const int ms = slot_model(lwd[j]);
                const float t = fmaxf((float)(now - ld[j]), 1.0f);  // max(d, 1) in fp32
                const float p1v = fast_rcp(fmaf(fast_lg2(t), kLn2f, 1.0f));
                const float p1 = fmaf(p1s, p1v, p1o);
                float p3 = 0.0f;
                if (need_win) {
                  const WinEnt e = win.gather128(ms);
                  p3 = (e.f < wend && e.fa < now) ? e.r * rcpw : 1.0f;
                }
                const float T = (p1 + p3) + fmaf(p4s, K.tokf[ms], p2s * K.p2f[ms]);
                Tj[j] = T;
                bs = T > best ? s : bs;
                second = fmaxf(second, fminf(best, T));
                best = fmaxf(best, T);
              }
#pragma unroll
              for (int o = 1; o < G; o <<= 1) {
                const float ob = __shfl_xor_sync(gmask, best, o);
                const float os2 = __shfl_xor_sync(gmask, second, o);
                const int obs = __shfl_xor_sync(gmask, bs, o);
                second = fmaxf(fmaxf(second, os2), fminf(best, ob));
                bs = best > ob ? bs : (ob > best ? obs : (obs < bs ? obs : bs));
                best = fmaxf(best, ob);
              }
              v = bs;
              const float margin = S.prm[3 * st];
              if (!(best - second > margin)) {
                // exact fp64 path (policy.cpp:39-78, 92-113): every lane of
                // the group walks the idle slots (identical result, no
                // reduction) -- only those whose screened total is within the
                // margin of the best (the group ORs its lanes' masks; no
                // pruning with the screen off), one glibc log per distinct
                // last_used
                unsigned idx = idm;
                if (margin < INFINITY) {
                  const float thr = best - margin;
                  unsigned near = 0;
#pragma unroll
                  for (int j = 0; j < J; ++j)
                    if (!(Tj[j] < thr)) near |= 1u << (lig + G * j);
#pragma unroll
                  for (int o = 1; o < G; o <<= 1) near |= __shfl_xor_sync(gmask, near, o);
                  idx &= near;
                }
                int f = -1;
                double flu = 0.0;
                int flex = 0;
                double bt = 0.0, blu = 0.0;
                int blex = 0, bv = -1;
                bool f_nan = false;
                double c_lu = -1.0, c_p1 = 0.0;
#pragma unroll 1
                for (unsigned q = idx; q; q &= q - 1u) {
                  const int s = __ffs(q) - 1;
                  const double lu = S.slot[s * st].done;
                  const int wd = S.slot[s * st].word;
                  const int ms = slot_model(wd);
                  const int lx = slot_lex(wd);
                  if (variant != CACE_MINUS_P1 && lu != c_lu) {
                    c_lu = lu;
                    c_p1 = exact_p1(now, lu, verbatim, P.log_variant, P.log_tab, P.log_tab2);
                  }
                  const double p1 = variant == CACE_MINUS_P1 ? 0.0 : c_p1;
                  const double p2 = variant == CACE_MINUS_P2 ? 0.0 : K.p2[ms];
                  double p3 = 0.0;
                  if (variant != CACE_MINUS_P3) {
                    const WinEnt e = win.gather128(ms);
                    p3 = (e.f - k < w && e.fa < now) ? (double)e.r / (double)w : 1.0;
                  }
                  const double p4 = variant == CACE_MINUS_P4 ? 0.0 : sc.w1 * (K.tok[ms] / norm);
                  const double T = ((p1 + p2) + p3) + p4;
                  if (f < 0 || lu < flu || (lu == flu && lx < flex)) {  // sorted-first so far
                    f = s;
                    flu = lu;
                    flex = lx;
                    f_nan = T != T;
                  }
                  if (T == T && (bv < 0 || T > bt || (T == bt && (lu < blu || (lu == blu && lx < blex))))) {
                    bt = T;
                    blu = lu;
                    blex = lx;
                    bv = s;
                  }
                }
                v = f_nan ? f : bv;
              }
            }
          }
        }
        // residents.erase(victim); evictions++ (engine.cpp:205-206)
        const int vm = slot_model(S.slot[v * st].word);
        if (WIDE) __syncwarp(gmask);  // the group's reads of the slots precede the leader's writes
        if (writer) S.slot_of[vm * st] = 0;
        he = hmix(he, dbits(ct) ^ ((uint64_t)vm << 32));
        if (DM == 1 && dslot >= 0) {
          if (dn_ev < P.dump.evict_cap) {
            if (P.dump.evict_model) P.dump.evict_model[dslot * P.dump.evict_cap + dn_ev] = vm;
            if (P.dump.evict_clock) P.dump.evict_clock[dslot * P.dump.evict_cap + dn_ev] = ct;
          }
          ++dn_ev;
        }
        ud = S.ud[0];  // unload_time_s
      }
      // start_load (engine.cpp:123-132), then blocked until its LoadComplete
      // (r, 0, .): completions strictly before r idle their slots.
      const double lt = K.lt[m];
      const double r = (ct + ud) + lt;
      lw = r - ct;
      lo_sum += lt;
      if (writer) {
        S.slot[v * st].word = m | (K.lex[m] << 18);
        S.slot_of[m * st] = (uint8_t)(v + 1);
      }
      ct = r;
      cw = 0u;
      hs = v;
    }

    // start_service at now = ct (engine.cpp:134-153); its ServiceComplete is
    // pushed with seq k (services start once per request, in order)
    const double now = ct;
    const double qd = now - a;
    const double ttft = qd + pf;
    const double e2e = ttft + dc;
    const double done = (now + pf) + dc;
    if (WIDE) __syncwarp(gmask);  // the group's reads of slot hs precede the write
    if (writer) {
      SlotEnt* const sp = &S.slot[hs * st];  // one address for both stores
      sp->done = done;
      sp->seq = k;
    }
    if (WIDE) __syncwarp(gmask);  // visible to the group's reads of the next request
    if ((mc >> 16) == CACE_COMPLETION) {
      sttft += ttft;
      mttft = ttft > mttft ? ttft : mttft;
    } else {
      se2e += e2e;
      me2e = e2e > me2e ? e2e : me2e;
    }
    ho = hmix(ho, dbits(ttft) ^ (hit ? 0ull : 1ull));
    if (DM == 1 && dslot >= 0) {
      if (dump_outcomes) {  // per-request outcomes in the caller's request order
        const int64_t o = doff + P.perm[base + k];
        if (P.dump.cold) P.dump.cold[o] = hit ? 0 : 1;
        if (P.dump.queue_wait) P.dump.queue_wait[o] = qd - lw;
        if (P.dump.load_wait) P.dump.load_wait[o] = lw;
        if (P.dump.prefill) P.dump.prefill[o] = pf;
        if (P.dump.decode) P.dump.decode[o] = dc;
        if (P.dump.ttft) P.dump.ttft[o] = ttft;
        if (P.dump.e2e) P.dump.e2e[o] = e2e;
      }
    }
    // metrics samples (compute_run_metrics, metrics.cpp:44-52): TTFT of
    // completion requests, then E2E of reasoning requests
#ifndef CACE_HOST_EMULATION
    if (DM == 2 || (DM == 1 && P.dump.samples)) {  // warp-collective (shadow lanes take part, write nothing)
      const bool comp = (mc >> 16) == CACE_COMPLETION;
      const uint32_t ci = R.ci;
      double* tc = S.samp + (comp ? 0 : kSampT * 32);
      tc[(ci % kSampT) * 32 + (threadIdx.x & 31)] = comp ? ttft : e2e;
      if (ci % kSampT == kSampT - 1) {
        __syncwarp();
        flush_samples(tc, samp_ptrs(S.samp), (int64_t)(comp ? 0 : samp_ncomp(S.samp)) + ci - (kSampT - 1), kSampT);
        __syncwarp();
      }
    }
#else
    if (DM != 0 && samples) {
      const bool comp = (mc >> 16) == CACE_COMPLETION;
      samples[comp ? R.ci : ncomp_t + R.ci] = comp ? ttft : e2e;
    }
#endif
    if (C > 1 && warp_win) {  // the head leaves the window (collective)
      win.prepare(m, R.nxt);
      win.commit(R.nxa);
    }
  }
  }

  rs.fini();
#ifndef CACE_HOST_EMULATION
  if (DM == 2 || (DM == 1 && P.dump.samples)) {  // partial tiles
    const uint32_t nco = samp_ncomp(S.samp), nre = n - nco;
    __syncwarp();
    if (nco % kSampT) flush_samples(S.samp, samp_ptrs(S.samp), nco - nco % kSampT, nco % kSampT);
    if (nre % kSampT)
      flush_samples(S.samp + kSampT * 32, samp_ptrs(S.samp), (int64_t)nco + nre - nre % kSampT, nre % kSampT);
  }
#endif
  if (shadow || lig != 0) return;
  cace_summary_t o;
  o.hits = hits;
  o.misses = n - hits;
  o.evictions = n - hits - (uint32_t)occ;  // every load after the fill evicts
  o.loads = n - hits;                      // loads == misses (test_engine.cpp:168)
  o.load_overhead_s = lo_sum;
  o.max_resident = occ;
  o.status = CACE_OK;
  o.n_completion = P.trace_ncomp[sc.trace];
  o.n_reasoning = n - P.trace_ncomp[sc.trace];
  o.sum_ttft_completion = sttft;
  o.sum_e2e_reasoning = se2e;
  o.max_ttft_completion = mttft;
  o.max_e2e_reasoning = me2e;
  o.eviction_hash = he;
  o.outcome_hash = ho;
  P.out[sidx] = o;
  if (DM == 1 && dslot >= 0 && P.dump.n_evict) P.dump.n_evict[dslot] = dn_ev;
}

constexpr uint64_t kShadowBit = 1ull << 62;  // plan entry = warp padding lane
constexpr int kLaneMaxModels = 64;           // lane kernel: window in <= 2 registers/lane

#ifndef CACE_HOST_EMULATION
#ifndef CACE_LANE_BLOCK
#define CACE_LANE_BLOCK 128
#endif
constexpr int LANE_BLOCK = CACE_LANE_BLOCK;  // threads per lane block
// MINB counts 128-thread blocks per SM (the register target), whatever LANE_BLOCK is
constexpr int kLaneBlockScale = 128 / LANE_BLOCK;
#ifndef CACE_LANE_MIN_BLOCKS
#define CACE_LANE_MIN_BLOCKS 5  // <= 96 registers: 5 blocks (20 warps) per SM
#endif

// Dynamic shared memory of one lane block: catalog columns, per-lane columns
// [M or C][LANE_BLOCK], then per warp the record double buffer and the
// window table.
inline __host__ __device__ size_t lane_smem_cat(int M) { return (size_t)M * (3 * 8 + 2 * 4 + 4); }
// 16-B aligned start of the per-lane columns
inline __host__ __device__ size_t lane_smem_lane_off(int M) { return (lane_smem_cat(M) + 15) & ~(size_t)15; }
inline __host__ __device__ size_t lane_smem_lane(int M, int C) {
  return (size_t)LANE_BLOCK * ((M + 1) * 8 + C * sizeof(SlotEnt) + M * 4 + 4 * 4 + M);
}
inline __host__ __device__ size_t lane_smem_warp(int M, bool dump) {
  // records, window table, 2 mbarriers, sample tile: a 16-B multiple keeps the next warp's records aligned
  return 64 * sizeof(ReqRec) + (size_t)M * sizeof(WinEnt) + 16 +
         (dump ? (2 * kSampT * 32 + 32 + 2) * sizeof(double) : 0);
}
inline size_t lane_smem_bytes(int M, int C, bool dump) {
  const size_t a = (lane_smem_lane_off(M) + lane_smem_lane(M, C) + 15) & ~(size_t)15;
  return a + (LANE_BLOCK / 32) * lane_smem_warp(M, dump);
}

// MINB = resident blocks per SM the register allocation targets, picked by
// how many waves of lane warps the sweep is (capi.cu, measured on the B200,
// profiles/r2/ab_occupancy_*): CACE_LANE_MIN_BLOCKS (5: 20 warps/SM, 96
// registers) for deep sweeps, where issue throughput bounds the step; 4 (16
// warps/SM, 114 registers, no spills) for 1.5-4.5 waves; 3 (12 warps/SM, up
// to 168 registers, the exact fallback unrolled: the shortest per-request
// dependency chain) below 1.5 waves, where each warp's chain bounds the step.
#ifndef CACE_LANE_LAT_MINB
#define CACE_LANE_LAT_MINB 3
#endif
constexpr int kLaneLatencyMinBlocks = CACE_LANE_LAT_MINB;
constexpr int kLaneMidMinBlocks = 4;

// DM: 0 summary only; 1 full dump (outcomes, eviction log, samples) for the
// scenarios with a dump slot; 2 metrics samples only (the RunMetrics
// pipeline: no outcome / eviction-log code or registers).
// RTC: a mixed-capacity launch -- C is the bound, each warp's capacity is its
// scenarios' effective capacity (the plan keeps warps capacity-uniform).
template <int C, int MW, int DM, int MINB = CACE_LANE_MIN_BLOCKS, int MC = 0, bool RTC = false>
__global__ void __launch_bounds__(LANE_BLOCK, MINB * kLaneBlockScale) replay_lane_kernel(ReplayParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int M = MC > 0 ? MC : P.cat.M;  // MC: compile-time pool size (immediate shared offsets)
  double* s_lt = reinterpret_cast<double*>(smem);
  double* s_p2 = s_lt + M;
  double* s_tok = s_p2 + M;
  float* s_p2f = reinterpret_cast<float*>(s_tok + M);
  float* s_tokf = s_p2f + M;
  int* s_lex = reinterpret_cast<int*>(s_tokf + M);
  // per-lane columns: 8- and 16-B ones first
  double* l_p4d = reinterpret_cast<double*>(smem + lane_smem_lane_off(M));                  // [M + 1][LB]
  SlotEnt* l_slot = reinterpret_cast<SlotEnt*>(l_p4d + (size_t)(M + 1) * LANE_BLOCK);       // [C][LB]
  float* l_p4f = reinterpret_cast<float*>(l_slot + (size_t)C * LANE_BLOCK);                // [M][LB]
  float* l_prm = l_p4f + (size_t)M * LANE_BLOCK;                                           // [4][LB]
  uint8_t* l_sof = reinterpret_cast<uint8_t*>(l_prm + (size_t)4 * LANE_BLOCK);            // [M][LB]
  unsigned char* wbase = smem + ((lane_smem_lane_off(M) + lane_smem_lane(M, C) + 15) & ~(size_t)15) +
                         (size_t)(threadIdx.x >> 5) * lane_smem_warp(M, DM != 0);
  ReqRec* w_rec = reinterpret_cast<ReqRec*>(wbase);
  WinEnt* w_win = reinterpret_cast<WinEnt*>(w_rec + 64);
  uint64_t* w_bar = reinterpret_cast<uint64_t*>(w_win + M);
  double* w_samp = reinterpret_cast<double*>(w_bar + 2);
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    s_lt[m] = P.cat.load_time[m];
    s_p2[m] = P.cat.p2[m];
    s_tok[m] = P.cat.tokens[m];
    s_p2f[m] = (float)P.cat.p2[m];
    s_tokf[m] = (float)P.cat.tokens[m];
    s_lex[m] = P.cat.lex[m];
  }
  __syncthreads();
  const int64_t gi = P.seg_begin + (int64_t)blockIdx.x * LANE_BLOCK + threadIdx.x;
  if (gi >= P.seg_end) return;  // whole warps: the plan pads groups to whole warps
  const uint64_t e = (uint64_t)P.order[gi];
  const bool shadow = (e & kShadowBit) != 0;
  const int64_t sidx = (int64_t)(e & (kShadowBit - 1));
  const cace_scenario_t& scn = P.scen[sidx];
  const int variant = scn.variant;
  const bool need_win = variant != CACE_LRU && variant != CACE_MINUS_P3;
  const int cap = RTC ? (int)min((int64_t)scn.num_accelerators * scn.models_per_accelerator, (int64_t)M) : C;
  // With capacity >= pool size every model fits: no eviction decision ever
  // happens, so the lookahead window is never read and is not maintained.
  const bool warp_win = __any_sync(kFull, need_win) && cap > 1 && cap < M;
  const CatShared K{s_lt, s_p2, s_tok, s_p2f, s_tokf, s_lex};
  const LaneSmem S{l_p4f + threadIdx.x, l_p4d + threadIdx.x, l_slot + threadIdx.x, l_prm + threadIdx.x,
                   l_p4d + (size_t)M * LANE_BLOCK + threadIdx.x, nullptr, l_sof + threadIdx.x, LANE_BLOCK,
                   w_rec, w_win, w_samp, w_bar};
  replay_scenario<C, MW, DM, MINB != kLaneLatencyMinBlocks, false, 1, MC, RTC>(P, sidx, shadow, warp_win, K, S,
                                                                             cap);
}

// ---- wide pools / capacities ----------------------------------------------
// Pools of up to 256 models (window in MW <= 8 registers per lane) and
// capacities up to kWideC: the lane-per-scenario replay with the capacity a
// runtime value under an unroll bound of kWideC, no per-lane p2 + p4 tables
// (replay_scenario<..., WIDE>), and a GROUP of G lanes per scenario: lane lig
// of a group owns slots lig + G j, so an eviction decision scans C / G slots
// per lane and combines the group's partial results with log2(G) shuffle
// rounds (BASELINE config 5: capacity 32, 8 lanes x 4 slots).  A warp holds
// 32 / G scenarios of one trace; the lookahead window stays warp-wide.
constexpr int LANE_BLOCK_WIDE = 128;
constexpr int kWideC = 32;
constexpr int kWideMaxModels = 256;
inline __host__ __device__ size_t lane_wide_lane(int M, int G) {
  return (size_t)(LANE_BLOCK_WIDE / G) * (kWideC * sizeof(SlotEnt) + 8 + 4 * 4 + 2 * 4 + M);
}
inline size_t lane_wide_smem_bytes(int M, bool dump, int G) {
  const size_t a = (lane_smem_lane_off(M) + lane_wide_lane(M, G) + 15) & ~(size_t)15;
  return a + (LANE_BLOCK_WIDE / 32) * lane_smem_warp(M, dump);
}

template <int MW, int DM, int G>
__global__ void __launch_bounds__(LANE_BLOCK_WIDE, 4) replay_lane_wide_kernel(ReplayParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int C = kWideC, SB = LANE_BLOCK_WIDE / G;  // scenarios per block
  const int M = P.cat.M;
  double* s_lt = reinterpret_cast<double*>(smem);
  double* s_p2 = s_lt + M;
  double* s_tok = s_p2 + M;
  float* s_p2f = reinterpret_cast<float*>(s_tok + M);
  float* s_tokf = s_p2f + M;
  int* s_lex = reinterpret_cast<int*>(s_tokf + M);
  // per-scenario columns (SB wide), shared by the scenario's G lanes
  SlotEnt* l_slot = reinterpret_cast<SlotEnt*>(smem + lane_smem_lane_off(M));  // [C][SB]
  double* l_ud = reinterpret_cast<double*>(l_slot + (size_t)C * SB);          // [1][SB]
  float* l_prm = reinterpret_cast<float*>(l_ud + SB);                         // [4][SB]
  float* l_wprm = l_prm + 4 * SB;                                             // [2][SB]
  uint8_t* l_sof = reinterpret_cast<uint8_t*>(l_wprm + 2 * SB);               // [M][SB]
  unsigned char* wbase = smem + ((lane_smem_lane_off(M) + lane_wide_lane(M, G) + 15) & ~(size_t)15) +
                         (size_t)(threadIdx.x >> 5) * lane_smem_warp(M, DM != 0);
  ReqRec* w_rec = reinterpret_cast<ReqRec*>(wbase);
  WinEnt* w_win = reinterpret_cast<WinEnt*>(w_rec + 64);
  uint64_t* w_bar = reinterpret_cast<uint64_t*>(w_win + M);
  double* w_samp = reinterpret_cast<double*>(w_bar + 2);
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    s_lt[m] = P.cat.load_time[m];
    s_p2[m] = P.cat.p2[m];
    s_tok[m] = P.cat.tokens[m];
    s_p2f[m] = (float)P.cat.p2[m];
    s_tokf[m] = (float)P.cat.tokens[m];
    s_lex[m] = P.cat.lex[m];
  }
  __syncthreads();
  const int col = threadIdx.x / G;  // the scenario's column in the block
  const int64_t gi = P.seg_begin + (int64_t)blockIdx.x * SB + col;
  const int64_t wfirst = P.seg_begin + (int64_t)blockIdx.x * SB + (threadIdx.x & ~31) / G;
  if (wfirst >= P.seg_end) return;  // whole warps (the plan pads groups to 32 scenarios)
  const uint64_t e = (uint64_t)P.order[gi];
  const bool shadow = (e & kShadowBit) != 0;
  const int64_t sidx = (int64_t)(e & (kShadowBit - 1));
  const cace_scenario_t& sc = P.scen[sidx];
  const int variant = sc.variant;
  // the warp's scenarios share the effective capacity (planner groups by it)
  const int cap = (int)min((int64_t)sc.num_accelerators * sc.models_per_accelerator, (int64_t)M);
  const bool need_win = variant != CACE_LRU && variant != CACE_MINUS_P3;
  const bool warp_win = __any_sync(kFull, need_win) && cap > 1 && cap < M;
  const CatShared K{s_lt, s_p2, s_tok, s_p2f, s_tokf, s_lex};
  const LaneSmem S{nullptr, nullptr, l_slot + col, l_prm + col, l_ud + col, l_wprm + col, l_sof + col, SB,
                   w_rec, w_win, w_samp, w_bar};
  replay_scenario<C, MW, DM, true, true, G>(P, sidx, shadow, warp_win, K, S, cap);
}
#endif  // CACE_HOST_EMULATION

}  // namespace cace

