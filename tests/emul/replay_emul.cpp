// TEST-ONLY host emulation of the replay kernel's device code.
//
// Compiles paper_2506_18796_b200/csrc/replay_lane.cuh's per-lane replay
// (replay_scenario<C>) as ordinary host C++ by shimming the handful of CUDA
// intrinsics it uses, so the engine's event algebra can be checked against
// the reference oracle on a CPU-only box.  This library is never loaded by
// the product (which has no CPU fallback); it exists only for tests/.
#include <math.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#define CACE_HOST_EMULATION 1
#define __device__
#define __host__
#define __global__
#define __forceinline__ inline
#define __noinline__
#define __launch_bounds__(...)
struct uint4 { unsigned x, y, z, w; };
template <typename T> static inline T __ldg(const T* p) { return *p; }
static inline double __hiloint2double(int hi, int lo) {
  uint64_t u = ((uint64_t)(uint32_t)hi << 32) | (uint32_t)lo;
  double d;
  std::memcpy(&d, &u, 8);
  return d;
}
static inline long long __double_as_longlong(double d) { long long u; std::memcpy(&u, &d, 8); return u; }
static inline int __double2hiint(double d) { return (int)(__double_as_longlong(d) >> 32); }
static inline unsigned __float_as_uint(float f) { unsigned u; std::memcpy(&u, &f, 4); return u; }
#define __logf(x) logf(x)
static inline float __fdividef(float a, float b) { return a / b; }
static inline int __ffs(unsigned x) { return __builtin_ffs((int)x); }
template <typename T> static inline T __shfl_xor_sync(unsigned, T x, int) { return x; }  // groups of one lane
static inline void __syncwarp(unsigned = 0xffffffffu) {}

#include "../../paper_2506_18796_b200/csrc/replay_lane.cuh"
#include "../../paper_2506_18796_b200/csrc/layout.hpp"

using namespace cace;

static const double kTab[256] = CACE_GLIBC_LOG_TAB;
static const double kTab2[256] = CACE_GLIBC_LOG_TAB2;

static int g_xr = 1;  // exact fallback variant: 1 rolled (16-warp kernels), 0 unrolled (12-warp)

template <int C, bool D>
static void one(const ReplayParams& P, int64_t i, const CatShared& K) {
  const int v = P.scen[i].variant;
  const bool need_win = v != CACE_LRU && v != CACE_MINUS_P3;
  std::vector<float> p4f(P.cat.M), prm(4);
  std::vector<double> p4d(P.cat.M + 1);
  std::vector<SlotEnt> slot(C);
  std::vector<uint8_t> slot_of(P.cat.M);
  const LaneSmem S{p4f.data(), p4d.data(), slot.data(), prm.data(), p4d.data() + P.cat.M, nullptr, slot_of.data(),
                   1, nullptr, nullptr, nullptr, nullptr};
  if (g_xr)
    replay_scenario<C, 2, D, true>(P, i, false, need_win, K, S);
  else
    replay_scenario<C, 2, D, false>(P, i, false, need_win, K, S);
}

// The mixed-capacity (runtime capacity <= 8) one-lane mode of shallow sweeps.
template <bool D>
static void one_rtc(const ReplayParams& P, int64_t i, const CatShared& K, int cap) {
  const int v = P.scen[i].variant;
  const bool need_win = v != CACE_LRU && v != CACE_MINUS_P3;
  std::vector<float> p4f(P.cat.M), prm(4);
  std::vector<double> p4d(P.cat.M + 1);
  std::vector<SlotEnt> slot(8);
  std::vector<uint8_t> slot_of(P.cat.M);
  const LaneSmem S{p4f.data(), p4d.data(), slot.data(), prm.data(), p4d.data() + P.cat.M, nullptr, slot_of.data(),
                   1, nullptr, nullptr, nullptr, nullptr};
  const bool win = need_win && cap > 1 && cap < P.cat.M;
  if (g_xr)
    replay_scenario<8, 2, D, true, false, 1, 0, true>(P, i, false, win, K, S, cap);
  else
    replay_scenario<8, 2, D, false, false, 1, 0, true>(P, i, false, win, K, S, cap);
}

// The wide-pool mode (pools up to 256 models, capacity <= 32 at run time).
template <bool D>
static void one_wide(const ReplayParams& P, int64_t i, const CatShared& K, int cap) {
  const int v = P.scen[i].variant;
  const bool need_win = v != CACE_LRU && v != CACE_MINUS_P3;
  std::vector<float> prm(4), wprm(2);
  std::vector<double> ud(1);
  std::vector<SlotEnt> slot(32);
  std::vector<uint8_t> slot_of(P.cat.M);
  const LaneSmem S{nullptr, nullptr, slot.data(), prm.data(), ud.data(), wprm.data(), slot_of.data(), 1,
                   nullptr, nullptr, nullptr, nullptr};
  if (g_xr)
    replay_scenario<32, 8, D, true, true>(P, i, false, need_win && cap < P.cat.M, K, S, cap);
  else
    replay_scenario<32, 8, D, false, true>(P, i, false, need_win && cap < P.cat.M, K, S, cap);
}

extern "C" int32_t emul_replay_batch(const cace_catalog_t* catalog, const cace_trace_t* traces,
                                     int32_t n_traces, const cace_scenario_t* sc, int64_t n,
                                     cace_summary_t* out, int32_t log_variant,
                                     const int32_t* dump_slot, const int64_t* dump_off,
                                     uint8_t* cold, double* ttft, double* e2e, double* qw, double* lw,
                                     int64_t evict_cap, int32_t* evict_model, double* evict_clock,
                                     int64_t* n_evict, int32_t xr, int32_t wide) {
  g_xr = xr;
  try {
    HostCatalog cat;
    cat.load(catalog);
    HostLayout lay;
    build_layout(cat, traces, n_traces, lay);
    std::vector<int32_t> lex(cat.lex.begin(), cat.lex.end());
    ReplayParams P{};
    P.rec = lay.rec.data();
    P.trace_off = lay.off.data();
    P.first0 = lay.first0.data();
    P.perm = lay.perm.data();
    P.trace_ncomp = lay.ncomp.data();
    P.cat = DevCatalog{cat.M, cat.lt.data(), cat.p2.data(), cat.tok.data(), lex.data()};
    P.log_tab = kTab;
    P.log_tab2 = kTab2;
    P.log_variant = log_variant;
    P.scen = sc;
    P.out = out;
    P.dump.slot = dump_slot;
    P.dump.dump_off = dump_off;
    P.dump.cold = cold;
    P.dump.ttft = ttft;
    P.dump.e2e = e2e;
    P.dump.queue_wait = qw;
    P.dump.load_wait = lw;
    P.dump.evict_cap = evict_cap;
    P.dump.evict_model = evict_model;
    P.dump.evict_clock = evict_clock;
    P.dump.n_evict = n_evict;
    if (cat.M > 256) return CACE_E_INVALID;
    std::vector<float> p2f, tokf;
    for (int m = 0; m < cat.M; ++m) {
      p2f.push_back((float)cat.p2[m]);
      tokf.push_back((float)cat.tok[m]);
    }
    const CatShared K{cat.lt.data(), cat.p2.data(), cat.tok.data(), p2f.data(), tokf.data(), lex.data()};
    for (int64_t i = 0; i < n; ++i) {
      const int32_t st = precheck(lay, sc[i]);
      const int64_t len = (sc[i].trace >= 0 && sc[i].trace < lay.T) ? lay.off[sc[i].trace + 1] - lay.off[sc[i].trace] : 0;
      if (st != CACE_OK || len == 0) {
        std::memset(&out[i], 0, sizeof(cace_summary_t));
        out[i].status = st;
        out[i].eviction_hash = out[i].outcome_hash = CACE_HASH_SEED;
        continue;
      }
      const int Cap = (int)effective_capacity(sc[i], cat.M);
      const bool D = dump_slot != nullptr;
      if (wide == 2 && Cap <= 8 && cat.M <= 64) {  // the mixed-capacity launch's code path
        D ? one_rtc<true>(P, i, K, Cap) : one_rtc<false>(P, i, K, Cap);
        continue;
      }
      if (wide == 1 || Cap > 16 || cat.M > 64) {  // the wide-pool lane kernel's code path
        if (Cap > 32 || cat.M > 256) return CACE_E_INVALID;
        D ? one_wide<true>(P, i, K, Cap) : one_wide<false>(P, i, K, Cap);
        continue;
      }
      switch (Cap) {
#define CASE(k) case k: D ? one<k, true>(P, i, K) : one<k, false>(P, i, K); break;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
        CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
        default: return CACE_E_INVALID;
      }
    }
    return 0;
  } catch (const Invalid& e) {
    return e.code;
  }
}
