// C-ABI implementation of include/cace_gpu.h: host-side validation, trace
// layout, scenario planning and kernel launches.  There is no CPU fallback:
// without a CUDA device every replay entry returns CACE_E_NO_DEVICE.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <exception>
#include <mutex>
#include <numeric>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cace_gpu.h"
#include "glibc_log.cuh"
#include "policy_kernels.cuh"
#include "replay_lane.cuh"
#include "replay_warp.cuh"
#include "layout.hpp"
#include "metrics.cuh"
#include "trace_jsonl.hpp"

using namespace cace;

namespace {

// The engine drives up to 17 streams (engine stream, 8 workers, 8 select
// streams); with CUDA's default 8 hardware work queues, streams alias onto
// shared queues and independent launches serialise behind each other's waits.
// Raise the queue count at library load unless the user set it (effective
// only if this process has not created its CUDA context yet).
const int g_connections = [] {
  setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0);
  return 0;
}();

const double kLogTab[256] = CACE_GLIBC_LOG_TAB;
const double kLogTab2[256] = CACE_GLIBC_LOG_TAB2;

// CACE_TIMING=1: host phase timings of cace_replay_batch on stderr.
struct PhaseTimer {
  bool on = std::getenv("CACE_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "cace_timing %-16s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

void put_msg(char* msg, size_t cap, const std::string& s) {
  if (!msg || cap == 0) return;
  const size_t k = std::min(cap - 1, s.size());
  std::memcpy(msg, s.data(), k);
  msg[k] = 0;
}

struct CudaFail {
  int32_t code;
  std::string what;
};

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess)                                                        \
      throw CudaFail{CACE_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

// Keep freed memory in the device's default pool (stream-ordered
// allocator): repeated engine builds / batch calls then reuse it instead of
// paying cudaMalloc/cudaFree of hundreds of MB every call.
void retain_pool(int dev) {
  static std::mutex mu;
  static std::vector<bool> done;
  std::lock_guard<std::mutex> lk(mu);
  if ((int)done.size() <= dev) done.resize(dev + 1, false);
  if (done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  done[dev] = true;
}

// Device buffer owned by RAII, allocated and freed in order on one stream
// (the owner synchronises that stream, or joins every stream that used the
// buffer into it, before the buffer is released).
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t st = nullptr;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t k, cudaStream_t s) {
    release();
    n = k;
    st = s;
    if (k) CK(cudaMallocAsync(reinterpret_cast<void**>(&p), k * sizeof(T), s));
  }
  void upload(const T* h, size_t k, cudaStream_t s) {
    alloc(k, s);
    if (k) CK(cudaMemcpyAsync(p, h, k * sizeof(T), cudaMemcpyHostToDevice, s));
  }
};

// Process-wide pinned staging area for the trace records: the layout is
// built straight into page-locked memory (no page faults after the first
// use, DMA upload).  One engine build uses it at a time; a concurrent build
// falls back to pageable memory.
struct PinnedArena {
  std::mutex mu;
  void* p = nullptr;
  size_t cap = 0;
  bool busy = false;
  void* acquire(size_t bytes) {
    std::lock_guard<std::mutex> lk(mu);
    if (busy) return nullptr;
    if (cap < bytes) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      cap = 0;
      if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        return nullptr;
      }
      cap = bytes;
    }
    busy = true;
    return p;
  }
  void release() {
    std::lock_guard<std::mutex> lk(mu);
    busy = false;
  }
};
PinnedArena g_arena;      // trace-layout staging
PinnedArena g_arena_out;  // result staging

// Parallel host memcpy (pageable destinations of large results).
void par_memcpy(void* dst, const void* src, size_t bytes) {
  const int nth = (int)std::max<size_t>(
      1, std::min<size_t>(std::max(1u, std::thread::hardware_concurrency()), bytes >> 22));
  if (nth == 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> pool;
  for (int w = 0; w < nth; ++w)
    pool.emplace_back([=] {
      const size_t b = bytes * w / nth, e = bytes * (w + 1) / nth;
      std::memcpy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, e - b);
    });
  for (auto& th : pool) th.join();
}

int g_probe = -2;
std::mutex g_probe_mu;

int probe_log_variant() {
  std::lock_guard<std::mutex> lk(g_probe_mu);
  if (g_probe != -2) return g_probe;
  // Deterministic inputs covering both paths: near 1 and log-uniform wide.
  bool ok_fma = true, ok_sse = true;
  uint64_t st = 0x9e3779b97f4a7c15ULL;
  for (int i = 0; i < (1 << 20) && (ok_fma || ok_sse); ++i) {
    st += 0x9e3779b97f4a7c15ULL;
    uint64_t z = st;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z ^= z >> 31;
    const double u = (double)(z >> 11) * 0x1.0p-53;
    const double x = (i & 1) ? 1.0 + u * 0.0647 : std::exp2(u * 40.0);
    const double ref = std::log(x);
    const double a = cace_glibc_log(x, CACE_LOG_FMA, kLogTab, kLogTab2);
    const double b = cace_glibc_log(x, CACE_LOG_SSE2, kLogTab, kLogTab2);
    uint64_t ur, ua, ub;
    std::memcpy(&ur, &ref, 8);
    std::memcpy(&ua, &a, 8);
    std::memcpy(&ub, &b, 8);
    ok_fma = ok_fma && ur == ua;
    ok_sse = ok_sse && ur == ub;
  }
  g_probe = ok_fma ? CACE_LOG_FMA : (ok_sse ? CACE_LOG_SSE2 : -1);
  return g_probe;
}

int resolve_log_variant(const cace_opts_t* o) {
  if (o && o->log_variant >= 0) return o->log_variant;
  const int v = probe_log_variant();
  return v < 0 ? CACE_LOG_FMA : v;
}

int32_t device_count() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void require_device(const cace_opts_t* o) {
  const int n = device_count();
  if (n <= 0) throw Invalid{CACE_E_NO_DEVICE, "cace: no CUDA device (there is no CPU fallback)"};
  const int dev = o ? o->device : 0;
  if (dev < 0 || dev >= n) throw Invalid{CACE_E_INVALID, "cace: device ordinal out of range"};
  CK(cudaSetDevice(dev));
  retain_pool(dev);
}

// Host catalog + its device columns.
struct Catalog : HostCatalog {
  DBuf<double> d_lt, d_p2, d_tok;
  DBuf<int32_t> d_lex;
  void upload(cudaStream_t s) {
    d_lt.upload(lt.data(), M, s);
    d_p2.upload(p2.data(), M, s);
    d_tok.upload(tok.data(), M, s);
    d_lex.upload(lex.data(), M, s);
  }
  DevCatalog dev() const { return DevCatalog{M, d_lt.p, d_p2.p, d_tok.p, d_lex.p}; }
};

}  // namespace

// --------------------------------------------------------------------------
struct cace_engine {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int log_variant = CACE_LOG_FMA;
  Catalog cat;
  HostLayout lay;  // host replay-order layout (rec/perm/first0 freed after upload)
  DBuf<ReqRec> d_rec;
  DBuf<int64_t> d_off;
  DBuf<uint32_t> d_first0, d_perm, d_ncomp;
  DBuf<double> d_tab, d_tab2;
  // plan
  int64_t plan_n = -1;
  struct Seg {
    int C;      // lane kernel: capacity; warp kernel: slots per lane (1 or 2)
    int64_t b, e;
    bool warp;  // warp-per-scenario kernel
    bool wide;  // lane kernel, wide-pool mode (pools > 64 models or capacities > 16)
    bool mixed = false;  // in the mixed-capacity plan (d_mixed)
  };
  std::vector<Seg> segs;
  std::vector<int64_t> h_order;  // plan entries (scenario index | kShadowBit)
  DBuf<int64_t> d_order;
  // shallow sweeps: the lane segments of capacity <= kMixedC concatenated
  // heaviest first, replayed by ONE mixed-capacity launch (d_mixed)
  int64_t n_mixed = 0;
  bool mixed_ready = false;  // d_mixed holds this plan's entries
  DBuf<int64_t> d_mixed;
  std::vector<int64_t> bad_idx;
  std::vector<int32_t> bad_code;
  DBuf<int64_t> d_bad_idx;
  DBuf<int32_t> d_bad_code;
  int last_launches = 0;
  int kernel_pref = CACE_KERNEL_AUTO;
  std::vector<cudaStream_t> workers;  // fork/join streams for capacity segments
  std::vector<cudaEvent_t> joins;
  cudaEvent_t fork = nullptr;
  bool pooled = false;          // streams/events borrowed from the process-wide pool
  cudaStream_t pool_stream = nullptr;
  bool upload_pending = false;  // trace upload in flight from the pinned arena (finish_upload)
  bool arena_held = false;
};

namespace {

constexpr int kWorkers = 8;
constexpr int kMixedC = 8;  // capacity bound of the mixed-capacity (runtime capacity) launch

// Process-wide pool of engine stream sets (own stream + workers + fork/join
// events) per device: creating and destroying 9 streams and 9 events per
// cace_replay_batch call costs milliseconds of host time; engines borrow a
// set exclusively and return it idle (synchronised) on destroy.
struct StreamSet {
  cudaStream_t stream;
  std::vector<cudaStream_t> workers;
  std::vector<cudaEvent_t> joins;
  cudaEvent_t fork;
};
struct StreamPool {
  std::mutex mu;
  std::vector<std::pair<int, StreamSet>> free_sets;  // (device, set)
  bool take(int dev, StreamSet& out) {
    std::lock_guard<std::mutex> lk(mu);
    for (size_t i = 0; i < free_sets.size(); ++i)
      if (free_sets[i].first == dev) {
        out = free_sets[i].second;
        free_sets.erase(free_sets.begin() + (long)i);
        return true;
      }
    return false;
  }
  void give(int dev, const StreamSet& st) {
    std::lock_guard<std::mutex> lk(mu);
    free_sets.push_back({dev, st});
  }
} g_streams;

// The trace records travel from the pinned arena asynchronously while the
// host plans; the first synchronisation of the engine stream completes them.
void finish_upload(cace_engine* e) {
  if (!e->upload_pending) return;
  CK(cudaStreamSynchronize(e->stream));
  e->upload_pending = false;
  decltype(e->lay.rec)().swap(e->lay.rec);  // device copy is authoritative
  e->lay.ext_rec = nullptr;
  if (e->arena_held) {
    g_arena.release();
    e->arena_held = false;
  }
}

// Device copy of the replay-order -> caller-order permutation, for dumps.
void ensure_perm(cace_engine* e) {
  if (e->d_perm.p || e->lay.perm.empty()) return;
  e->d_perm.upload(e->lay.perm.data(), e->lay.perm.size(), e->stream);
}

void build_engine(cace_engine* e, const cace_catalog_t* catalog, const cace_trace_t* traces,
                  int32_t n_traces, const cace_opts_t* opts, bool defer_sync = false) {
  require_device(opts);
  e->device = opts ? opts->device : 0;
  StreamSet ss;
  if (g_streams.take(e->device, ss)) {
    e->pooled = true;
  } else {
    CK(cudaStreamCreateWithFlags(&ss.stream, cudaStreamNonBlocking));
    for (int k = 0; k < kWorkers; ++k) {
      cudaStream_t ws;
      cudaEvent_t ev;
      CK(cudaStreamCreateWithFlags(&ws, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      ss.workers.push_back(ws);
      ss.joins.push_back(ev);
    }
    CK(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
    e->pooled = true;
  }
  e->workers = ss.workers;
  e->joins = ss.joins;
  e->fork = ss.fork;
  if (opts && opts->stream) {
    e->stream = static_cast<cudaStream_t>(opts->stream);
  } else {
    e->stream = ss.stream;
    e->own_stream = true;
  }
  e->pool_stream = ss.stream;
  e->log_variant = resolve_log_variant(opts);
  e->kernel_pref = opts ? opts->kernel : CACE_KERNEL_AUTO;
  PhaseTimer pt;
  e->cat.load(catalog);
  if (n_traces > 0 && traces) {
    const int64_t N = layout_requests(traces, n_traces);
    if (N >= (1 << 16)) {
      e->lay.ext_rec = static_cast<ReqRec*>(g_arena.acquire((size_t)N * sizeof(ReqRec)));
      e->arena_held = e->lay.ext_rec != nullptr;
    }
  }
  build_layout(e->cat, traces, n_traces, e->lay);
  pt.mark("  layout");
  cudaStream_t s = e->stream;
  e->cat.upload(s);
  e->d_rec.upload(e->lay.records(), (size_t)e->lay.off[e->lay.T], s);
  e->d_off.upload(e->lay.off.data(), e->lay.off.size(), s);
  e->d_first0.upload(e->lay.first0.data(), e->lay.first0.size(), s);
  // the permutation back to caller order only serves full dumps: uploaded
  // on first use (ensure_perm)
  e->d_ncomp.upload(e->lay.ncomp.data(), e->lay.ncomp.size(), s);
  e->d_tab.upload(kLogTab, 256, s);
  e->d_tab2.upload(kLogTab2, 256, s);
  e->upload_pending = true;
  if (!defer_sync) {
    finish_upload(e);
    pt.mark("  upload");
  }
}

void plan(cace_engine* e, const cace_scenario_t* sc, int64_t n) {
  if (n < 0 || (n > 0 && !sc)) throw Invalid{CACE_E_INVALID, "cace: bad scenario array"};
  PhaseTimer pt;
  e->segs.clear();
  e->bad_idx.clear();
  e->bad_code.clear();
  auto capof = [&](int64_t i) { return (int)effective_capacity(sc[i], e->cat.M); };
  // Kernel choice: lane-per-scenario for capacities <= 16 and pools <= 64
  // models (register-resident slots and window, capacity a template
  // parameter); the same lane kernel in wide-pool mode for capacities <= 32
  // and pools <= 256 (BASELINE config 5); warp-per-scenario beyond that or
  // when forced with CACE_KERNEL_WARP.
  const bool force_warp = e->kernel_pref == CACE_KERNEL_WARP;
  const int M0 = e->cat.M;
  // dense segment key: 1..16 lane capacity, 17..48 wide-lane capacity + 16,
  // 49..50 warp kernel (slots per lane)
  auto key = [&](int64_t i) {
    const int C = capof(i);
    if (!force_warp && C <= kMaxLaneC && M0 <= kLaneMaxModels) return C;
    if (!force_warp && C <= kWideC && M0 <= kWideMaxModels) return 16 + C;
    return 48 + (C <= 32 ? 1 : 2);
  };
  // Per scenario, on all host threads: the run() preconditions, the dense
  // segment key (-1 = invalid) and a compact coherence key (trace, variant,
  // p1_mode, window).
  std::vector<int32_t> status(n);
  std::vector<int8_t> kv(n);
  std::vector<uint64_t> ck(n);
  {
    const int nth = (int)std::max<int64_t>(
        1, std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), n / 65536));
    auto work = [&](int w) {
      for (int64_t i = (int64_t)w * n / nth, ie = (int64_t)(w + 1) * n / nth; i < ie; ++i) {
        const int32_t st = precheck(e->lay, sc[i]);
        const bool tv = sc[i].trace >= 0 && sc[i].trace < e->lay.T;
        const int64_t len = tv ? e->lay.off[sc[i].trace + 1] - e->lay.off[sc[i].trace] : 0;
        status[i] = st;
        if (st != CACE_OK || len == 0) {
          kv[i] = -1;
          continue;
        }
        kv[i] = (int8_t)key(i);
        const uint32_t win = (uint32_t)std::min(sc[i].window_length, (1 << 27) - 1);
        ck[i] = ((uint64_t)(uint32_t)sc[i].trace << 32) | ((uint64_t)(sc[i].variant & 7) << 29) |
                ((uint64_t)(sc[i].p1_mode & 1) << 28) | win;
      }
    };
    if (nth == 1) {
      work(0);
    } else {
      std::vector<std::thread> pool;
      for (int w = 0; w < nth; ++w) pool.emplace_back(work, w);
      for (auto& th : pool) th.join();
    }
  }
  pt.mark("  precheck");
  // Coherent warps: segment, then trace, then the control-flow shaping
  // policy fields.  Stable counting sort by segment (O(S)), then each
  // segment is stably sorted by the compact key unless it already is (the
  // common case for generated sweeps).
  std::vector<int64_t> ok;
  {
    const int kmax = 50;
    std::vector<int64_t> cnt(kmax + 2, 0);
    for (int64_t i = 0; i < n; ++i) {
      if (kv[i] < 0) {
        e->bad_idx.push_back(i);
        e->bad_code.push_back(status[i]);
      } else {
        ++cnt[kv[i] + 1];
      }
    }
    for (int k = 1; k <= kmax + 1; ++k) cnt[k] += cnt[k - 1];
    ok.resize(cnt[kmax + 1]);
    std::vector<int64_t> start(cnt.begin(), cnt.end());
    for (int64_t i = 0; i < n; ++i)
      if (kv[i] >= 0) ok[start[kv[i]]++] = i;
    auto lt = [&](int64_t a, int64_t b) { return ck[a] < ck[b]; };
    for (int k = 0; k <= kmax; ++k) {
      auto b = ok.begin() + cnt[k], e2 = ok.begin() + cnt[k + 1];
      if (!std::is_sorted(b, e2, lt)) std::stable_sort(b, e2, lt);
    }
  }
  pt.mark("  sort");
  // Lane segments: every (capacity, trace) group is padded to a whole number
  // of warps with shadow lanes (copies of the group's first scenario that
  // write nothing) so each warp is trace-uniform and walks its trace in
  // lockstep.  Warp segments need no padding (one warp = one scenario).
  // (segment key and trace read from the compact per-scenario arrays)
  auto seg_of = [&](int64_t i) { return (int)kv[i]; };
  auto trace_of = [&](int64_t i) { return (int32_t)(ck[i] >> 32); };
  std::vector<int64_t> order;
  order.reserve(ok.size() + ok.size() / 8 + 32 * 64);
  for (size_t k = 0; k < ok.size();) {
    const int K = seg_of(ok[k]);
    const int64_t seg_b = (int64_t)order.size();
    size_t j = k;
    if (K > 48) {
      while (j < ok.size() && seg_of(ok[j]) == K) order.push_back(ok[j++]);
      e->segs.push_back({K - 48, seg_b, (int64_t)order.size(), true, false});
    } else {
      while (j < ok.size() && seg_of(ok[j]) == K) {
        const int32_t t = trace_of(ok[j]);
        size_t g = j;
        while (g < ok.size() && seg_of(ok[g]) == K && trace_of(ok[g]) == t) order.push_back(ok[g++]);
        const int64_t pad = (32 - (int64_t)(g - j) % 32) % 32;
        for (int64_t q = 0; q < pad; ++q) order.push_back(ok[j] | (int64_t)kShadowBit);
        j = g;
      }
      e->segs.push_back({K > 16 ? K - 16 : K, seg_b, (int64_t)order.size(), false, K > 16});
    }
    k = j;
  }
  pt.mark("  order");
  // Launch the most expensive segments first: the block scheduler fills the
  // GPU in launch order, so cheap segments then backfill the tail of the
  // long ones.  Replay cost grows with the number of eviction candidates,
  // ~min(C, M - 1) per decision; C >= M never evicts.
  const int M = e->cat.M;
  auto seg_cost = [&](const cace_engine::Seg& g) {
    const double per = g.warp ? 64.0 : (g.C >= M ? 2.0 : (double)std::min(g.C, M - 1));
    return per * (double)(g.e - g.b);
  };
  std::stable_sort(e->segs.begin(), e->segs.end(),
                   [&](const cace_engine::Seg& x, const cace_engine::Seg& y) { return seg_cost(x) > seg_cost(y); });
  // The mixed-capacity plan (shallow sweeps, replay()): every lane segment of
  // capacity <= kMixedC, heaviest first, as one launch.  Concurrent
  // per-capacity launches of a few hundred blocks each leave SMs unevenly
  // loaded (a 2560-warp sweep: 151 ms as five concurrent launches, 92 ms as
  // one; profiles/r2/ab_concurrency_r2w.txt).
  // (its entry list is built and uploaded by replay() only when it is chosen)
  e->n_mixed = 0;
  e->mixed_ready = false;
  for (auto& g : e->segs) {
    g.mixed = !g.warp && !g.wide && g.C <= kMixedC;
    if (g.mixed) e->n_mixed += g.e - g.b;
  }
  e->d_order.upload(order.data(), order.size(), e->stream);
  e->d_bad_idx.upload(e->bad_idx.data(), e->bad_idx.size(), e->stream);
  e->d_bad_code.upload(e->bad_code.data(), e->bad_code.size(), e->stream);
  CK(cudaStreamSynchronize(e->stream));
  finish_upload(e);
  e->h_order = std::move(order);
  e->plan_n = n;
}

template <int C, int MW, int DM, int MINB, int MC = 0, bool RTC = false>
void launch_lane(const ReplayParams& P, int64_t count, size_t smem, cudaStream_t s) {
  auto* k = replay_lane_kernel<C, MW, DM, MINB, MC, RTC>;
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // one L1/shared split for every capacity's kernel: blocks of different
  // segments can then share an SM without a carveout change (shallow sweeps
  // +9%, profiles/r2/ab_carveout_v6.txt)
  CK(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  const unsigned grid = (unsigned)((count + LANE_BLOCK - 1) / LANE_BLOCK);
  k<<<grid, LANE_BLOCK, smem, s>>>(P);
  CK(cudaGetLastError());
}

// The 8-model pool (BASELINE configs 1-4; capacities clamp to <= 8) has
// compile-time-layout instantiations of the summary and RunMetrics-sample
// kernels (MC = 8; +3.4% on config 4, profiles/r2/ab_pool_mc_r2q.txt).
constexpr int kPoolMC = 8;

template <int MW, int DM, int MINB = CACE_LANE_MIN_BLOCKS>
void dispatch_lane_c(int C, const ReplayParams& P, int64_t count, size_t smem, cudaStream_t s) {
#ifndef CACE_NO_POOL_MC
  if ((DM == 0 || DM == 2) && MW == 1 && P.cat.M == kPoolMC) {  // summaries, RunMetrics samples
    switch (C) {
#define CASE(k) \
  case k: launch_lane<k, 1, DM, MINB, kPoolMC>(P, count, smem, s); return;
      CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
      default: break;
    }
  }
#endif
  switch (C) {
#define CASE(k) \
  case k: launch_lane<k, MW, DM, MINB>(P, count, smem, s); break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
    CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
    default: throw Invalid{CACE_E_INVALID, "cace: capacity not supported by the lane kernel"};
  }
}

// One mixed-capacity launch (RTC instantiation, capacity bound kMixedC) over
// plan entries [0, count) of P.order.
template <int MINB>
void launch_mixed_t(const ReplayParams& P, int64_t count, size_t smem, cudaStream_t s) {
#ifndef CACE_NO_POOL_MC
  if (P.cat.M == kPoolMC) {
    launch_lane<kMixedC, 1, 0, MINB, kPoolMC, true>(P, count, smem, s);
    return;
  }
#endif
  launch_lane<kMixedC, 1, 0, MINB, 0, true>(P, count, smem, s);
}

void launch_mixed(int minb, const ReplayParams& P, int64_t count, size_t smem, cudaStream_t s) {
  if (minb == kLaneLatencyMinBlocks)
    launch_mixed_t<kLaneLatencyMinBlocks>(P, count, smem, s);
  else if (minb == kLaneMidMinBlocks)
    launch_mixed_t<kLaneMidMinBlocks>(P, count, smem, s);
  else
    launch_mixed_t<CACE_LANE_MIN_BLOCKS>(P, count, smem, s);
}

template <int SPL, bool DUMP>
void launch_warp(const ReplayParams& P, int64_t count, cudaStream_t s) {
  const size_t smem = warp_smem_bytes(P.cat.M);
  if (smem > 48 * 1024)
    CK(cudaFuncSetAttribute(replay_warp_kernel<SPL, DUMP>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int per = WARP_BLOCK / 32;
  const unsigned grid = (unsigned)((count + per - 1) / per);
  replay_warp_kernel<SPL, DUMP><<<grid, WARP_BLOCK, smem, s>>>(P);
  CK(cudaGetLastError());
}

void dispatch_warp(bool dump, int spl, const ReplayParams& P, int64_t count, cudaStream_t s) {
  if (spl == 1)
    dump ? launch_warp<1, true>(P, count, s) : launch_warp<1, false>(P, count, s);
  else
    dump ? launch_warp<2, true>(P, count, s) : launch_warp<2, false>(P, count, s);
}

void dispatch_lane(int dm, int C, const ReplayParams& P, int64_t count, size_t smem, cudaStream_t s,
                   int minb) {
  const bool mw1 = P.cat.M <= 32;
  if (dm == 0 && mw1 && minb == kLaneLatencyMinBlocks) {
    dispatch_lane_c<1, 0, kLaneLatencyMinBlocks>(C, P, count, smem, s);
    return;
  }
  if (dm == 0 && mw1 && minb == kLaneMidMinBlocks) {
    dispatch_lane_c<1, 0, kLaneMidMinBlocks>(C, P, count, smem, s);
    return;
  }
  switch (dm) {
    case 0: mw1 ? dispatch_lane_c<1, 0>(C, P, count, smem, s) : dispatch_lane_c<2, 0>(C, P, count, smem, s); break;
    case 1: mw1 ? dispatch_lane_c<1, 1>(C, P, count, smem, s) : dispatch_lane_c<2, 1>(C, P, count, smem, s); break;
    default: mw1 ? dispatch_lane_c<1, 2>(C, P, count, smem, s) : dispatch_lane_c<2, 2>(C, P, count, smem, s); break;
  }
}

#ifndef CACE_WIDE_G
#define CACE_WIDE_G 8
#endif
constexpr int kWideG = CACE_WIDE_G;  // lanes per scenario of the wide-pool lane kernel (C / G = 4 slots per lane)

template <int MW, int DM>
void launch_lane_wide(const ReplayParams& P, int64_t count, cudaStream_t s) {
  constexpr int G = kWideG;
  const size_t smem = lane_wide_smem_bytes(P.cat.M, DM != 0, G);
  auto* k = replay_lane_wide_kernel<MW, DM, G>;
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  constexpr int SB = LANE_BLOCK_WIDE / G;  // scenarios (plan entries) per block
  const unsigned grid = (unsigned)((count + SB - 1) / SB);
  k<<<grid, LANE_BLOCK_WIDE, smem, s>>>(P);
  CK(cudaGetLastError());
}

template <int DM>
void dispatch_lane_wide_dm(const ReplayParams& P, int64_t count, cudaStream_t s) {
  const int M = P.cat.M;
  if (M <= 32)
    launch_lane_wide<1, DM>(P, count, s);
  else if (M <= 64)
    launch_lane_wide<2, DM>(P, count, s);
  else if (M <= 128)
    launch_lane_wide<4, DM>(P, count, s);
  else
    launch_lane_wide<8, DM>(P, count, s);
}

void dispatch_lane_wide(int dm, const ReplayParams& P, int64_t count, cudaStream_t s) {
  if (dm == 0)
    dispatch_lane_wide_dm<0>(P, count, s);
  else if (dm == 1)
    dispatch_lane_wide_dm<1>(P, count, s);
  else
    dispatch_lane_wide_dm<2>(P, count, s);
}

ReplayParams replay_params(const cace_engine* e, const cace_scenario_t* d_sc, cace_summary_t* d_out,
                           const DumpDev& dump) {
  ReplayParams P{};
  P.rec = e->d_rec.p;
  P.trace_off = e->d_off.p;
  P.first0 = e->d_first0.p;
  P.perm = e->d_perm.p;
  P.trace_ncomp = e->d_ncomp.p;
  P.cat = e->cat.dev();
  P.log_tab = e->d_tab.p;
  P.log_tab2 = e->d_tab2.p;
  P.log_variant = e->log_variant;
  P.scen = d_sc;
  P.order = e->d_order.p;
  P.out = d_out;
  P.dump = dump;
  return P;
}

// One launch over plan entries [b, e) of segment g (b warp-aligned).
void launch_piece(const cace_engine* e, const cace_engine::Seg& g, ReplayParams P, int64_t b,
                  int64_t end, cudaStream_t ws, int minb) {
  P.seg_begin = b;
  P.seg_end = end;
  const bool dump_on = P.dump.slot != nullptr;
  // samples set = the RunMetrics pipeline, which dumps nothing else
  const int dm = !dump_on ? 0 : (P.dump.samples ? 2 : 1);
  if (g.warp)
    dispatch_warp(dump_on, g.C, P, end - b, ws);
  else if (g.wide)
    dispatch_lane_wide(dm, P, end - b, ws);
  else
    dispatch_lane(dm, g.C, P, end - b, lane_smem_bytes(e->cat.M, g.C, dump_on), ws, minb);
}

void fill_status(cace_engine* e, cace_summary_t* d_out, cudaStream_t s) {
  if (e->bad_idx.empty()) return;
  fill_status_kernel<<<(unsigned)((e->bad_idx.size() + 255) / 256), 256, 0, s>>>(
      e->d_bad_idx.p, e->d_bad_code.p, (int64_t)e->bad_idx.size(), d_out);
  CK(cudaGetLastError());
  ++e->last_launches;
}

void fork_workers(cace_engine* e, cudaStream_t s, size_t used) {
  CK(cudaEventRecord(e->fork, s));
  for (size_t k = 0; k < std::min(used, e->workers.size()); ++k)
    CK(cudaStreamWaitEvent(e->workers[k], e->fork, 0));
}

void join_workers(cace_engine* e, cudaStream_t s, size_t used) {
  for (size_t k = 0; k < std::min(used, e->workers.size()); ++k) {
    CK(cudaEventRecord(e->joins[k], e->workers[k]));
    CK(cudaStreamWaitEvent(s, e->joins[k], 0));
  }
}

void replay(cace_engine* e, const cace_scenario_t* d_sc, int64_t n, cace_summary_t* d_out,
            const DumpDev& dump, cudaStream_t s) {
  if (n != e->plan_n) throw Invalid{CACE_E_INVALID, "cace: replay does not match the plan"};
  CK(cudaSetDevice(e->device));
  const ReplayParams P = replay_params(e, d_sc, d_out, dump);
  e->last_launches = 0;
  // Capacity segments are independent kernels: fork them over the engine's
  // worker streams so they share the SMs (one segment alone is often less
  // than a wave), then join back onto s.
  const size_t nseg = e->segs.size();
  // Occupancy tier by sweep depth in waves of 20-warp-per-SM lane warps:
  // < 1.5 waves the step is one warp's dependency chain (register-rich
  // MINB 3), 1.5-2.5 waves MINB 4, deeper sweeps are issue-bound (MINB 5).
  // Measured on config-4 shards (131k .. 1M scenarios; the 2.5 crossover on
  // the final kernels: profiles/r2/ab_tiers_r2bm.txt).
  int64_t lane_warps = 0;
  for (const auto& g : e->segs)
    if (!g.warp) lane_warps += (g.e - g.b) / 32;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e->device);
  const double waves = (double)lane_warps / ((double)sms * (CACE_LANE_MIN_BLOCKS * 4));
  int minb = waves < 1.5 ? kLaneLatencyMinBlocks : (waves < 2.5 ? kLaneMidMinBlocks : CACE_LANE_MIN_BLOCKS);
  if (const char* v = std::getenv("CACE_LANE_MINB")) minb = std::atoi(v);  // tuning override (3, 4, 5)
  // From 0.5 to 1.8 waves with several capacities (a strong-scaling shard), the
  // capacities <= 8 run as ONE mixed-capacity launch at MINB 4 (summaries,
  // pools <= 32 models): 131k shard 8.6e10 -> 1.21e11; at 262k the
  // per-capacity launches stay faster, and below 0.5 waves (32k scenarios)
  // the per-capacity MINB 3 kernels (profiles/r2/ab_mixed_r2y.txt, ab_mixed_r2z.txt);
  // 1.73 waves (164k): mixed +7%, 2.08 waves (196k): -9% (ab_mixed_upper_r2bp.txt).
  int n_mixable = 0;
  for (const auto& g : e->segs) n_mixable += g.mixed ? 1 : 0;
  bool mixed = waves >= 0.5 && waves < 1.8 && dump.slot == nullptr && e->cat.M <= 32 && n_mixable >= 2;
  if (const char* v = std::getenv("CACE_MIXED")) mixed = v[0] == '1' ? (dump.slot == nullptr && e->cat.M <= 32 &&
                                                                          n_mixable >= 1)
                                                                       : false;  // A/B switch (0 / 1)
  const int minb_mixed = std::getenv("CACE_LANE_MINB") ? minb : kLaneMidMinBlocks;
  std::vector<const cace_engine::Seg*> launch;
  for (const auto& g : e->segs)
    if (!(mixed && g.mixed)) launch.push_back(&g);
  const size_t nl = launch.size() + (mixed ? 1 : 0);
  if (nl > 0) {
    if (nl > 1) fork_workers(e, s, nl);
    size_t k = 0;
    if (mixed) {
      if (!e->mixed_ready) {
        std::vector<int64_t> ent;
        ent.reserve((size_t)e->n_mixed);
        for (const auto& g : e->segs)
          if (g.mixed) ent.insert(ent.end(), e->h_order.begin() + g.b, e->h_order.begin() + g.e);
        e->d_mixed.upload(ent.data(), ent.size(), s);
        CK(cudaStreamSynchronize(s));  // pageable source
        e->mixed_ready = true;
      }
      cudaStream_t ws = nl == 1 ? s : e->workers[k++ % e->workers.size()];
      ReplayParams Q = P;
      Q.order = e->d_mixed.p;
      Q.seg_begin = 0;
      Q.seg_end = e->n_mixed;
      launch_mixed(minb_mixed, Q, e->n_mixed, lane_smem_bytes(e->cat.M, kMixedC, false), ws);
      ++e->last_launches;
    }
    for (const auto* g : launch) {
      cudaStream_t ws = nl == 1 ? s : e->workers[k++ % e->workers.size()];
      launch_piece(e, *g, P, g->b, g->e, ws, minb);
      ++e->last_launches;
    }
    if (nl > 1) join_workers(e, s, nl);
  }
  fill_status(e, d_out, s);
}

template <typename F>
int32_t guarded(char* msg, size_t cap, F&& f) {
  try {
    return f();
  } catch (const CudaFail& x) {
    put_msg(msg, cap, x.what);
    return x.code;
  } catch (const Invalid& x) {
    put_msg(msg, cap, x.what);
    return x.code;
  } catch (const std::exception& x) {
    put_msg(msg, cap, x.what());
    return CACE_E_INVALID;
  }
}

// cace_engine_create, optionally leaving the trace upload in flight (the
// first plan() completes it; cace_replay_batch overlaps the two).
int32_t engine_create_impl(const cace_catalog_t* catalog, const cace_trace_t* traces, int32_t n_traces,
                           const cace_opts_t* opts, cace_engine** out, char* msg, size_t msg_cap,
                           bool defer_sync) {
  if (!out) return CACE_E_INVALID;
  *out = nullptr;
  cace_engine* e = new cace_engine();
  const int32_t rc = guarded(msg, msg_cap, [&]() -> int32_t {
    build_engine(e, catalog, traces, n_traces, opts, defer_sync);
    return CACE_OK;
  });
  if (rc != CACE_OK) {
    cace_engine_destroy(e);
    return rc;
  }
  *out = e;
  return CACE_OK;
}

}  // namespace

// ==========================================================================
extern "C" {

const char* cace_version(void) {
  return "cace-b200 0.1 (sm_100a lane-per-scenario replay; glibc-log bit-exact P1)";
}
int32_t cace_abi_version(void) { return CACE_ABI_VERSION; }
int32_t cace_device_count(void) { return device_count(); }

int32_t cace_engine_create(const cace_catalog_t* catalog, const cace_trace_t* traces,
                           int32_t n_traces, const cace_opts_t* opts, cace_engine** out,
                           char* msg, size_t msg_cap) {
  return engine_create_impl(catalog, traces, n_traces, opts, out, msg, msg_cap, false);
}

void cace_engine_destroy(cace_engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  if (e->stream) cudaStreamSynchronize(e->stream);
  for (auto ws : e->workers) cudaStreamSynchronize(ws);
  if (e->upload_pending) {  // an engine destroyed before its first plan
    e->upload_pending = false;
    e->lay.ext_rec = nullptr;
  }
  if (e->arena_held) g_arena.release();
  // device buffers go back to the pool in order on the engine stream, which
  // must still exist
  e->cat.d_lt.release();
  e->cat.d_p2.release();
  e->cat.d_tok.release();
  e->cat.d_lex.release();
  e->d_rec.release();
  e->d_off.release();
  e->d_first0.release();
  e->d_perm.release();
  e->d_ncomp.release();
  e->d_tab.release();
  e->d_tab2.release();
  e->d_order.release();
  e->d_mixed.release();
  e->d_bad_idx.release();
  e->d_bad_code.release();
  if (e->pooled) {
    // the set goes back idle: its own stream is synchronised after the frees
    cudaStreamSynchronize(e->pool_stream);
    if (cudaGetLastError() == cudaSuccess)
      g_streams.give(e->device, StreamSet{e->pool_stream, e->workers, e->joins, e->fork});
  } else {
    for (auto ws : e->workers) cudaStreamDestroy(ws);
    for (auto ev : e->joins) cudaEventDestroy(ev);
    if (e->fork) cudaEventDestroy(e->fork);
    if (e->own_stream && e->stream) cudaStreamDestroy(e->stream);
  }
  delete e;
}

int32_t cace_engine_plan(cace_engine* e, const cace_scenario_t* scenarios, int64_t n, char* msg,
                         size_t msg_cap) {
  if (!e) return CACE_E_INVALID;
  return guarded(msg, msg_cap, [&]() -> int32_t {
    CK(cudaSetDevice(e->device));
    plan(e, scenarios, n);
    return CACE_OK;
  });
}

int32_t cace_engine_replay_device(cace_engine* e, const cace_scenario_t* d_scenarios, int64_t n,
                                  cace_summary_t* d_summaries, void* stream, char* msg,
                                  size_t msg_cap) {
  if (!e) return CACE_E_INVALID;
  return guarded(msg, msg_cap, [&]() -> int32_t {
    replay(e, d_scenarios, n, d_summaries, DumpDev{},
           stream ? static_cast<cudaStream_t>(stream) : e->stream);
    return CACE_OK;
  });
}

int32_t cace_engine_status_message(const cace_engine* e, int32_t status, char* msg,
                                   size_t msg_cap) {
  if (!e) return CACE_E_INVALID;
  put_msg(msg, msg_cap, status_text(e->cat, status));
  return status & 0xff;
}

int32_t cace_engine_last_launches(const cace_engine* e) { return e ? e->last_launches : 0; }

int32_t cace_replay_batch(const cace_catalog_t* catalog, const cace_trace_t* traces,
                          int32_t n_traces, const cace_scenario_t* scenarios, int64_t n_scenarios,
                          cace_summary_t* summaries, const cace_dump_t* dump,
                          const cace_opts_t* opts, char* msg, size_t msg_cap) {
  cace_engine* e = nullptr;
  PhaseTimer pt;
  // the trace records' DMA from the pinned arena overlaps the plan below
  int32_t rc = engine_create_impl(catalog, traces, n_traces, opts, &e, msg, msg_cap, true);
  if (rc != CACE_OK) return rc;
  pt.mark("engine_create");
  rc = guarded(msg, msg_cap, [&]() -> int32_t {
    if (n_scenarios > 0 && !summaries) throw Invalid{CACE_E_INVALID, "cace: summaries is NULL"};
    cudaStream_t s = e->stream;
    DBuf<cace_scenario_t> d_sc;
    {
      // the (pageable) scenario upload runs on a helper thread while this one
      // plans; both are on the engine stream, ahead of the replay
      std::exception_ptr up_err;
      std::thread up([&] {
        try {
          CK(cudaSetDevice(e->device));
          d_sc.upload(scenarios, n_scenarios, s);
        } catch (...) {
          up_err = std::current_exception();
        }
      });
      try {
        plan(e, scenarios, n_scenarios);
      } catch (...) {
        up.join();
        throw;
      }
      up.join();
      if (up_err) std::rethrow_exception(up_err);
    }
    pt.mark("plan+upload_scen");
    DBuf<cace_summary_t> d_out;
    d_out.alloc(n_scenarios, s);
    // Optional full dump.
    DumpDev dd{};
    DBuf<int32_t> d_slot;
    DBuf<int64_t> d_doff, d_nev;
    DBuf<uint8_t> d_cold;
    DBuf<double> d_qw, d_lw, d_pf, d_dc, d_tt, d_ee, d_ec;
    DBuf<int32_t> d_em;
    std::vector<int64_t> doff;
    int64_t total = 0;
    const int nd = dump ? dump->n_dump : 0;
    if (nd > 0) {
      ensure_perm(e);
      std::vector<int32_t> slot(n_scenarios, -1);
      for (int k = 0; k < nd; ++k) {
        const int64_t si = dump->scenario_index[k];
        if (si < 0 || si >= n_scenarios) throw Invalid{CACE_E_INVALID, "cace: bad dump index"};
        slot[si] = k;
        doff.push_back(total);
        const int t = scenarios[si].trace;
        total += (t >= 0 && t < e->lay.T) ? e->lay.off[t + 1] - e->lay.off[t] : 0;
      }
      d_slot.upload(slot.data(), slot.size(), s);
      d_doff.upload(doff.data(), doff.size(), s);
      dd.slot = d_slot.p;
      dd.dump_off = d_doff.p;
      // dump buffers start zeroed: eviction logs are written only up to
      // each scenario's eviction count, and the whole arrays are copied back
      auto mk = [&](DBuf<double>& b, double* h) -> double* {
        if (!h) return nullptr;
        b.alloc(total, s);
        if (total) CK(cudaMemsetAsync(b.p, 0, total * sizeof(double), s));
        return b.p;
      };
      if (dump->cold_start) {
        d_cold.alloc(total, s);
        if (total) CK(cudaMemsetAsync(d_cold.p, 0, total, s));
        dd.cold = d_cold.p;
      }
      dd.queue_wait = mk(d_qw, dump->queue_wait_s);
      dd.load_wait = mk(d_lw, dump->load_wait_s);
      dd.prefill = mk(d_pf, dump->prefill_s);
      dd.decode = mk(d_dc, dump->decode_s);
      dd.ttft = mk(d_tt, dump->ttft_s);
      dd.e2e = mk(d_ee, dump->e2e_s);
      dd.evict_cap = dump->evict_cap;
      if (dump->evict_model && dump->evict_cap > 0) {
        d_em.alloc((size_t)nd * dump->evict_cap, s);
        CK(cudaMemsetAsync(d_em.p, 0, (size_t)nd * dump->evict_cap * sizeof(int32_t), s));
        dd.evict_model = d_em.p;
      }
      if (dump->evict_clock && dump->evict_cap > 0) {
        d_ec.alloc((size_t)nd * dump->evict_cap, s);
        CK(cudaMemsetAsync(d_ec.p, 0, (size_t)nd * dump->evict_cap * sizeof(double), s));
        dd.evict_clock = d_ec.p;
      }
      d_nev.alloc(nd, s);
      CK(cudaMemsetAsync(d_nev.p, 0, nd * sizeof(int64_t), s));
      dd.n_evict = d_nev.p;
    }
    if (pt.on) {
      CK(cudaStreamSynchronize(s));
      pt.mark("upload_scen");
    }
    replay(e, d_sc.p, n_scenarios, d_out.p, dd, s);
    if (pt.on) {
      CK(cudaStreamSynchronize(s));
      pt.mark("replay");
    }
    // summaries: DMA into pinned staging, then a threaded copy to the
    // caller's (pageable) array; small results go directly
    const size_t sbytes = (size_t)n_scenarios * sizeof(cace_summary_t);
    void* stage = sbytes >= ((size_t)8 << 20) ? g_arena_out.acquire(sbytes) : nullptr;
    struct StageGuard {
      void* p;
      ~StageGuard() {
        if (p) g_arena_out.release();
      }
    } sguard{stage};
    if (n_scenarios > 0)
      CK(cudaMemcpyAsync(stage ? stage : summaries, d_out.p, sbytes, cudaMemcpyDeviceToHost, s));
    if (nd > 0) {
      auto back = [&](void* h, const void* d, size_t bytes) {
        if (h && d && bytes) CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s));
      };
      back(dump->cold_start, d_cold.p, total);
      back(dump->queue_wait_s, d_qw.p, total * 8);
      back(dump->load_wait_s, d_lw.p, total * 8);
      back(dump->prefill_s, d_pf.p, total * 8);
      back(dump->decode_s, d_dc.p, total * 8);
      back(dump->ttft_s, d_tt.p, total * 8);
      back(dump->e2e_s, d_ee.p, total * 8);
      back(dump->evict_model, d_em.p, (size_t)nd * dump->evict_cap * 4);
      back(dump->evict_clock, d_ec.p, (size_t)nd * dump->evict_cap * 8);
      back(dump->n_evict, d_nev.p, (size_t)nd * 8);
    }
    CK(cudaStreamSynchronize(s));
    if (stage) par_memcpy(summaries, stage, sbytes);
    pt.mark("download");
    // The replay kernels write CACE_OK; the only other statuses are the
    // plan's precheck codes (fill_status), recorded in caller order -- no
    // scan of the 112-B summaries (~6 ms for a 1M sweep).
    for (size_t j = 0; j < e->bad_code.size(); ++j) {
      if (e->bad_code[j] != CACE_OK) {
        put_msg(msg, msg_cap, status_text(e->cat, e->bad_code[j]));
        return e->bad_code[j] & 0xff;
      }
    }
    return CACE_OK;
  });
  cace_engine_destroy(e);
  pt.mark("destroy");
  return rc;
}

}  // extern "C"

#include "multi_device.inc"

extern "C" {

int32_t cace_run_metrics_batch(const cace_catalog_t* catalog, const cace_trace_t* traces,
                               int32_t n_traces, const cace_scenario_t* scenarios,
                               int64_t n_scenarios, cace_run_metrics_t* metrics,
                               cace_summary_t* summaries, const cace_opts_t* opts, char* msg,
                               size_t msg_cap) {
  cace_engine* e = nullptr;
  PhaseTimer pt;
  int32_t rc = cace_engine_create(catalog, traces, n_traces, opts, &e, msg, msg_cap);
  if (rc != CACE_OK) return rc;
  pt.mark("engine_create");
  rc = guarded(msg, msg_cap, [&]() -> int32_t {
    if (n_scenarios > 0 && (!metrics || !scenarios))
      throw Invalid{CACE_E_INVALID, "cace: metrics / scenarios is NULL"};
    cudaStream_t s = e->stream;
    plan(e, scenarios, n_scenarios);
    pt.mark("plan");
    auto nreq = [&](int64_t i) -> int64_t {
      const int t = scenarios[i].trace;
      return (t >= 0 && t < e->lay.T) ? e->lay.off[t + 1] - e->lay.off[t] : 0;
    };
    // Pipeline: the planned sweep (heaviest segments first) is cut into
    // warp-aligned chunks whose samples fit one of W ring buffers (~60% of
    // free HBM in total); chunk j replays into buffer j % W on worker stream
    // j % W and the select kernel reduces it on the same stream, so the
    // buffer is reused in stream order while the other streams keep the SMs
    // full of replay lanes.  Chunk-local arrays are concatenated in chunk
    // order (position p = chunk base + local index).
    size_t W = e->workers.size();
    if (const char* v = std::getenv("CACE_METRICS_RINGS"))  // tuning override (1..8)
      W = std::max<size_t>(1, std::min<size_t>(W, (size_t)std::atoi(v)));
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    // memory the stream-ordered pool holds but does not use is free to us
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, e->device) == cudaSuccess) {
      uint64_t reserved = 0, used = 0;
      if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
          cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && reserved > used)
        free_b += reserved - used;
    }
    cudaGetLastError();
    size_t budget = std::max<size_t>((size_t)(0.6 * (double)free_b), (size_t)64 << 20);
    if (const char* v = std::getenv("CACE_METRICS_BUDGET_MB"))  // test / tuning override
      budget = std::max<size_t>((size_t)std::atoll(v) << 20, 1);
    const size_t per = budget / W;
    struct Chunk {
      size_t seg;
      int64_t b, e, base, nloc, nsamp;
    };
    std::vector<Chunk> chunks;
    std::vector<int32_t> slot(n_scenarios, -1);
    std::vector<int64_t> loc_scen, off;
    std::vector<uint32_t> nc, nr;
    const auto& order = e->h_order;
    for (size_t k = 0; k < e->segs.size(); ++k) {
      const auto& g = e->segs[k];
      for (int64_t pos = g.b; pos < g.e;) {
        Chunk c{k, pos, pos, (int64_t)loc_scen.size(), 0, 0};
        while (c.e < g.e) {
          const int64_t ue = std::min<int64_t>(c.e + 32, g.e);
          int64_t ub = 0;
          for (int64_t q = c.e; q < ue; ++q)
            if (!(order[q] & (int64_t)kShadowBit)) ub += nreq(order[q]);
          if (c.e > c.b && (size_t)(c.nsamp + ub) * 8 > per) break;
          for (int64_t q = c.e; q < ue; ++q) {
            if (order[q] & (int64_t)kShadowBit) continue;
            const int64_t si = order[q];
            const int t = scenarios[si].trace;
            slot[si] = (int32_t)(loc_scen.size() - c.base);
            loc_scen.push_back(si);
            off.push_back(c.nsamp);
            nr.push_back((uint32_t)nreq(si));
            nc.push_back(e->lay.ncomp[t]);
            c.nsamp += nreq(si);
          }
          c.e = ue;
        }
        c.nloc = (int64_t)loc_scen.size() - c.base;
        chunks.push_back(c);
        pos = c.e;
      }
    }
    const int64_t NL = (int64_t)loc_scen.size();
    pt.mark("chunks");
    // A 32-scenario unit larger than budget / W still forms its own chunk,
    // so the rings are a soft budget: use only as many rings as the largest
    // chunk allows inside the budget (fewer rings, less overlap), and fail
    // early when one chunk alone does not fit the free memory.
    int64_t max_chunk = 1;
    for (const auto& c : chunks) max_chunk = std::max(max_chunk, c.nsamp);
    if ((size_t)max_chunk * 8 > free_b)
      throw Invalid{CACE_E_INVALID, "cace: run_metrics: one warp of scenarios needs " +
                                        std::to_string((size_t)max_chunk * 8 >> 20) +
                                        " MB of samples, more than the free device memory"};
    const size_t WR = std::max<size_t>(1, std::min<size_t>(W, budget / ((size_t)max_chunk * 8)));
    std::vector<int64_t> ring_len(W, 0);
    for (size_t j = 0; j < chunks.size(); ++j)
      ring_len[j % WR] = std::max(ring_len[j % WR], chunks[j].nsamp);
    DBuf<cace_scenario_t> d_sc;
    d_sc.upload(scenarios, n_scenarios, s);
    DBuf<cace_summary_t> d_out;
    d_out.alloc(n_scenarios, s);
    DBuf<int32_t> d_slot;
    DBuf<int64_t> d_off;
    DBuf<uint32_t> d_nc, d_nr;
    DBuf<double> d_stat;
    d_slot.upload(slot.data(), n_scenarios, s);
    d_off.upload(off.data(), NL, s);
    d_nc.upload(nc.data(), NL, s);
    d_nr.upload(nr.data(), NL, s);
    d_stat.alloc((size_t)std::max<int64_t>(NL, 1) * 8, s);
    std::vector<DBuf<double>> ring(W);
    for (size_t r = 0; r < W; ++r)
      if (ring_len[r] > 0) ring[r].alloc(ring_len[r], s);
    DumpDev dd{};
    dd.slot = d_slot.p;
    const ReplayParams P0 = replay_params(e, d_sc.p, d_out.p, dd);
    e->last_launches = 0;
    // Selects run on their own high-priority streams: the block scheduler
    // then places their CTAs ahead of queued replay blocks as SMs free up,
    // which returns ring buffers sooner.  Per ring r: replay (worker r, after
    // the previous select of r) -> select (select stream r).
    struct StreamSet {
      std::vector<cudaStream_t> st;
      std::vector<cudaEvent_t> rep, sel;
      ~StreamSet() {
        for (auto x : st) cudaStreamDestroy(x);
        for (auto x : rep) cudaEventDestroy(x);
        for (auto x : sel) cudaEventDestroy(x);
      }
    } ss;
    int prio_lo = 0, prio_hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    const size_t nring = std::min(WR, chunks.size());
    for (size_t r = 0; r < nring; ++r) {
      cudaStream_t x;
      cudaEvent_t a, b;
      CK(cudaStreamCreateWithPriority(&x, cudaStreamNonBlocking, prio_hi));
      ss.st.push_back(x);
      CK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
      ss.rep.push_back(a);
      CK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
      ss.sel.push_back(b);
    }
    // CACE_TIMING: per-chunk device timeline (replay start / end, select end)
    std::vector<cudaEvent_t> tl;
    if (pt.on)
      for (size_t j = 0; j < 3 * chunks.size() + 1; ++j) {
        cudaEvent_t x;
        CK(cudaEventCreate(&x));
        tl.push_back(x);
      }
    if (pt.on) CK(cudaEventRecord(tl.back(), s));
    // speculative first select digit (CACE_METRICS_SPEC: 0 off, 2 = test hook)
    const int metrics_spec = std::getenv("CACE_METRICS_SPEC") ? std::atoi(std::getenv("CACE_METRICS_SPEC")) : 1;
    fork_workers(e, s, chunks.size());
    for (size_t j = 0; j < chunks.size(); ++j) {
      const Chunk& c = chunks[j];
      const size_t r = j % WR;
      cudaStream_t ws = e->workers[r];
      if (j >= WR) CK(cudaStreamWaitEvent(ws, ss.sel[r], 0));  // ring r is free again
      if (pt.on) CK(cudaEventRecord(tl[3 * j], ws));
      ReplayParams P = P0;
      P.dump.dump_off = d_off.p + c.base;
      P.dump.samples = ring[r].p;
      launch_piece(e, e->segs[c.seg], P, c.b, c.e, ws, CACE_LANE_MIN_BLOCKS);
      ++e->last_launches;
      CK(cudaEventRecord(ss.rep[r], ws));
      if (pt.on) CK(cudaEventRecord(tl[3 * j + 1], ws));
      CK(cudaStreamWaitEvent(ss.st[r], ss.rep[r], 0));
      if (c.nloc > 0) {
        MetricsParams mp{ring[r].p, d_off.p + c.base, d_nc.p + c.base, d_nr.p + c.base,
                         d_stat.p + (size_t)c.base * 8, metrics_spec};
        metrics_select_kernel<<<(unsigned)(2 * c.nloc), METRICS_BLOCK, 0, ss.st[r]>>>(mp);
        CK(cudaGetLastError());
        ++e->last_launches;
      }
      CK(cudaEventRecord(ss.sel[r], ss.st[r]));
      if (pt.on) CK(cudaEventRecord(tl[3 * j + 2], ss.st[r]));
    }
    for (size_t r = 0; r < nring; ++r) CK(cudaStreamWaitEvent(s, ss.sel[r], 0));
    join_workers(e, s, chunks.size());
    fill_status(e, d_out.p, s);
    std::vector<cace_summary_t> summ(n_scenarios);
    std::vector<double> stat((size_t)NL * 8);
    if (n_scenarios > 0)
      CK(cudaMemcpyAsync(summ.data(), d_out.p, n_scenarios * sizeof(cace_summary_t), cudaMemcpyDeviceToHost, s));
    if (NL > 0) CK(cudaMemcpyAsync(stat.data(), d_stat.p, (size_t)NL * 8 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    pt.mark("replay+select");
    if (pt.on) {
      for (size_t j = 0; j < chunks.size(); ++j) {
        float a = 0, b = 0, d = 0;
        cudaEventElapsedTime(&a, tl.back(), tl[3 * j]);
        cudaEventElapsedTime(&b, tl.back(), tl[3 * j + 1]);
        cudaEventElapsedTime(&d, tl.back(), tl[3 * j + 2]);
        std::fprintf(stderr, "cace_chunk %3zu ring %zu C %2d n %6lld  replay %8.2f -> %8.2f  select -> %8.2f ms\n", j,
                     j % W, e->segs[chunks[j].seg].C, (long long)chunks[j].nloc, a, b, d);
      }
      for (auto x : tl) cudaEventDestroy(x);
    }
    for (auto& r : ring) r.release();
    // RunMetrics (compute_run_metrics, metrics.cpp:35-62)
    std::vector<int64_t> pos(n_scenarios, -1);
    for (int64_t p = 0; p < NL; ++p) pos[loc_scen[p]] = p;
    for (int64_t i = 0; i < n_scenarios; ++i) {
      const cace_summary_t& o = summ[i];
      cace_run_metrics_t& m = metrics[i];
      std::memset(&m, 0, sizeof(m));
      m.status = o.status;
      if (o.status != CACE_OK) continue;
      const int64_t p = pos[i];
      if (p < 0 || o.hits + o.misses == 0) {  // p < 0: a valid scenario on an empty trace
        m.status = CACE_E_METRICS_EMPTY;
        continue;
      }
      if (nc[p] == 0) {
        m.status = CACE_E_METRICS_NO_TTFT;
        continue;
      }
      if (nr[p] - nc[p] == 0) {
        m.status = CACE_E_METRICS_NO_E2E;
        continue;
      }
      m.cache_hit_rate = (double)o.hits / (double)(o.hits + o.misses);
      m.load_overhead_s = o.load_overhead_s;
      m.evictions = (double)o.evictions;
      const double* st = stat.data() + (size_t)p * 8;
      auto fill = [&](cace_latency_summary_t& ls, uint64_t cnt, double sum, const double* q) {
        ls.count = cnt;
        ls.mean_s = sum / (double)cnt;  // replay-order sum (the reference sums the sorted samples)
        ls.p50_s = q[0];
        ls.p95_s = q[1];
        ls.p99_s = q[2];
        ls.max_s = q[3];
      };
      fill(m.ttft_completion, nc[p], o.sum_ttft_completion, st);
      fill(m.e2e_reasoning, nr[p] - nc[p], o.sum_e2e_reasoning, st + 4);
    }
    if (summaries && n_scenarios > 0) std::memcpy(summaries, summ.data(), n_scenarios * sizeof(cace_summary_t));
    pt.mark("post");
    for (int64_t i = 0; i < n_scenarios; ++i)
      if (metrics[i].status != CACE_OK) {
        put_msg(msg, msg_cap, status_text(e->cat, metrics[i].status));
        return metrics[i].status & 0xff;
      }
    return CACE_OK;
  });
  cace_engine_destroy(e);
  pt.mark("destroy");
  return rc;
}

int32_t cace_metrics_select(const double* samples, const int64_t* off, const uint32_t* ncomp,
                            const uint32_t* nreq, int64_t n_segments, double* stat, int32_t spec,
                            const cace_opts_t* opts, char* msg, size_t msg_cap) {
  return guarded(msg, msg_cap, [&]() -> int32_t {
    require_device(opts);
    if (n_segments <= 0) return CACE_OK;
    if (!samples || !off || !ncomp || !nreq || !stat) throw Invalid{CACE_E_INVALID, "cace: NULL argument"};
    int64_t total = 0;
    for (int64_t b = 0; b < n_segments; ++b) {
      if (ncomp[b] > nreq[b] || off[b] < 0) throw Invalid{CACE_E_INVALID, "cace: bad segment"};
      total = std::max<int64_t>(total, off[b] + (int64_t)nreq[b]);
    }
    {
      // the select compacts each segment in place: segments must not overlap
      std::vector<int64_t> ord(n_segments);
      std::iota(ord.begin(), ord.end(), 0);
      std::sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return off[a] < off[b]; });
      for (int64_t q = 1; q < n_segments; ++q)
        if (nreq[ord[q - 1]] > 0 && nreq[ord[q]] > 0 && off[ord[q - 1]] + (int64_t)nreq[ord[q - 1]] > off[ord[q]])
          throw Invalid{CACE_E_INVALID, "cace: overlapping sample segments"};
    }
    cudaStream_t s = opts && opts->stream ? static_cast<cudaStream_t>(opts->stream) : nullptr;
    DBuf<double> d_samp, d_stat;
    DBuf<int64_t> d_off;
    DBuf<uint32_t> d_nc, d_nr;
    d_samp.upload(samples, std::max<int64_t>(total, 1), s);
    d_off.upload(off, n_segments, s);
    d_nc.upload(ncomp, n_segments, s);
    d_nr.upload(nreq, n_segments, s);
    d_stat.alloc((size_t)n_segments * 8, s);
    MetricsParams mp{d_samp.p, d_off.p, d_nc.p, d_nr.p, d_stat.p, spec};
    metrics_select_kernel<<<(unsigned)(2 * n_segments), METRICS_BLOCK, 0, s>>>(mp);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(stat, d_stat.p, (size_t)n_segments * 8 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return CACE_OK;
  });
}

// ---------------- trace ingestion (parse_trace / load_trace) --------------

struct cace_trace_jsonl {
  ParsedTrace t;
};

int32_t cace_trace_parse_jsonl(const char* text, size_t len, cace_trace_jsonl** out, char* msg,
                               size_t msg_cap) {
  if (!out) return CACE_E_INVALID;
  *out = nullptr;
  if (!text && len) return CACE_E_INVALID;
  try {
    auto* h = new cace_trace_jsonl();
    try {
      h->t = parse_trace_jsonl(text ? text : "", len);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
    return CACE_OK;
  } catch (const jsonl::TraceError& x) {
    put_msg(msg, msg_cap, x.what);
    return CACE_E_PARSE;
  } catch (const std::exception& x) {
    put_msg(msg, msg_cap, x.what());
    return CACE_E_INVALID;
  }
}

int32_t cace_trace_load_jsonl(const char* path, cace_trace_jsonl** out, char* msg, size_t msg_cap) {
  if (!out || !path) return CACE_E_INVALID;
  *out = nullptr;
  // load_trace (workload.cpp:274-280)
  FILE* f = std::fopen(path, "rb");
  if (!f) {
    put_msg(msg, msg_cap, std::string("trace: cannot open: ") + path);
    return CACE_E_IO;
  }
  std::string buf;
  std::fseek(f, 0, SEEK_END);
  const long sz = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  if (sz > 0) {
    buf.resize((size_t)sz);
    const size_t got = std::fread(&buf[0], 1, (size_t)sz, f);
    buf.resize(got);
  }
  std::fclose(f);
  return cace_trace_parse_jsonl(buf.data(), buf.size(), out, msg, msg_cap);
}

int64_t cace_trace_jsonl_size(const cace_trace_jsonl* h) {
  return h ? (int64_t)h->t.arrival.size() : 0;
}

void cace_trace_jsonl_header(const cace_trace_jsonl* h, int32_t* pattern, uint64_t* seed,
                             double* rate, double* duration, int32_t* windows) {
  if (!h) return;
  if (pattern) *pattern = h->t.pattern;
  if (seed) *seed = h->t.seed;
  if (rate) *rate = h->t.rate;
  if (duration) *duration = h->t.duration;
  if (windows) *windows = h->t.windows;
}

void cace_trace_jsonl_copy(const cace_trace_jsonl* h, uint64_t* request_id, double* arrival,
                           int32_t* language, int32_t* task_class, int32_t* prompt_tokens,
                           int32_t* output_tokens) {
  if (!h) return;
  const ParsedTrace& t = h->t;
  const size_t n = t.arrival.size();
  if (request_id && n) std::memcpy(request_id, t.request_id.data(), n * 8);
  if (arrival && n) std::memcpy(arrival, t.arrival.data(), n * 8);
  if (language && n) std::memcpy(language, t.language.data(), n * 4);
  if (task_class && n) std::memcpy(task_class, t.task_class.data(), n * 4);
  if (prompt_tokens && n) std::memcpy(prompt_tokens, t.prompt.data(), n * 4);
  if (output_tokens && n) std::memcpy(output_tokens, t.output.data(), n * 4);
}

void cace_trace_jsonl_free(cace_trace_jsonl* h) { delete h; }

// ---------------- policy-level batch entry points ------------------------

int32_t cace_select_victim_batch(const cace_catalog_t* catalog, int64_t n_instances,
                                 int32_t max_entries, const int32_t* n_entries,
                                 const int32_t* entry_model, const double* entry_last_used,
                                 const uint8_t* entry_busy, int32_t max_window,
                                 const int32_t* n_window, const int32_t* window_models,
                                 const double* clock, const cace_scenario_t* policy,
                                 int32_t* victim_out, const cace_opts_t* opts, char* msg,
                                 size_t msg_cap) {
  return guarded(msg, msg_cap, [&]() -> int32_t {
    require_device(opts);
    Catalog cat;
    cat.load(catalog);
    if (n_instances <= 0) return CACE_OK;
    cudaStream_t s = opts && opts->stream ? static_cast<cudaStream_t>(opts->stream) : nullptr;
    cat.upload(s);
    const size_t NE = (size_t)n_instances * max_entries, NW = (size_t)n_instances * max_window;
    DBuf<int32_t> d_ne, d_em, d_nw, d_wm, d_v, d_st;
    DBuf<double> d_lu, d_clk, d_tab, d_tab2;
    DBuf<uint8_t> d_busy;
    DBuf<cace_scenario_t> d_pol;
    d_ne.upload(n_entries, n_instances, s);
    d_em.upload(entry_model, NE, s);
    d_lu.upload(entry_last_used, NE, s);
    d_busy.upload(entry_busy, NE, s);
    d_nw.upload(n_window, n_instances, s);
    if (NW) d_wm.upload(window_models, NW, s);
    d_clk.upload(clock, n_instances, s);
    d_pol.upload(policy, n_instances, s);
    d_tab.upload(kLogTab, 256, s);
    d_tab2.upload(kLogTab2, 256, s);
    d_v.alloc(n_instances, s);
    d_st.alloc(n_instances, s);
    select_victim_kernel<<<(unsigned)((n_instances + 127) / 128), 128, 0, s>>>(
        cat.dev(), n_instances, max_entries, d_ne.p, d_em.p, d_lu.p, d_busy.p, max_window, d_nw.p,
        d_wm.p, d_clk.p, d_pol.p, d_tab.p, d_tab2.p, resolve_log_variant(opts), d_v.p, d_st.p);
    CK(cudaGetLastError());
    std::vector<int32_t> st(n_instances);
    CK(cudaMemcpyAsync(victim_out, d_v.p, n_instances * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(st.data(), d_st.p, n_instances * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int64_t b = 0; b < n_instances; ++b)
      if (st[b] != CACE_OK) {
        const int m = st[b] >> 8;
        put_msg(msg, msg_cap,
                (st[b] & 0xff) == CACE_E_CLOCK
                    ? "eviction_score: clock precedes last_used_s for " + model_name(cat.ids, m)
                    : "catalog: unknown model_id " + model_name(cat.ids, m));
        return st[b] & 0xff;
      }
    return CACE_OK;
  });
}

int32_t cace_eviction_score_batch(const cace_catalog_t* catalog, int64_t n_instances,
                                  const int32_t* model, const double* last_used,
                                  int32_t max_window, const int32_t* n_window,
                                  const int32_t* window_models, const double* clock,
                                  const cace_scenario_t* policy, double* out,
                                  const cace_opts_t* opts, char* msg, size_t msg_cap) {
  return guarded(msg, msg_cap, [&]() -> int32_t {
    require_device(opts);
    Catalog cat;
    cat.load(catalog);
    if (n_instances <= 0) return CACE_OK;
    cudaStream_t s = opts && opts->stream ? static_cast<cudaStream_t>(opts->stream) : nullptr;
    cat.upload(s);
    const size_t NW = (size_t)n_instances * max_window;
    DBuf<int32_t> d_m, d_nw, d_wm, d_st;
    DBuf<double> d_lu, d_clk, d_out, d_tab, d_tab2;
    DBuf<cace_scenario_t> d_pol;
    d_m.upload(model, n_instances, s);
    d_lu.upload(last_used, n_instances, s);
    d_nw.upload(n_window, n_instances, s);
    if (NW) d_wm.upload(window_models, NW, s);
    d_clk.upload(clock, n_instances, s);
    d_pol.upload(policy, n_instances, s);
    d_tab.upload(kLogTab, 256, s);
    d_tab2.upload(kLogTab2, 256, s);
    d_out.alloc((size_t)n_instances * 5, s);
    d_st.alloc(n_instances, s);
    eviction_score_kernel<<<(unsigned)((n_instances + 127) / 128), 128, 0, s>>>(
        cat.dev(), n_instances, d_m.p, d_lu.p, max_window, d_nw.p, d_wm.p, d_clk.p, d_pol.p,
        d_tab.p, d_tab2.p, resolve_log_variant(opts), d_out.p, d_st.p);
    CK(cudaGetLastError());
    std::vector<int32_t> st(n_instances);
    CK(cudaMemcpyAsync(out, d_out.p, (size_t)n_instances * 5 * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(st.data(), d_st.p, n_instances * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int64_t b = 0; b < n_instances; ++b)
      if (st[b] != CACE_OK) {
        put_msg(msg, msg_cap,
                "eviction_score: clock precedes last_used_s for " + model_name(cat.ids, model[b]));
        return CACE_E_CLOCK;
      }
    return CACE_OK;
  });
}

int32_t cace_dedup_window_batch(int64_t n_instances, int32_t max_pending, const int32_t* n_pending,
                                const int32_t* pending_models, const int32_t* length,
                                int32_t* out_models, int32_t* n_out, const cace_opts_t* opts,
                                char* msg, size_t msg_cap) {
  return guarded(msg, msg_cap, [&]() -> int32_t {
    require_device(opts);
    for (int64_t b = 0; b < n_instances; ++b)
      if (length[b] < 1) {  // policy.cpp:23
        put_msg(msg, msg_cap, "dedup_window: length must be >= 1");
        return CACE_E_DEDUP_LENGTH;
      }
    if (n_instances <= 0) return CACE_OK;
    cudaStream_t s = opts && opts->stream ? static_cast<cudaStream_t>(opts->stream) : nullptr;
    const size_t NP = (size_t)n_instances * max_pending;
    DBuf<int32_t> d_np, d_pm, d_len, d_om, d_no;
    d_np.upload(n_pending, n_instances, s);
    if (NP) d_pm.upload(pending_models, NP, s);
    d_len.upload(length, n_instances, s);
    d_om.alloc(NP ? NP : 1, s);
    d_no.alloc(n_instances, s);
    dedup_window_kernel<<<(unsigned)((n_instances + 127) / 128), 128, 0, s>>>(
        n_instances, max_pending, d_np.p, d_pm.p, d_len.p, d_om.p, d_no.p);
    CK(cudaGetLastError());
    if (NP) CK(cudaMemcpyAsync(out_models, d_om.p, NP * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(n_out, d_no.p, n_instances * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return CACE_OK;
  });
}

int32_t cace_service_times_batch(const cace_catalog_t* catalog, int64_t n, const int32_t* model,
                                 const int32_t* prompt_tokens, const int32_t* output_tokens,
                                 double* prefill_s, double* decode_s, const cace_opts_t* opts,
                                 char* msg, size_t msg_cap) {
  return guarded(msg, msg_cap, [&]() -> int32_t {
    require_device(opts);
    Catalog cat;
    cat.load(catalog);
    for (int64_t i = 0; i < n; ++i) {
      const int m = model[i];
      if (m < 0 || m >= cat.M) throw Invalid{CACE_E_LOOKUP, "catalog: unknown model index"};
      if (cat.bad_rates(m)) {  // engine.cpp:17-20
        put_msg(msg, msg_cap, "service_times: rates must be positive for " + model_name(cat.ids, m));
        return CACE_E_RATES;
      }
    }
    if (n <= 0) return CACE_OK;
    cudaStream_t s = opts && opts->stream ? static_cast<cudaStream_t>(opts->stream) : nullptr;
    DBuf<double> d_pr, d_dr, d_pf, d_dc;
    DBuf<int32_t> d_m, d_p, d_o;
    d_pr.upload(cat.pr.data(), cat.M, s);
    d_dr.upload(cat.dr.data(), cat.M, s);
    d_m.upload(model, n, s);
    d_p.upload(prompt_tokens, n, s);
    d_o.upload(output_tokens, n, s);
    d_pf.alloc(n, s);
    d_dc.alloc(n, s);
    service_times_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, d_m.p, d_p.p, d_o.p, d_pr.p,
                                                                      d_dr.p, d_pf.p, d_dc.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(prefill_s, d_pf.p, n * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(decode_s, d_dc.p, n * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return CACE_OK;
  });
}

int32_t cace_log_selftest(const double* x, int64_t n, int32_t log_variant, double* out,
                          const cace_opts_t* opts, char* msg, size_t msg_cap) {
  return guarded(msg, msg_cap, [&]() -> int32_t {
    require_device(opts);
    if (n <= 0) return CACE_OK;
    cudaStream_t s = opts && opts->stream ? static_cast<cudaStream_t>(opts->stream) : nullptr;
    const int v = log_variant >= 0 ? log_variant : resolve_log_variant(opts);
    DBuf<double> d_x, d_o, d_tab, d_tab2;
    d_x.upload(x, n, s);
    d_o.alloc(n, s);
    d_tab.upload(kLogTab, 256, s);
    d_tab2.upload(kLogTab2, 256, s);
    log_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, d_x.p, v, d_tab.p, d_tab2.p, d_o.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, d_o.p, n * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return CACE_OK;
  });
}

void cace_log_host(const double* x, int64_t n, int32_t log_variant, double* out) {
  const int v = log_variant >= 0 ? log_variant : resolve_log_variant(nullptr);
  for (int64_t i = 0; i < n; ++i) out[i] = cace_glibc_log(x[i], v, kLogTab, kLogTab2);
}

int32_t cace_probe_log_variant(void) { return probe_log_variant(); }

}  // extern "C"
