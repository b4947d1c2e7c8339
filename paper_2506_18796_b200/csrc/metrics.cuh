// Per-scenario order statistics for RunMetrics (compute_run_metrics,
// metrics.cpp:35-62; nearest-rank summarize, metrics.cpp:14-33).
//
// The replay kernels (DUMP instantiation with dump.samples set) write, per
// scenario, the TTFT of its completion requests followed by the E2E of its
// reasoning requests.  One CTA per (scenario, class) segment then finds the
// nearest-rank p50 / p95 / p99 and the max by an MSD radix select over the
// samples' IEEE bit patterns (latencies are >= +0, so unsigned order is
// numeric order): 8 passes of 8 bits, one 256-bin shared histogram per
// distinct target prefix, warp-aggregated increments (__match_any_sync) so
// the heavily shared exponent bytes do not serialise on one bank.  The
// selected values are the exact samples the reference's sorted vector holds
// at those ranks.
#pragma once
#include <math.h>
#include <stdint.h>

namespace cace {

struct MetricsParams {
  double* samples;         // batch sample buffer (the select compacts it in place)
  const int64_t* off;      // [B] first sample of batch scenario b
  const uint32_t* ncomp;   // [B] completion requests of b's trace
  const uint32_t* nreq;    // [B] requests of b's trace
  double* stat;            // [B][2][4]: {p50, p95, p99, max} for TTFT (class 0) and E2E (class 1)
  int spec;                // speculative first digit: 0 off, 1 on, 2 on with wrong guesses (test hook)
};

// Zero-based nearest rank of summarize (metrics.cpp:18-22):
// r = clamp(ceil(q * n), 1, n), the same fp64 operations as the reference.
__host__ __device__ inline uint32_t nearest_rank0(double q, uint32_t n) {
  const double r = ceil(q * (double)n);
  uint64_t ri = r < 1.0 ? 1u : (uint64_t)r;
  if (ri > n) ri = n;
  return (uint32_t)(ri - 1);
}

constexpr int METRICS_BLOCK = 256;
constexpr int METRICS_LIST = 5120;  // keys kept in shared memory once the prefixes are narrow
constexpr int METRICS_UNROLL = 8;   // keys per thread per tile
constexpr int METRICS_SAMPLE = 2048;      // keys sampled to guess the targets' top bytes
constexpr uint32_t METRICS_SPEC_MIN = 16384;  // segments at least this long speculate

// Selected digit bookkeeping, one warp per target (see the kernel).
__device__ inline void metrics_place(const uint32_t* h, int lane, uint32_t* krem, uint64_t* prefix,
                                     uint32_t* cnt, int shift, uint32_t* found = nullptr) {
  uint32_t c[8], sum = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    c[j] = h[lane * 8 + j];
    sum += c[j];
  }
  uint32_t incl = sum;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t excl = incl - sum;
  const uint32_t k = *krem;
  __syncwarp();  // every lane has read krem before one lane rewrites it
  if (k >= excl && k < incl) {  // exactly one lane holds rank k's bin
    uint32_t cum = excl;
    int d = -1;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (d < 0) {
        if (k < cum + c[j])
          d = j;
        else
          cum += c[j];
      }
    }
    *krem = k - cum;
    *prefix |= (uint64_t)(lane * 8 + d) << shift;
    *cnt = c[d];  // keys under the extended prefix
    if (found) *found = 1;
  }
}

// One histogram pass over src[0, slen).  FIRST: the first pass (empty
// prefixes: the digit is the key's top byte; also reduces the max).  HI32:
// shift >= 32, so prefixes and digit live in the high word (32-bit compares).
// COMPACT: keys under a target prefix are written back in place (see the
// kernel).  Lanes with equal bins add once (__match_any_sync).
template <bool FIRST, bool HI32, bool COMPACT>
__device__ __forceinline__ void metrics_pass(uint64_t* src, uint32_t slen, int shift, uint64_t mask,
                                             uint64_t q0, uint64_t q1, uint64_t q2, bool d1, bool d2,
                                             uint32_t* hist, uint32_t* nlist, uint64_t& mx) {
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const uint32_t mh = (uint32_t)(mask >> 32);
  const uint32_t h0 = (uint32_t)(q0 >> 32), h1 = (uint32_t)(q1 >> 32), h2 = (uint32_t)(q2 >> 32);
  for (uint32_t base = 0; base < slen; base += METRICS_BLOCK * METRICS_UNROLL) {
    uint64_t v[METRICS_UNROLL];
#pragma unroll
    for (int u = 0; u < METRICS_UNROLL; ++u) {
      const uint32_t i = base + u * METRICS_BLOCK + threadIdx.x;
      v[u] = i < slen ? src[i] : 0ull;
    }
    if (COMPACT) __syncthreads();  // the whole tile is read before any write-back
#pragma unroll
    for (int u = 0; u < METRICS_UNROLL; ++u) {
      const bool valid = base + u * METRICS_BLOCK + threadIdx.x < slen;
      const unsigned act = __ballot_sync(0xffffffffu, valid);
      if (!act) continue;
      bool m0, m1, m2;
      int d;
      if (FIRST) {
        m0 = true;
        m1 = m2 = false;
        d = (int)(v[u] >> 56);
      } else if (HI32) {
        const uint32_t ph = (uint32_t)(v[u] >> 32) & mh;
        m0 = ph == h0;
        m1 = ph == h1;
        m2 = ph == h2;
        d = (int)(((uint32_t)(v[u] >> 32) >> (shift - 32)) & 255u);
      } else {
        const uint64_t pv = v[u] & mask;
        m0 = pv == q0;
        m1 = pv == q1;
        m2 = pv == q2;
        d = (int)((v[u] >> shift) & 255u);
      }
      if (valid) {
        if (FIRST) mx = max(mx, v[u]);
        // one histogram per distinct prefix; lanes with the same bin add once
        const int key = m0 ? d : ((d1 && m1) ? 256 + d : ((d2 && m2) ? 512 + d : -1));
        const unsigned peers = __match_any_sync(act, key);
        if (key >= 0 && (peers & lt_mask) == 0) atomicAdd(&hist[key], (uint32_t)__popc(peers));
      }
      if (COMPACT) {
        const bool keep = valid && (m0 || m1 || m2);
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        uint32_t wb = 0;
        if (lane == 0 && bal) wb = atomicAdd(nlist, (uint32_t)__popc(bal));
        wb = __shfl_sync(0xffffffffu, wb, 0);
        if (keep) src[wb + __popc(bal & lt_mask)] = v[u];
      }
    }
  }
}

// The first two digits in one read, given guessed top bytes g0..g2: histogram
// of bits 55..48 of the keys whose top byte is g_t (one histogram per
// distinct guess), count of keys whose top byte is below g_t, and the max.
__device__ __forceinline__ void metrics_spec_pass(const uint64_t* x, uint32_t len, uint32_t g0, uint32_t g1,
                                                  uint32_t g2, bool d1, bool d2, uint32_t* hist,
                                                  uint32_t& l0, uint32_t& l1, uint32_t& l2, uint64_t& mx) {
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (uint32_t base = 0; base < len; base += METRICS_BLOCK * METRICS_UNROLL) {
    uint64_t v[METRICS_UNROLL];
#pragma unroll
    for (int u = 0; u < METRICS_UNROLL; ++u) {
      const uint32_t i = base + u * METRICS_BLOCK + threadIdx.x;
      v[u] = i < len ? x[i] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < METRICS_UNROLL; ++u) {
      const bool valid = base + u * METRICS_BLOCK + threadIdx.x < len;
      const unsigned act = __ballot_sync(0xffffffffu, valid);
      if (!act) continue;
      if (valid) {
        const uint32_t hi = (uint32_t)(v[u] >> 32);
        const uint32_t top = hi >> 24;
        const int d = (int)((hi >> 16) & 255u);
        l0 += top < g0;
        l1 += top < g1;
        l2 += top < g2;
        mx = max(mx, v[u]);
        const int key = top == g0 ? d : ((d1 && top == g1) ? 256 + d : ((d2 && top == g2) ? 512 + d : -1));
        const unsigned peers = __match_any_sync(act, key);
        if (key >= 0 && (peers & lt_mask) == 0) atomicAdd(&hist[key], (uint32_t)__popc(peers));
      }
    }
  }
}

__global__ void __launch_bounds__(METRICS_BLOCK) metrics_select_kernel(MetricsParams P) {
  const int seg = blockIdx.x;  // 2 * b + class
  const int b = seg >> 1, cls = seg & 1;
  const uint32_t nc = P.ncomp[b], n = P.nreq[b];
  const uint32_t len = cls ? n - nc : nc;
  // the segment is this CTA's own: later passes compact it in place
  uint64_t* x = reinterpret_cast<uint64_t*>(P.samples + P.off[b] + (cls ? nc : 0));
  double* out = P.stat + (size_t)seg * 4;
  if (len == 0) {  // compute_run_metrics throws; the host reports it
    if (threadIdx.x < 4) out[threadIdx.x] = 0.0;
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ uint32_t hist[3][256];
  __shared__ uint64_t s_prefix[3];
  __shared__ uint32_t s_krem[3];
  __shared__ uint32_t s_cnt[3];  // keys under each target's prefix
  __shared__ int s_src[3];  // target whose histogram this target shares (distinct prefixes only)
  __shared__ uint64_t s_max[METRICS_BLOCK / 32];
  __shared__ uint64_t s_list[METRICS_LIST];  // keys matching a target prefix (after compaction)
  __shared__ uint32_t s_nlist;
  __shared__ uint32_t s_less[3], s_found[3], s_tk[3], s_tc[3];

  if (threadIdx.x < 3) {
    const double q = threadIdx.x == 0 ? 0.50 : (threadIdx.x == 1 ? 0.95 : 0.99);
    s_krem[threadIdx.x] = nearest_rank0(q, len);
    s_prefix[threadIdx.x] = 0;
    s_cnt[threadIdx.x] = len;
  }
  __syncthreads();

  // MSD passes.  Keys under the targets' current prefixes (the selected bins
  // of the previous pass, `need` of them) are the only ones later passes
  // look at, so the working set shrinks as soon as it pays:
  //  * need <= METRICS_LIST: copied once into shared memory;
  //  * need <= half the working set: compacted in place in global memory
  //    during the pass (tiles are read completely before any of their keys
  //    is written back, and a key is only written at a position that has
  //    already been read), which handles heavy bins of identical samples.
  // The max (last order statistic) is reduced during the first pass.
  uint64_t* src = x;
  uint32_t slen = len;
  bool in_smem = false;
  uint64_t mx = 0;
  int start = 56;
  if (P.spec && len >= METRICS_SPEC_MIN) {
    // Speculative first digit: the targets' top bytes (sign + 7 exponent
    // bits) guessed from a strided sample, then one full read does digits 1
    // and 2 (keys below each guess are counted, so a wrong guess is detected
    // exactly: the target rank must fall inside the guessed bin).  A miss
    // restarts the plain passes, so results never depend on the guess.
    uint32_t* h0 = &hist[0][0];
    for (int i = threadIdx.x; i < 256; i += METRICS_BLOCK) h0[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < METRICS_SAMPLE; i += METRICS_BLOCK) {
      const uint32_t d = (uint32_t)(x[(uint64_t)i * len / METRICS_SAMPLE] >> 56);
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      if ((peers & ((1u << lane) - 1u)) == 0) atomicAdd(&h0[d], (uint32_t)__popc(peers));
    }
    __syncthreads();
    if (warp < 3) {
      uint64_t g = 0;
      if (lane == 0) s_tk[warp] = (uint32_t)((uint64_t)s_krem[warp] * METRICS_SAMPLE / len);
      __syncwarp();
      metrics_place(h0, lane, &s_tk[warp], &g, &s_tc[warp], 56);
      // the lane that found the bin holds g; the others hold 0
      uint32_t gh = __reduce_or_sync(0xffffffffu, (uint32_t)(g >> 32));
      g = gh;
      if (P.spec == 2) g ^= 1u << 24;  // test hook: every guess wrong -> the fallback path
      if (lane == 0) s_prefix[warp] = (uint64_t)g << 32;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
      const int t = threadIdx.x;
      int sr = t;
      for (int u = 0; u < t; ++u)
        if (s_prefix[u] == s_prefix[t]) {
          sr = u;
          break;
        }
      s_src[t] = sr;
      s_less[t] = 0;
      s_found[t] = 0;
    }
    for (int i = threadIdx.x; i < 3 * 256; i += METRICS_BLOCK) (&hist[0][0])[i] = 0;
    __syncthreads();
    uint32_t l0 = 0, l1 = 0, l2 = 0;
    metrics_spec_pass(x, len, (uint32_t)(s_prefix[0] >> 56), (uint32_t)(s_prefix[1] >> 56),
                      (uint32_t)(s_prefix[2] >> 56), s_src[1] == 1, s_src[2] == 2, &hist[0][0], l0, l1, l2, mx);
    l0 = __reduce_add_sync(0xffffffffu, l0);
    l1 = __reduce_add_sync(0xffffffffu, l1);
    l2 = __reduce_add_sync(0xffffffffu, l2);
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) {
      atomicAdd(&s_less[0], l0);
      atomicAdd(&s_less[1], l1);
      atomicAdd(&s_less[2], l2);
      s_max[warp] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t m = s_max[0];
      for (int w = 1; w < METRICS_BLOCK / 32; ++w) m = max(m, s_max[w]);
      out[3] = __longlong_as_double((long long)m);
    }
    if (threadIdx.x < 3) {
      const uint32_t k = s_krem[threadIdx.x];
      s_krem[threadIdx.x] = k >= s_less[threadIdx.x] ? k - s_less[threadIdx.x] : 0xffffffffu;
    }
    __syncthreads();
    if (warp < 3) metrics_place(hist[s_src[warp]], lane, &s_krem[warp], &s_prefix[warp], &s_cnt[warp], 48, &s_found[warp]);
    __syncthreads();
    if (s_found[0] & s_found[1] & s_found[2]) {
      start = 40;
    } else {
      __syncthreads();  // every thread has read s_found
      if (threadIdx.x < 3) {
        const double q = threadIdx.x == 0 ? 0.50 : (threadIdx.x == 1 ? 0.95 : 0.99);
        s_krem[threadIdx.x] = nearest_rank0(q, len);
        s_prefix[threadIdx.x] = 0;
        s_cnt[threadIdx.x] = len;
      }
      mx = 0;
      __syncthreads();
    }
  }
  for (int shift = start; shift >= 0; shift -= 8) {
    const uint64_t mask = shift == 56 ? 0ull : (~0ull << (shift + 8));
    const uint64_t q0 = s_prefix[0], q1 = s_prefix[1], q2 = s_prefix[2];
    const uint32_t need = s_cnt[0] + (q1 != q0 ? s_cnt[1] : 0u) + (q2 != q0 && q2 != q1 ? s_cnt[2] : 0u);
    bool compact = false;
    if (shift < 56 && !in_smem && need <= (uint32_t)METRICS_LIST) {
      if (threadIdx.x == 0) s_nlist = 0;
      __syncthreads();
      for (uint32_t base = 0; base < slen; base += METRICS_BLOCK * 4) {
        uint64_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t i = base + u * METRICS_BLOCK + threadIdx.x;
          v[u] = i < slen ? src[i] : 0ull;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint64_t pv = v[u] & mask;
          if (base + u * METRICS_BLOCK + threadIdx.x < slen && (pv == q0 || pv == q1 || pv == q2))
            s_list[atomicAdd(&s_nlist, 1u)] = v[u];
        }
      }
      __syncthreads();
      src = s_list;
      slen = s_nlist;
      in_smem = true;
    } else if (shift < 56 && !in_smem && need <= slen / 2) {
      compact = true;
    }
    if (threadIdx.x < 3) {
      const int t = threadIdx.x;
      int sr = t;
      for (int u = 0; u < t; ++u)
        if (s_prefix[u] == s_prefix[t]) {
          sr = u;
          break;
        }
      s_src[t] = sr;
    }
    if (compact && threadIdx.x == 0) s_nlist = 0;  // (not after the shared copy: slen was just read from it)
    for (int i = threadIdx.x; i < 3 * 256; i += METRICS_BLOCK) (&hist[0][0])[i] = 0;
    __syncthreads();
    const bool d1 = s_src[1] == 1, d2 = s_src[2] == 2;  // distinct histograms needed
    uint32_t* hf = &hist[0][0];
    if (shift == 56)
      metrics_pass<true, true, false>(src, slen, shift, mask, q0, q1, q2, d1, d2, hf, &s_nlist, mx);
    else if (shift >= 32)
      compact ? metrics_pass<false, true, true>(src, slen, shift, mask, q0, q1, q2, d1, d2, hf, &s_nlist, mx)
              : metrics_pass<false, true, false>(src, slen, shift, mask, q0, q1, q2, d1, d2, hf, &s_nlist, mx);
    else
      compact ? metrics_pass<false, false, true>(src, slen, shift, mask, q0, q1, q2, d1, d2, hf, &s_nlist, mx)
              : metrics_pass<false, false, false>(src, slen, shift, mask, q0, q1, q2, d1, d2, hf, &s_nlist, mx);
    if (shift == 56) {
      for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) s_max[warp] = mx;
    }
    __syncthreads();
    if (shift == 56 && threadIdx.x == 0) {
      uint64_t m = s_max[0];
      for (int w = 1; w < METRICS_BLOCK / 32; ++w) m = max(m, s_max[w]);
      out[3] = __longlong_as_double((long long)m);
    }
    if (compact) slen = s_nlist;
    // digit of each target: warp t scans its (shared) histogram
    if (warp < 3) metrics_place(hist[s_src[warp]], lane, &s_krem[warp], &s_prefix[warp], &s_cnt[warp], shift);
    __syncthreads();
  }
  if (threadIdx.x < 3) out[threadIdx.x] = __longlong_as_double((long long)s_prefix[threadIdx.x]);
}

}  // namespace cace
