// Bit-exact restatement of glibc 2.39 `log` (the function the reference calls
// for P1, policy.cpp:51 -> log@@GLIBC_2.29) for the device and the host.
//
// glibc's log is the table-driven ARM optimized-routines algorithm
// (sysdeps/ieee754/dbl-64/e_log.c; constants in glibc_log_data.h, extracted by
// tools/gen_glibc_log_data.py).  It is NOT correctly rounded, and its two
// x86-64 ifunc variants round differently:
//   * CACE_LOG_FMA  — `__log_fma`, selected when the host CPU has FMA+AVX2
//     (the compiler contracted a*b+c into FMAs; the exact contraction pattern
//     below was read from the library's disassembly, libm.so.6 @0x79d50).
//   * CACE_LOG_SSE2 — the plain `__log` (@0x2b3d0) and the AVX build
//     (@0x834f0), no contraction; r uses the tab2 {chi,clo} split.
// The host probes its own libm once (capi: cace_probe_log_variant) and the
// kernels evaluate the matching variant, so P1 is bit-identical to the
// reference's std::log on the same machine.  Neither CUDA's log() (<=1 ulp)
// nor a correctly rounded log reproduces these bits.
#pragma once
#include <stdint.h>

#include "glibc_log_data.h"

#if defined(__CUDACC__)
#define CACE_HD __host__ __device__ __forceinline__
#else
#define CACE_HD inline
#endif

#if defined(__CUDA_ARCH__)
#define CL_FMA(a, b, c) __fma_rn((a), (b), (c))
#define CL_ADD(a, b) __dadd_rn((a), (b))
#define CL_SUB(a, b) __dsub_rn((a), (b))
#define CL_MUL(a, b) __dmul_rn((a), (b))
#define CL_AS_U64(x) ((uint64_t)__double_as_longlong(x))
#define CL_AS_F64(u) __longlong_as_double((long long)(u))
#define CL_LDG(p) __ldg(p)
#else
#include <math.h>
#include <string.h>
// Host build must use -ffp-contract=off so these stay separate roundings.
#define CL_FMA(a, b, c) fma((a), (b), (c))
#define CL_ADD(a, b) ((a) + (b))
#define CL_SUB(a, b) ((a) - (b))
#define CL_MUL(a, b) ((a) * (b))
static inline uint64_t cl_as_u64(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
static inline double cl_as_f64(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }
#define CL_AS_U64(x) cl_as_u64(x)
#define CL_AS_F64(u) cl_as_f64(u)
#define CL_LDG(p) (*(p))
#endif

#ifndef CACE_LOG_FMA
#define CACE_LOG_FMA 0
#define CACE_LOG_SSE2 1
#endif

// Special inputs (x <= 0, subnormal, inf, nan): never reached on the replay
// path (t = max(clock - last_used, 1) is finite and >= 1) but kept total.
CACE_HD double cace_log_special(double x, uint64_t ix) {
  if (x != x) return x;                                   // nan
  if (ix == 0x7ff0000000000000ULL) return x;              // +inf
  if ((ix << 1) == 0) return -1.0 / 0.0 * 1.0 + (x - x);  // +-0 -> -inf
  if (ix >> 63) return (x - x) / (x - x);                 // negative -> nan
  return 0.0;                                             // subnormal: caller rescales
}

// tab: 256 doubles {invc, logc} x 128; tab2: 256 doubles {chi, clo} x 128.
CACE_HD double cace_glibc_log(double x, int variant, const double* tab, const double* tab2) {
  const double B0 = CACE_GLIBC_LOG_B0, B1 = CACE_GLIBC_LOG_B1, B2 = CACE_GLIBC_LOG_B2,
               B3 = CACE_GLIBC_LOG_B3, B4 = CACE_GLIBC_LOG_B4, B5 = CACE_GLIBC_LOG_B5,
               B6 = CACE_GLIBC_LOG_B6, B7 = CACE_GLIBC_LOG_B7, B8 = CACE_GLIBC_LOG_B8,
               B9 = CACE_GLIBC_LOG_B9, B10 = CACE_GLIBC_LOG_B10;
  const double A0 = CACE_GLIBC_LOG_A0, A1 = CACE_GLIBC_LOG_A1, A2 = CACE_GLIBC_LOG_A2,
               A3 = CACE_GLIBC_LOG_A3, A4 = CACE_GLIBC_LOG_A4;
  const double Ln2hi = CACE_GLIBC_LOG_LN2HI, Ln2lo = CACE_GLIBC_LOG_LN2LO;

  uint64_t ix = CL_AS_U64(x);
  // |x - 1| small: 1 - 0x1p-4 <= x < 1 + 0x1.09p-4
  if (ix - 0x3fee000000000000ULL < 0x3090000000000ULL) {
    if (ix == 0x3ff0000000000000ULL) return 0.0;
    const double r = CL_SUB(x, 1.0);
    const double r2 = CL_MUL(r, r);
    const double r3 = CL_MUL(r, r2);
    if (variant == CACE_LOG_FMA) {
      double pa = CL_FMA(r, B2, B1);
      double pb = CL_FMA(r, B5, B4);
      double pc = CL_FMA(r, B8, B7);
      pa = CL_FMA(r2, B3, pa);
      pb = CL_FMA(r2, B6, pb);
      pc = CL_FMA(r2, B9, pc);
      pc = CL_FMA(r3, B10, pc);
      double p = CL_FMA(pc, r3, pb);
      p = CL_FMA(p, r3, pa);
      const double rw = CL_FMA(r, 0x1p27, r);       // r + w, w = r*2^27 fused
      const double rhi = CL_FMA(-0x1p27, r, rw);    // (r + w) - w fused
      const double rhi2 = CL_MUL(rhi, rhi);
      const double rlo = CL_SUB(r, rhi);
      const double hi = CL_FMA(rhi2, B0, r);        // r + rhi*rhi*B0
      const double rmh = CL_SUB(r, hi);
      const double rpr = CL_ADD(r, rhi);
      double lo = CL_FMA(rhi2, B0, rmh);            // r - hi + w
      lo = CL_FMA(CL_MUL(B0, rlo), rpr, lo);        // lo += B0*rlo*(rhi+r)
      const double y = CL_FMA(p, r3, lo);           // y = r3*P + lo
      return CL_ADD(hi, y);
    } else {
      double pc = CL_ADD(CL_ADD(CL_MUL(r, B8), B7), CL_MUL(r2, B9));
      pc = CL_ADD(pc, CL_MUL(B10, r3));
      double pb = CL_ADD(CL_ADD(CL_MUL(r, B5), B4), CL_MUL(r2, B6));
      pb = CL_ADD(pb, CL_MUL(pc, r3));
      double pa = CL_ADD(CL_ADD(CL_MUL(r, B2), B1), CL_MUL(r2, B3));
      pa = CL_ADD(pa, CL_MUL(pb, r3));
      double y = CL_MUL(pa, r3);
      const double w = CL_MUL(r, 0x1p27);
      const double rhi = CL_SUB(CL_ADD(r, w), w);
      const double rlo = CL_SUB(r, rhi);
      const double w2 = CL_MUL(CL_MUL(rhi, rhi), B0);
      const double hi = CL_ADD(r, w2);
      double lo = CL_ADD(CL_SUB(r, hi), w2);
      lo = CL_ADD(CL_MUL(CL_ADD(r, rhi), CL_MUL(B0, rlo)), lo);
      y = CL_ADD(y, lo);
      return CL_ADD(y, hi);
    }
  }
  const uint32_t top = (uint32_t)(ix >> 48);
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
    if (ix != 0 && (ix >> 63) == 0 && (top & 0x7ff0u) == 0) {
      // subnormal: normalise (x * 2^52) and fall through with k adjusted.
      ix = CL_AS_U64(CL_MUL(x, 0x1p52)) - (52ULL << 52);
    } else {
      return cace_log_special(x, ix);
    }
  }
  const uint64_t OFF = 0x3fe6000000000000ULL;
  const uint64_t tmp = ix - OFF;
  const int i = (int)((tmp >> (52 - CACE_GLIBC_LOG_TABLE_BITS)) % 128);
  const int k = (int)((int64_t)tmp >> 52);
  const uint64_t iz = ix - (tmp & (0xfffULL << 52));
  const double invc = CL_LDG(tab + 2 * i);
  const double logc = CL_LDG(tab + 2 * i + 1);
  const double z = CL_AS_F64(iz);
  const double kd = (double)k;
  if (variant == CACE_LOG_FMA) {
    const double w = CL_FMA(kd, Ln2hi, logc);
    const double r = CL_FMA(z, invc, -1.0);
    const double q = CL_FMA(r, A2, A1);
    const double hi = CL_ADD(r, w);
    const double r2 = CL_MUL(r, r);
    double lo = CL_ADD(CL_SUB(w, hi), r);
    lo = CL_FMA(kd, Ln2lo, lo);
    const double r3 = CL_MUL(r, r2);
    double p = CL_FMA(r, A4, A3);
    lo = CL_FMA(r2, A0, lo);
    p = CL_FMA(p, r2, q);
    const double y = CL_FMA(r3, p, lo);
    return CL_ADD(y, hi);
  } else {
    const double chi = CL_LDG(tab2 + 2 * i);
    const double clo = CL_LDG(tab2 + 2 * i + 1);
    const double r = CL_MUL(CL_SUB(CL_SUB(z, chi), clo), invc);
    const double w = CL_ADD(CL_MUL(kd, Ln2hi), logc);
    const double hi = CL_ADD(w, r);
    const double lo = CL_ADD(CL_ADD(CL_SUB(w, hi), r), CL_MUL(kd, Ln2lo));
    const double r2 = CL_MUL(r, r);
    double p = CL_ADD(CL_ADD(A1, CL_MUL(r, A2)), CL_MUL(r2, CL_ADD(A3, CL_MUL(r, A4))));
    double y = CL_ADD(CL_ADD(lo, CL_MUL(r2, A0)), CL_MUL(CL_MUL(r, r2), p));
    return CL_ADD(y, hi);
  }
}
