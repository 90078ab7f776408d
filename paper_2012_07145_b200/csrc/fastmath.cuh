// log1p for K2's hot loops: the feature transform log1p(f) (reference
// costmodel.py:278, np.log1p) and the softplus log1p(exp(-|z|))
// (costmodel.py:271-272, np.logaddexp).  libdevice's log1p spends ~95 SASS
// instructions per call on range splits this path never needs; this one is
// ~35 for x >= 0 and falls back to it for anything else (x < 0, inf, nan).
//
// Method: u = 1 + x rounded, with its exact error c from TwoSum, so that
// log1p(x) = log(u) + c/u to well below an ulp (the reciprocal of u
// needs only one Newton step).  log(u) is fdlibm's e_log.c reduction and
// polynomial: u = 2^k m, m in [sqrt(2)/2, sqrt(2)), f = m - 1 exact,
// s = f / (2 + f), log(1 + f) = f - (hfsq - s (hfsq + R(s^2))); the division
// is a reciprocal estimate with two Newton steps and one residual
// correction.  Error < 1 ulp, measured against long-double log1p on 10^7
// points (tools/check_log1p.cpp); libdevice's is also <= 1 ulp.  Both
// compile for the host too, so the check runs without a GPU.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>

#ifndef GS_HD
#ifdef __CUDACC__
#define GS_HD __host__ __device__ __forceinline__
#else
#define GS_HD inline
#endif
#endif

namespace gs {

GS_HD double bits_to_d(uint64_t b) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)b);
#else
  double d; std::memcpy(&d, &b, 8); return d;
#endif
}
GS_HD uint64_t d_to_bits(double d) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t b; std::memcpy(&b, &d, 8); return b;
#endif
}

// uncontracted fp64 ops (nvcc would fuse a*b+c into FMAs and move the
// rounding away from what tools/check_log1p.cpp measured on the host)
#ifdef __CUDA_ARCH__
#define GS_M(a, b) __dmul_rn((a), (b))
#define GS_A(a, b) __dadd_rn((a), (b))
#define GS_S(a, b) __dsub_rn((a), (b))
#else
#define GS_M(a, b) ((a) * (b))
#define GS_A(a, b) ((a) + (b))
#define GS_S(a, b) ((a) - (b))
#endif

// coarse reciprocal (>= 20 correct bits) of a positive normal double
GS_HD double rcp_est(double d) {
#ifdef __CUDA_ARCH__
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  return r;
#else
  return (double)(1.0f / (float)d);
#endif
}

// log1p(x) for 0 <= x < 2^1000 (finite); callers route everything else to
// ::log1p
GS_HD double log1p_pos_core(double x) {
  constexpr double Lg1 = 6.666666666666735130e-01, Lg2 = 3.999999999940941908e-01,
                   Lg3 = 2.857142874366239149e-01, Lg4 = 2.222219843214978396e-01,
                   Lg5 = 1.818357216161805012e-01, Lg6 = 1.531383769920937332e-01,
                   Lg7 = 1.479819860511658591e-01;
  constexpr double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  // TwoSum(1, x): u + c == 1 + x exactly
  const double u = GS_A(1.0, x);
  const double bv = GS_S(u, 1.0);
  const double c = GS_A(GS_S(1.0, GS_S(u, bv)), GS_S(x, bv));
  // u = 2^k m, m in [sqrt(2)/2, sqrt(2))
  uint64_t ub = d_to_bits(u);
  uint32_t hi = (uint32_t)(ub >> 32);
  int k = (int)(hi >> 20) - 1023;
  hi &= 0x000fffffu;
  const int up = hi > 0x6a09eu;            // mantissa above sqrt(2): halve it
  k += up;
  const uint64_t mb = ((uint64_t)(hi | (up ? 0x3fe00000u : 0x3ff00000u)) << 32) | (ub & 0xffffffffull);
  const double f = GS_S(bits_to_d(mb), 1.0);
  // s = f / (2 + f): estimate, two Newton steps, one residual correction
  const double d = GS_A(2.0, f);
  double r = rcp_est(d);
  r = fma(r, fma(-d, r, 1.0), r);
  r = fma(r, fma(-d, r, 1.0), r);
  double s = GS_M(f, r);
  s = fma(r, fma(-d, s, f), s);
  const double z = GS_M(s, s), w = GS_M(z, z);
  const double t1 = GS_M(w, fma(w, fma(w, Lg6, Lg4), Lg2));
  const double t2 = GS_M(z, fma(w, fma(w, fma(w, Lg7, Lg5), Lg3), Lg1));
  const double R = GS_A(t2, t1);
  const double hfsq = GS_M(GS_M(0.5, f), f);
  const double dk = (double)k;
  // c / u: |c/u| <= 2^-53 relative to 1, but for small x it is up to
  // 2^-53 / x relative to the result, so 1/u gets one Newton step (2^-44);
  // it joins the low-order terms as in fdlibm's s_log1p.c
  double ru = rcp_est(u);
  ru = fma(ru, fma(-u, ru, 1.0), ru);
  const double cu = GS_M(c, ru);
  return GS_S(GS_M(dk, ln2_hi),
              GS_S(GS_S(hfsq, GS_A(GS_M(s, GS_A(hfsq, R)), GS_A(GS_M(dk, ln2_lo), cu))), f));
}

// the library path, out of line: inlined at every call site it doubled the
// hot loops' code (instruction-cache misses)
#ifdef __CUDACC__
__device__ __noinline__ double log1p_lib(double x) { return ::log1p(x); }
#endif

GS_HD double log1p_fast(double x) {
  if (x >= 0.0 && x < 0x1p1000) return log1p_pos_core(x);
#ifdef __CUDA_ARCH__
  return log1p_lib(x);
#else
  return std::log1p(x);
#endif
}

}  // namespace gs
