/* Bit-exact restatements of the two libm routines the reference's numba
 * kernels call, usable from host C (gcc -ffp-contract=off) and from CUDA
 * device code (nvcc -fmad=false):
 *
 *   ucp_exp  == glibc 2.39 x86_64 `exp` as resolved by its IFUNC on an
 *               FMA3+AVX2 host (`__exp_fma`): the table-driven algorithm of
 *               sysdeps/ieee754/dbl-64/e_exp.c with GCC's FMA contraction
 *               pattern (8 FMA + 1 sub + 1 add + 2 mul on the main path),
 *               recovered from `objdump -d libm.so.6`.
 *   ucp_erf  == glibc `erf` (fdlibm s_erf.c, generic x86_64 build: no FMA),
 *               which calls the IFUNC exp above.
 *
 * Where the reference calls them: kernels.py:413,427,428,473 (np.exp inside
 * @njit -> llvm.exp -> glibc exp) and kernels.py:404 (math.erf -> glibc erf).
 *
 * Every multiply/add below must be evaluated exactly as written -- the host
 * build uses -ffp-contract=off and the device build -fmad=false; fused
 * operations are spelled explicitly with UCP_FMA.
 */
#pragma once
#include <stdint.h>
#include "ucp_exp_data.h"

#if defined(__CUDACC__)
#define UCP_HD __host__ __device__ __forceinline__
#else
#include <math.h>
#include <string.h>
#define UCP_HD static inline
#endif

UCP_HD uint64_t ucp_asu64(double x) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u;
  memcpy(&u, &x, 8);
  return u;
#endif
}

UCP_HD double ucp_asf64(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double x;
  memcpy(&x, &u, 8);
  return x;
#endif
}

UCP_HD double ucp_fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return fma(a, b, c);
#endif
}
#define UCP_FMA ucp_fma

/* Rare path of exp for |x| in [512, 1024) (glibc `specialcase`).  Never
 * reached by the Witsenhausen kernels (|arguments| <= 72) but kept so the
 * port is total. */
UCP_HD double ucp_exp_special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ull) == 0) {
    sbits -= 1009ull << 52;
    double scale = ucp_asf64(sbits);
    double y = UCP_FMA(scale, tmp, scale);
    return y * ucp_asf64(0x7f00000000000000ull); /* 0x1p1009 */
  }
  sbits += 1022ull << 52;
  double scale = ucp_asf64(sbits);
  double st = scale * tmp; /* not fused: the product is reused below */
  double y = scale + st;
  if (y < 1.0) {
    double lo = (scale - y) + st;
    double hi = 1.0 + y;
    lo = ((1.0 - hi) + y) + lo;
    y = (hi + lo) - 1.0;
    if (y == 0.0) y = 0.0;
  }
  return ucp_asf64(0x0010000000000000ull) * y; /* 0x1p-1022 */
}

/* glibc exp with an explicit table pointer (global, constant or shared). */
UCP_HD double ucp_exp_tab(double x, const uint64_t* tab) {
  uint64_t ix = ucp_asu64(x);
  uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ffu;
  if (abstop - 0x3c9u >= 0x3fu) {
    if ((int32_t)(abstop - 0x3c9u) < 0) return 1.0 + x; /* |x| < 2^-54 */
    if (abstop >= 0x409u) {                               /* |x| >= 1024 */
      if (ix == 0xfff0000000000000ull) return 0.0;
      if (abstop >= 0x7ffu) return 1.0 + x;
      if (ix >> 63) return 0.0;                         /* __math_uflow */
      return ucp_asf64(0x7ff0000000000000ull);          /* __math_oflow */
    }
    abstop = 0; /* large |x|: handled by ucp_exp_special */
  }
  double kd = UCP_FMA(x, ucp_asf64(UCP_EXP_INVLN2N), ucp_asf64(UCP_EXP_SHIFT));
  uint64_t ki = ucp_asu64(kd);
  kd = kd - ucp_asf64(UCP_EXP_SHIFT);
  double r = UCP_FMA(kd, ucp_asf64(UCP_EXP_NEGLN2HIN), x);
  r = UCP_FMA(kd, ucp_asf64(UCP_EXP_NEGLN2LON), r);
  uint64_t idx = 2u * (ki & 127u);
  uint64_t top = ki << 45;
  double tail = ucp_asf64(tab[idx]);
  uint64_t sbits = tab[idx + 1] + top;
  double p23 = UCP_FMA(r, ucp_asf64(UCP_EXP_C3), ucp_asf64(UCP_EXP_C2));
  double tr = r + tail;
  double r2 = r * r;
  double p45 = UCP_FMA(r, ucp_asf64(UCP_EXP_C5), ucp_asf64(UCP_EXP_C4));
  double t1 = UCP_FMA(p23, r2, tr);
  double r4 = r2 * r2;
  double tmp = UCP_FMA(r4, p45, t1);
  if (abstop == 0) return ucp_exp_special(tmp, sbits, ki);
  double scale = ucp_asf64(sbits);
  return UCP_FMA(scale, tmp, scale);
}

/* Main path of ucp_exp_tab only, for |x| < 512 (every exp argument of the
 * Witsenhausen kernels lies in [-72.1, 0]).  Bitwise identical to
 * ucp_exp_tab there: for |x| < 2^-54 the main path yields fma(1, x, 1) ==
 * 1.0 + x, the value of glibc's tiny-argument branch (kd = 0, r = x, tmp = x).
 * `tab2[i]` = {tail bits, scale bits} of entry i, so one 128-bit load fetches
 * both (LDS.128 from shared memory). */
typedef struct { uint64_t tail, sbits; } ucp_exp_entry;

UCP_HD double ucp_exp_core(double x, const ucp_exp_entry* tab2) {
  double kd = UCP_FMA(x, ucp_asf64(UCP_EXP_INVLN2N), ucp_asf64(UCP_EXP_SHIFT));
  uint64_t ki = ucp_asu64(kd);
  kd = kd - ucp_asf64(UCP_EXP_SHIFT);
  double r = UCP_FMA(kd, ucp_asf64(UCP_EXP_NEGLN2HIN), x);
  r = UCP_FMA(kd, ucp_asf64(UCP_EXP_NEGLN2LON), r);
  ucp_exp_entry e = tab2[ki & 127u];
  double tail = ucp_asf64(e.tail);
  uint64_t sbits = e.sbits + (ki << 45);
  double p23 = UCP_FMA(r, ucp_asf64(UCP_EXP_C3), ucp_asf64(UCP_EXP_C2));
  double tr = r + tail;
  double r2 = r * r;
  double p45 = UCP_FMA(r, ucp_asf64(UCP_EXP_C5), ucp_asf64(UCP_EXP_C4));
  double t1 = UCP_FMA(p23, r2, tr);
  double r4 = r2 * r2;
  double tmp = UCP_FMA(r4, p45, t1);
  double scale = ucp_asf64(sbits);
  return UCP_FMA(scale, tmp, scale);
}

/* fdlibm erf coefficients (bit patterns of glibc's s_erf.c constants). */
#define UCP_D(u) ucp_asf64(u##ull)

/* glibc erf; `tab` is forwarded to the two exp calls of the |x|>=1.25 branch. */
UCP_HD double ucp_erf_tab(double x, const uint64_t* tab) {
  uint64_t ux = ucp_asu64(x);
  int32_t hx = (int32_t)(ux >> 32);
  int32_t ix = hx & 0x7fffffff;
  if (ix >= 0x7ff00000) { /* erf(nan)=nan, erf(+-inf)=+-1 */
    int32_t i = (int32_t)(((uint32_t)hx >> 31) << 1);
    return (double)(1 - i) + 1.0 / x;
  }
  if (ix < 0x3feb0000) { /* |x| < 0.84375 */
    if (ix < 0x3e300000) { /* |x| < 2^-28 */
      if (ix < 0x00800000) {
        return 0.0625 * (16.0 * x + UCP_D(0x40006eba8214db69) * x);
      }
      return x + UCP_D(0x3fc06eba8214db69) * x; /* x + efx*x */
    }
    double z = x * x;
    double r1 = UCP_D(0x3fc06eba8214db68) + z * UCP_D(0xbfd4cd7d691cb913);
    double z2 = z * z;
    double r2 = UCP_D(0xbf9d2a51dbd7194f) + z * UCP_D(0xbf77a291236668e4);
    double z4 = z2 * z2;
    double s1 = 1.0 + z * UCP_D(0x3fd97779cddadc09);
    double s2 = UCP_D(0x3fb0a54c5536ceba) + z * UCP_D(0x3f74d022c4d36b0f);
    double s3 = UCP_D(0x3f215dc9221c1a10) + z * UCP_D(0xbed09c4342a26120);
    double r = (r1 + z2 * r2) + z4 * UCP_D(0xbef8ead6120016ac);
    double s = (s1 + z2 * s2) + z4 * s3;
    double y = r / s;
    return x + x * y;
  }
  if (ix < 0x3ff40000) { /* 0.84375 <= |x| < 1.25 */
    double s = fabs(x) - 1.0;
    double P1 = UCP_D(0xbf6359b8bef77538) + s * UCP_D(0x3fda8d00ad92b34d);
    double ss2 = s * s;
    double Q1 = 1.0 + s * UCP_D(0x3fbb3e6618eee323);
    double ss4 = ss2 * ss2;
    double P2 = UCP_D(0xbfd7d240fbb8c3f1) + s * UCP_D(0x3fd45fca805120e4);
    double ss6 = ss4 * ss2;
    double Q2 = UCP_D(0x3fe14af092eb6f33) + s * UCP_D(0x3fb2635cd99fe9a7);
    double P3 = UCP_D(0xbfbc63983d3e28ec) + s * UCP_D(0x3fa22a36599795eb);
    double Q3 = UCP_D(0x3fc02660e763351f) + s * UCP_D(0x3f8bedc26b51dd1c);
    double P4 = UCP_D(0xbf61bf380a96073f);
    double Q4 = UCP_D(0x3f888b545735151d);
    double P = ((P1 + ss2 * P2) + ss4 * P3) + ss6 * P4;
    double Q = ((Q1 + ss2 * Q2) + ss4 * Q3) + ss6 * Q4;
    const double erx = UCP_D(0x3feb0ac160000000);
    if (hx >= 0) return erx + P / Q;
    return -erx - P / Q;
  }
  if (ix >= 0x40180000) { /* |x| >= 6 */
    const double tiny = 1e-300;
    if (hx >= 0) return 1.0 - tiny;
    return tiny - 1.0;
  }
  double ax = fabs(x);
  double s = 1.0 / (x * x);
  double R, S;
  double ss2 = s * s;
  double ss4 = ss2 * ss2;
  double ss6 = ss4 * ss2;
  if (ix < 0x4006db6e) { /* |x| < 1/0.35 */
    double R1 = UCP_D(0xbf843412600d6435) + s * UCP_D(0xbfe63416e4ba7360);
    double S1 = 1.0 + s * UCP_D(0x4033a6b9bd707687);
    double R2 = UCP_D(0xc0251e0441b0e726) + s * UCP_D(0xc04f300ae4cba38d);
    double S2 = UCP_D(0x4061350c526ae721) + s * UCP_D(0x407b290dd58a1a71);
    double ss8 = ss4 * ss4;
    double R3 = UCP_D(0xc0644cb184282266) + s * UCP_D(0xc067135cebccabb2);
    double S3 = UCP_D(0x40842b1921ec2868) + s * UCP_D(0x407ad02157700314);
    double R4 = UCP_D(0xc054526557e4d2f2) + s * UCP_D(0xc023a0efc69ac25c);
    double S4 = UCP_D(0x405b28a3ee48ae2c) + s * UCP_D(0x401a47ef8e484a93);
    R = ((R1 + ss2 * R2) + ss4 * R3) + ss6 * R4;
    S = (((S1 + ss2 * S2) + ss4 * S3) + ss6 * S4) + ss8 * UCP_D(0xbfaeeff2ee749a62);
  } else { /* |x| >= 1/0.35 */
    double R1 = UCP_D(0xbf84341239e86f4a) + s * UCP_D(0xbfe993ba70c285de);
    double S1 = 1.0 + s * UCP_D(0x403e568b261d5190);
    double R2 = UCP_D(0xc031c209555f995a) + s * UCP_D(0xc064145d43c5ed98);
    double S2 = UCP_D(0x40745cae221b9f0a) + s * UCP_D(0x409802eb189d5118);
    double R3 = UCP_D(0xc083ec881375f228) + s * UCP_D(0xc09004616a2e5992);
    double S3 = UCP_D(0x40a8ffb7688c246a) + s * UCP_D(0x40a3f219cedf3be6);
    double S4 = UCP_D(0x407da874e79fe763) + s * UCP_D(0xc03670e242712d62);
    R = ((R1 + ss2 * R2) + ss4 * R3) + ss6 * UCP_D(0xc07e384e9bdc383f);
    S = ((S1 + ss2 * S2) + ss4 * S3) + ss6 * S4;
  }
  double z = ucp_asf64(ucp_asu64(ax) & 0xffffffff00000000ull);
  double e1 = ucp_exp_tab((-z) * z - 0.5625, tab);
  double e2 = ucp_exp_tab((z - ax) * (z + ax) + R / S, tab);
  double r = e1 * e2;
  if (hx >= 0) return 1.0 - r / ax;
  return r / ax - 1.0;
}

#define UCP_INV_SQRT_2PI_BITS 0x3fd9884533d43651ull /* 1/np.sqrt(2*pi) */
#define UCP_INV_SQRT_2_BITS 0x3fe6a09e667f3bccull   /* 1/np.sqrt(2) */

/* Gaussian cdf with the reference's hard cut at |z| >= GAUSS_CUT = 12
 * (kernels.py:398-404, numpy twin :235-240). */
UCP_HD double ucp_phi_cdf_tab(double z, const uint64_t* tab) {
  if (z <= -12.0) return 0.0;
  if (z >= 12.0) return 1.0;
  return 0.5 * (1.0 + ucp_erf_tab(z * ucp_asf64(UCP_INV_SQRT_2_BITS), tab));
}

