// Third-party code notice: the algorithms below are ports of GNU C Library (glibc) 2.39
// libm routines (sysdeps/ieee754/dbl-64: s_log1p.c, s_sin.c, e_exp.c, s_erf.c), and the
// tables in glibc_tables.h are data extracted from glibc's libm.so.6.  glibc is licensed
// under the GNU Lesser General Public License v2.1 or later; these files are
// distributed under the same terms (LGPL-2.1-or-later, see
// https://www.gnu.org/licenses/old-licenses/lgpl-2.1.html).  Copyright (C) the Free
// Software Foundation, Inc. and the glibc contributors.
//
// glibc-2.39-faithful double-precision log1p / sin / cos, host+device.
//
// Why: the reference draws normals in `boxmuller_block` (sobench/_kernels.py:178-190)
// with numba's math.log1p/sin/cos, which call the host glibc.  On FMA+AVX2 hosts
// glibc dispatches (IFUNC) to variants compiled with -mfma, so a bit-exact port
// must reproduce both the algorithm (sysdeps/ieee754/dbl-64/s_log1p.c, s_sin.c)
// and exactly where GCC contracted a*b+c into one FMA.  The FMA placement below
// was read off the disassembly of libm.so.6 (glibc 2.39-0ubuntu8.5):
//   __log1p_fma @0x7aff0, __sin_fma @0x7b2d0, __cos_fma @0x7bad0.
// Every fused operation is an explicit fma(); everything else must be compiled
// WITHOUT contraction (gcc -ffp-contract=off, nvcc -fmad=false), so the same
// source is bit-identical on the CPU test harness and on sm_100a.
//
// Domain: log1p over all finite x > -1 (plus the x <= -1 specials);
// sin/cos over |x| < 105414350 (glibc's reduce_sincos range).  Box-Muller only
// ever evaluates sin/cos on [0, 2*pi).  Larger |x| (glibc __branred) returns NaN.
#pragma once
#include <stdint.h>
#include <math.h>
#include <string.h>
#if !defined(__cplusplus)
#include <stdbool.h>
#endif

#if defined(__CUDACC__)
#define SIMOPT_HD __host__ __device__ __forceinline__
#else
#define SIMOPT_HD static inline
#endif

SIMOPT_HD uint64_t gm_bits(double x) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u; memcpy(&u, &x, 8); return u;
#endif
}
SIMOPT_HD double gm_from_bits(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double x; memcpy(&x, &u, 8); return x;
#endif
}
SIMOPT_HD int32_t gm_hi(double x) { return (int32_t)(gm_bits(x) >> 32); }
SIMOPT_HD uint32_t gm_lo(double x) { return (uint32_t)gm_bits(x); }
SIMOPT_HD double gm_set_hi(double x, int32_t hi) {
  return gm_from_bits(((uint64_t)(uint32_t)hi << 32) | (gm_bits(x) & 0xffffffffULL));
}
SIMOPT_HD double gm_fma(double a, double b, double c) { return fma(a, b, c); }
SIMOPT_HD double gm_abs(double x) { return gm_from_bits(gm_bits(x) & 0x7fffffffffffffffULL); }
SIMOPT_HD double gm_copysign(double x, double s) {
  return gm_from_bits((gm_bits(x) & 0x7fffffffffffffffULL) | (gm_bits(s) & 0x8000000000000000ULL));
}

#define GM_LN2_HI_V 0x1.62e42fee00000p-1
#define GM_LN2_LO_V 0x1.a39ef35793c76p-33
#define GM_LP1_V 0x1.5555555555593p-1
#define GM_LP2_V 0x1.999999997fa04p-2
#define GM_LP3_V 0x1.2492494229359p-2
#define GM_LP4_V 0x1.c71c51d8e78afp-3
#define GM_LP5_V 0x1.7466496cb03dep-3
#define GM_LP6_V 0x1.39a09d078c69fp-3
#define GM_LP7_V 0x1.2f112df3e5244p-3
#define GM_SN3_V -0x1.5555555555515p-3
#define GM_SN5_V 0x1.11110e829872fp-7
#define GM_CS2_V 0x1.0000000000000p-1
#define GM_CS4_V -0x1.5555555555535p-5
#define GM_CS6_V 0x1.6c16bedd9e239p-10
#define GM_S1_V -0x1.5555555555555p-3
#define GM_S2_V 0x1.1111111110ecep-7
#define GM_S3_V -0x1.a01a019db08b8p-13
#define GM_S4_V 0x1.71de27b9a7ed9p-19
#define GM_S5_V -0x1.addffc2fcdf59p-26
#define GM_BIG_V 0x1.8p45
#define GM_HP0_V 0x1.921fb54442d18p0
#define GM_HP1_V 0x1.1a62633145c07p-54
#define GM_MP1_V 0x1.921fb58000000p0
#define GM_MP2_V -0x1.dde973c000000p-27
#define GM_PP3_V -0x1.cb3b398000000p-55
#define GM_PP4_V -0x1.d747f23e32ed7p-83
#define GM_HPINV_V 0x1.45f306dc9c883p-1
#define GM_TOINT_V 0x1.8p52
#define GM_E_INVLN2N_V 0x1.71547652b82fep+7
#define GM_E_SHIFT_V 0x1.8p52
#define GM_E_NEGLN2HIN_V -0x1.62e42fefa0000p-8
#define GM_E_NEGLN2LON_V -0x1.cf79abc9e3b3ap-47
#define GM_E_C2_V 0x1.ffffffffffdbdp-2
#define GM_E_C3_V 0x1.555555555543cp-3
#define GM_E_C4_V 0x1.55555cf172b91p-5
#define GM_E_C5_V 0x1.1111167a4d017p-7

// Polynomial / reduction constants.  On the device they live in constant memory
// so DFMA/DADD take them as c[bank][offset] operands (a 64-bit literal would be
// re-materialised with two UMOVs at every use); on the host they are literals.
#if defined(__CUDACC__)
static __constant__ double gm_kconst[] = {
  GM_LN2_HI_V,
  GM_LN2_LO_V,
  GM_LP1_V,
  GM_LP2_V,
  GM_LP3_V,
  GM_LP4_V,
  GM_LP5_V,
  GM_LP6_V,
  GM_LP7_V,
  GM_SN3_V,
  GM_SN5_V,
  GM_CS2_V,
  GM_CS4_V,
  GM_CS6_V,
  GM_S1_V,
  GM_S2_V,
  GM_S3_V,
  GM_S4_V,
  GM_S5_V,
  GM_BIG_V,
  GM_HP0_V,
  GM_HP1_V,
  GM_MP1_V,
  GM_MP2_V,
  GM_PP3_V,
  GM_PP4_V,
  GM_HPINV_V,
  GM_TOINT_V,
  GM_E_INVLN2N_V,
  GM_E_SHIFT_V,
  GM_E_NEGLN2HIN_V,
  GM_E_NEGLN2LON_V,
  GM_E_C2_V,
  GM_E_C3_V,
  GM_E_C4_V,
  GM_E_C5_V,
};
#endif
static const double gm_kconst_host[] = {
  GM_LN2_HI_V,
  GM_LN2_LO_V,
  GM_LP1_V,
  GM_LP2_V,
  GM_LP3_V,
  GM_LP4_V,
  GM_LP5_V,
  GM_LP6_V,
  GM_LP7_V,
  GM_SN3_V,
  GM_SN5_V,
  GM_CS2_V,
  GM_CS4_V,
  GM_CS6_V,
  GM_S1_V,
  GM_S2_V,
  GM_S3_V,
  GM_S4_V,
  GM_S5_V,
  GM_BIG_V,
  GM_HP0_V,
  GM_HP1_V,
  GM_MP1_V,
  GM_MP2_V,
  GM_PP3_V,
  GM_PP4_V,
  GM_HPINV_V,
  GM_TOINT_V,
  GM_E_INVLN2N_V,
  GM_E_SHIFT_V,
  GM_E_NEGLN2HIN_V,
  GM_E_NEGLN2LON_V,
  GM_E_C2_V,
  GM_E_C3_V,
  GM_E_C4_V,
  GM_E_C5_V,
};
#if defined(__CUDA_ARCH__)
#define GM_K(i) gm_kconst[i]
#else
#define GM_K(i) gm_kconst_host[i]
#endif
#define GM_LN2_HI GM_K(0)
#define GM_LN2_LO GM_K(1)
#define GM_LP1 GM_K(2)
#define GM_LP2 GM_K(3)
#define GM_LP3 GM_K(4)
#define GM_LP4 GM_K(5)
#define GM_LP5 GM_K(6)
#define GM_LP6 GM_K(7)
#define GM_LP7 GM_K(8)
#define GM_SN3 GM_K(9)
#define GM_SN5 GM_K(10)
#define GM_CS2 GM_K(11)
#define GM_CS4 GM_K(12)
#define GM_CS6 GM_K(13)
#define GM_S1 GM_K(14)
#define GM_S2 GM_K(15)
#define GM_S3 GM_K(16)
#define GM_S4 GM_K(17)
#define GM_S5 GM_K(18)
#define GM_BIG GM_K(19)
#define GM_HP0 GM_K(20)
#define GM_HP1 GM_K(21)
#define GM_MP1 GM_K(22)
#define GM_MP2 GM_K(23)
#define GM_PP3 GM_K(24)
#define GM_PP4 GM_K(25)
#define GM_HPINV GM_K(26)
#define GM_TOINT GM_K(27)
#define GM_E_INVLN2N GM_K(28)
#define GM_E_SHIFT GM_K(29)
#define GM_E_NEGLN2HIN GM_K(30)
#define GM_E_NEGLN2LON GM_K(31)
#define GM_E_C2 GM_K(32)
#define GM_E_C3 GM_K(33)
#define GM_E_C4 GM_K(34)
#define GM_E_C5 GM_K(35)


// ---------------------------------------------------------------------------
// log1p  (fdlibm algorithm as shipped in glibc s_log1p.c, FMA variant)
// ---------------------------------------------------------------------------

SIMOPT_HD double glibc_log1p(double x) {
  const int32_t hx = gm_hi(x);
  const int32_t ax = hx & 0x7fffffff;
  double f, c = 0.0, u;
  int32_t k, hu;
  if (hx < 0x3FDA827A) {                    // x < 0.41422
    if (ax >= 0x3ff00000) {                 // x <= -1.0
      if (x == -1.0) return -INFINITY;
      return NAN;
    }
    if (ax < 0x3e200000) {                  // |x| < 2**-29
      if (ax < 0x3c900000) return x;        // |x| < 2**-54
      return gm_fma(-(x * x), 0.5, x);      // x - x*x*0.5  (7b2c0)
    }
    // asm 7b02e: k=0 iff (uint32)(hx + 0x402d413c) > 0x402d413c
    if ((uint32_t)hx + 0x402d413cu > 0x402d413cu) {
      k = 0; f = x; hu = 1;
      goto poly;
    }
  } else if (hx >= 0x7ff00000) {
    return x + x;
  }
  // k != 0 branch
  if (hx < 0x43400000) {
    u = 1.0 + x;
    hu = gm_hi(u);
    k = (hu >> 20) - 1023;
    c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);
    c = c / u;
  } else {
    u = x;
    hu = gm_hi(u);
    k = (hu >> 20) - 1023;
    c = 0.0;
  }
  hu &= 0x000fffff;
  if (hu < 0x6a09e) {
    u = gm_set_hi(u, hu | 0x3ff00000);
  } else {
    k += 1;
    u = gm_set_hi(u, hu | 0x3fe00000);
    hu = (0x00100000 - hu) >> 2;
  }
  f = u - 1.0;
poly: {
    const double hfsq = (f * 0.5) * f;
    if (hu == 0) {                          // |f| < 2**-20
      if (f == 0.0) {
        if (k == 0) return 0.0;
        const double kd = (double)k;
        c = gm_fma(kd, GM_LN2_LO, c);
        return gm_fma(kd, GM_LN2_HI, c);
      }
      const double R = gm_fma(-f, 0x1.5555555555555p-1, 1.0) * hfsq;
      if (k == 0) return f - R;
      const double kd = (double)k;
      return gm_fma(kd, GM_LN2_HI, -((R - gm_fma(kd, GM_LN2_LO, c)) - f));
    }
    const double s = f / (f + 2.0);
    const double z = s * s;
    const double R2 = gm_fma(z, GM_LP3, GM_LP2);
    const double R3 = gm_fma(z, GM_LP5, GM_LP4);
    const double R4 = gm_fma(z, GM_LP7, GM_LP6);
    const double z2 = z * z;
    const double z4 = z2 * z2;
    const double z6 = z2 * z4;
    double R = gm_fma(z, GM_LP1, z2 * R2);
    R = gm_fma(z4, R3, R);
    R = gm_fma(z6, R4, R);
    const double shr = s * (R + hfsq);
    if (k == 0) return f - (hfsq - shr);
    const double kd = (double)k;
    const double t = (hfsq - (gm_fma(kd, GM_LN2_LO, c) + shr)) - f;
    return gm_fma(kd, GM_LN2_HI, -t);
  }
}

// ---------------------------------------------------------------------------
// sin / cos  (IBM accurate library as refactored in glibc s_sin.c, FMA variant)
// `tab` points at the 440 doubles of __sincostab (global, constant or shared).
// ---------------------------------------------------------------------------

// TAYLOR_SIN(xx, a, da) (asm 7b950 / 7c0d0)
SIMOPT_HD double gm_taylor_sin(double a, double da) {
  const double xx = a * a;
  double p = gm_fma(GM_S5, xx, GM_S4);
  p = gm_fma(p, xx, GM_S3);
  p = gm_fma(p, xx, GM_S2);
  p = gm_fma(p, xx, GM_S1);
  const double t = gm_fma(xx, gm_fma(p, a, -(0.5 * da)), da);
  return a + t;
}

// do_sin(x, dx) (asm 7b35d..7b43d, 7b9ba..)
SIMOPT_HD double gm_do_sin(double x, double dx, const double* tab) {
  const double xold = x;
  if (gm_abs(x) < 0.126) return gm_taylor_sin(x, dx);
  if (x <= 0) dx = -dx;
  const double ux = GM_BIG + gm_abs(x);
  x = gm_abs(x) - (ux - GM_BIG);
  const int k = (int)(gm_lo(ux) << 2);
  const double xx = x * x;
  const double s = x + gm_fma(x * xx, gm_fma(xx, GM_SN5, GM_SN3), dx);
  const double c = gm_fma(x, dx, xx * gm_fma(xx, gm_fma(xx, GM_CS6, GM_CS4), GM_CS2));
  const double sn = tab[k], ssn = tab[k + 1], cs = tab[k + 2], ccs = tab[k + 3];
  double cor = gm_fma(s, ccs, ssn);
  cor = gm_fma(-c, sn, cor);
  cor = gm_fma(s, cs, cor);
  return gm_copysign(sn + cor, xold);
}

// do_cos(x, dx) (asm 7b5e0.., 7b780.., 7bb36..)
SIMOPT_HD double gm_do_cos(double x, double dx, const double* tab) {
  if (x < 0) dx = -dx;
  const double ux = GM_BIG + gm_abs(x);
  x = (gm_abs(x) - (ux - GM_BIG)) + dx;
  const int k = (int)(gm_lo(ux) << 2);
  const double xx = x * x;
  const double s = gm_fma(x * xx, gm_fma(xx, GM_SN5, GM_SN3), x);
  const double c = xx * gm_fma(xx, gm_fma(xx, GM_CS6, GM_CS4), GM_CS2);
  const double sn = tab[k], ssn = tab[k + 1], cs = tab[k + 2], ccs = tab[k + 3];
  double cor = gm_fma(-s, ssn, ccs);
  cor = gm_fma(-c, cs, cor);
  cor = gm_fma(-s, sn, cor);
  return cs + cor;
}

// reduce_sincos (asm 7b476.., 7bd53..)
SIMOPT_HD int gm_reduce_sincos(double x, double* a, double* da) {
  const double t = gm_fma(x, GM_HPINV, GM_TOINT);
  const double xn = t - GM_TOINT;
  const int n = (int)(gm_lo(t) & 3u);
  const double y = gm_fma(-xn, GM_MP2, gm_fma(-xn, GM_MP1, x));
  const double t2 = gm_fma(-xn, GM_PP3, y);
  double db = gm_fma(-xn, GM_PP3, y - t2);
  const double b = gm_fma(-xn, GM_PP4, t2);
  db = db + gm_fma(-xn, GM_PP4, t2 - b);
  *a = b;
  *da = db;
  return n;
}

SIMOPT_HD double gm_do_sincos(double a, double da, int n, const double* tab) {
  const double r = (n & 1) ? gm_do_cos(a, da, tab) : gm_do_sin(a, da, tab);
  return (n & 2) ? -r : r;
}

SIMOPT_HD double glibc_sin(double x, const double* tab) {
  const int32_t k = gm_hi(x) & 0x7fffffff;
  if (k < 0x3e500000) return x;                       // |x| < 2^-26
  if (k < 0x3feb6000) return gm_do_sin(x, 0.0, tab);  // |x| < 0.855469
  if (k < 0x400368fd) {                               // |x| < 2.426265
    const double t = GM_HP0 - gm_abs(x);
    return gm_copysign(gm_do_cos(t, GM_HP1, tab), x);
  }
  if (k < 0x419921FB) {                               // |x| < 105414350
    double a, da;
    const int n = gm_reduce_sincos(x, &a, &da);
    return gm_do_sincos(a, da, n, tab);
  }
  return NAN;  // outside the ported domain (glibc: __branred / x/x)
}

SIMOPT_HD double glibc_cos(double x, const double* tab) {
  const int32_t k = gm_hi(x) & 0x7fffffff;
  if (k < 0x3e400000) return 1.0;                     // |x| < 2^-27
  if (k < 0x3feb6000) return gm_do_cos(x, 0.0, tab);
  if (k < 0x400368fd) {
    const double y = GM_HP0 - gm_abs(x);
    const double a = y + GM_HP1;
    const double da = (y - a) + GM_HP1;
    return gm_do_sin(a, da, tab);
  }
  if (k < 0x419921FB) {
    double a, da;
    const int n = gm_reduce_sincos(x, &a, &da);
    return gm_do_sincos(a, da, n + 1, tab);
  }
  return NAN;
}

// Box-Muller pair exactly as boxmuller_block (sobench/_kernels.py:184-190):
//   r = sqrt(-2.0 * log1p(-u1)); th = TAU * u2; (r*cos(th), r*sin(th))
#define GM_TAU 6.283185307179586
SIMOPT_HD void glibc_boxmuller(double u1, double u2, const double* tab, double* z0, double* z1) {
  const double r = sqrt(-2.0 * glibc_log1p(-u1));
  const double th = GM_TAU * u2;
  *z0 = r * glibc_cos(th, tab);
  *z1 = r * glibc_sin(th, tab);
}

// ---------------------------------------------------------------------------
// exp  (glibc >= 2.28 e_exp.c, Szabolcs Nagy's table method, N = 128; FMA variant
// __exp_fma @0x79b60).  `etab` = __exp_data.tab (256 words, glibc_tables.h).
// ---------------------------------------------------------------------------


// specialcase(tmp, sbits, ki) for 512 <= |x| < 1024 (asm 79c60..79d27)
SIMOPT_HD double gm_exp_special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ULL) == 0) {
    sbits -= 1009ULL << 52;
    const double scale = gm_from_bits(sbits);
    return 0x1p1009 * gm_fma(scale, tmp, scale);   // may overflow to inf, as glibc
  }
  sbits += 1022ULL << 52;
  const double scale = gm_from_bits(sbits);
  const double st = scale * tmp;
  double y = scale + st;
  if (y < 1.0) {
    double lo = (scale - y) + st;
    const double hi = 1.0 + y;
    lo = ((1.0 - hi) + y) + lo;
    y = (lo + hi) - 1.0;
    if (y == 0.0) y = 0.0;  // avoid -0.0
  }
  return 0x1p-1022 * y;
}

SIMOPT_HD double glibc_exp(double x, const uint64_t* etab) {
  const uint64_t ix = gm_bits(x);
  uint32_t abstop = (uint32_t)((ix >> 52) & 0x7ff);
  if (abstop - 0x3c9u > 0x3eu) {                 // |x| < 2^-54 or |x| >= 512 or nan/inf
    if ((int32_t)(abstop - 0x3c9u) < 0) return 1.0 + x;
    if (abstop >= 0x409) {                       // |x| >= 1024
      if (ix == 0xfff0000000000000ULL) return 0.0;
      if (abstop == 0x7ff) return 1.0 + x;
      return (ix >> 63) ? 0.0 : INFINITY;        // __math_uflow(0) / __math_oflow(0)
    }
    abstop = 0;                                  // large |x|: handled by specialcase
  }
  const double kd0 = gm_fma(x, GM_E_INVLN2N, GM_E_SHIFT);
  const uint64_t ki = gm_bits(kd0);
  const double kd = kd0 - GM_E_SHIFT;
  double r = gm_fma(kd, GM_E_NEGLN2HIN, x);
  r = gm_fma(kd, GM_E_NEGLN2LON, r);
  const uint32_t idx = 2u * (uint32_t)(ki & 127u);
  const uint64_t top = ki << 45;
  const double tail = gm_from_bits(etab[idx]);
  const uint64_t sbits = etab[idx + 1] + top;
  const double r2 = r * r;
  const double p23 = gm_fma(r, GM_E_C3, GM_E_C2);
  const double p45 = gm_fma(r, GM_E_C5, GM_E_C4);
  double tmp = gm_fma(p23, r2, r + tail);
  tmp = gm_fma(r2 * r2, p45, tmp);
  if (abstop == 0) return gm_exp_special(tmp, sbits, ki);
  const double scale = gm_from_bits(sbits);
  return gm_fma(scale, tmp, scale);
}

// ---------------------------------------------------------------------------
// erf (glibc 2.39 s_erf.c as compiled into libm.so.6: `erf` @0x2df70, SSE2 code, no
// FMA; the two exp calls go through the exp IFUNC, i.e. __exp_fma = glibc_exp).  Every
// operation below follows the disassembly's order and operands; constants are the
// .rodata words the code loads (tools/extract_glibc_tables.py prints them).  Used by
// newsvendor_cost_block (_kernels.py:219-220) through numba's math.erf.
// ---------------------------------------------------------------------------
SIMOPT_HD double glibc_erf(double x, const uint64_t* etab) {
  const int32_t hx = gm_hi(x);
  const int32_t ix = hx & 0x7fffffff;
  if (ix > 0x7fefffff) {  // inf or NaN: (1 - 2 sign) + 1/x
    const double one = 1.0 / x;
    return (double)(1 - ((hx >> 31) & 1) * 2) + one;
  }
  if (ix <= 0x3feaffff) {  // |x| < 0.84375
    if (ix <= 0x3e2fffff) {  // |x| < 2^-28
      if ((hx & 0x7f800000) == 0)  // avoid underflow: 0.0625 * (16 x + efx8 x)
        return ((x * 16.0) + (x * 0x1.06eba8214db69p+1)) * 0.0625;
      return (x * 0x1.06eba8214db69p-3) + x;
    }
    const double z = x * x;
    const double z2 = z * z;
    double r = (z * -0x1.7a291236668e4p-8) - 0x1.d2a51dbd7194fp-6;
    r = (r * z2) + ((z * -0x1.4cd7d691cb913p-2) + 0x1.06eba8214db68p-3);
    const double z4 = z2 * z2;
    r = r + (z4 * -0x1.8ead6120016acp-16);
    double q3 = ((z * 0x1.4d022c4d36b0fp-8) + 0x1.0a54c5536cebap-4) * z2;
    const double q1 = (z * 0x1.97779cddadc09p-2) + 1.0;
    double q5 = ((z * -0x1.09c4342a26120p-18) + 0x1.15dc9221c1a10p-13) * z4;
    const double s = q5 + (q3 + q1);
    return ((r / s) * x) + x;
  }
  if (ix <= 0x3ff3ffff) {  // 0.84375 <= |x| < 1.25
    const double s = gm_abs(x) - 1.0;
    const double s2 = s * s;
    double p = ((s * 0x1.45fca805120e4p-2) - 0x1.7d240fbb8c3f1p-2) * s2;
    const double s4 = s2 * s2;
    p = p + ((s * 0x1.a8d00ad92b34dp-2) - 0x1.359b8bef77538p-9);
    const double s6 = s2 * s4;
    p = p + (((s * 0x1.22a36599795ebp-5) - 0x1.c63983d3e28ecp-4) * s4);
    p = p + (s6 * -0x1.1bf380a96073fp-9);
    double q = ((s * 0x1.2635cd99fe9a7p-4) + 0x1.14af092eb6f33p-1) * s2;
    q = q + ((s * 0x1.b3e6618eee323p-4) + 1.0);
    q = q + (((s * 0x1.bedc26b51dd1cp-7) + 0x1.02660e763351fp-3) * s4);
    q = q + (s6 * 0x1.88b545735151dp-7);
    const double pq = p / q;
    return hx >= 0 ? pq + 0x1.b0ac160000000p-1 : -0x1.b0ac160000000p-1 - pq;
  }
  if (ix > 0x4017ffff) {  // |x| >= 6
    return hx >= 0 ? 1.0 - 0x1.56e1fc2f8f359p-997 : 0x1.56e1fc2f8f359p-997 - 1.0;
  }
  const double ax = gm_abs(x);
  const double s = 1.0 / (x * x);
  const double s2 = s * s;
  const double s4 = s2 * s2;
  const double s6 = s2 * s4;
  double R, S;
  if (ix > 0x4006db6d) {  // |x| >= 1/0.35: rb / sb
    R = ((s * -0x1.4145d43c5ed98p+7) - 0x1.1c209555f995ap+4) * s2;
    R = R + ((s * -0x1.993ba70c285dep-1) - 0x1.4341239e86f4ap-7);
    R = R + (((s * -0x1.004616a2e5992p+10) - 0x1.3ec881375f228p+9) * s4);
    R = R + (s6 * -0x1.e384e9bdc383fp+8);
    double A = ((s * 0x1.802eb189d5118p+10) + 0x1.45cae221b9f0ap+8) * s2;
    A = A + ((s * 0x1.e568b261d5190p+4) + 1.0);
    const double B = ((s * 0x1.3f219cedf3be6p+11) + 0x1.8ffb7688c246ap+11) * s4;
    const double C = ((s * -0x1.670e242712d62p+4) + 0x1.da874e79fe763p+8) * s6;
    S = (B + A) + C;
  } else {  // 1.25 <= |x| < 1/0.35: ra / sa
    R = ((s * -0x1.f300ae4cba38dp+5) - 0x1.51e0441b0e726p+3) * s2;
    R = R + ((s * -0x1.63416e4ba7360p-1) - 0x1.43412600d6435p-7);
    R = R + (((s * -0x1.7135cebccabb2p+7) - 0x1.44cb184282266p+7) * s4);
    R = R + (((s * -0x1.3a0efc69ac25cp+3) - 0x1.4526557e4d2f2p+6) * s6);
    double A = ((s * 0x1.b290dd58a1a71p+8) + 0x1.1350c526ae721p+7) * s2;
    A = A + ((s * 0x1.3a6b9bd707687p+4) + 1.0);
    const double B = ((s * 0x1.ad02157700314p+8) + 0x1.42b1921ec2868p+9) * s4;
    const double C = ((s * 0x1.a47ef8e484a93p+2) + 0x1.b28a3ee48ae2cp+6) * s6;
    const double s8 = s4 * s4;
    S = (C + (A + B)) + (s8 * -0x1.eeff2ee749a62p-5);
  }
  const double z = gm_from_bits(gm_bits(ax) & 0xffffffff00000000ULL);
  const double e1 = glibc_exp(((-z) * z) - 0.5625, etab);
  const double rs = R / S;
  const double e2 = glibc_exp(((z - ax) * (z + ax)) + rs, etab);
  const double r = e2 * e1;
  return hx >= 0 ? 1.0 - (r / ax) : (r / ax) - 1.0;
}

// Stable logistic as sigmoid_block (sobench/_kernels.py:159-169).
SIMOPT_HD double glibc_sigmoid(double t, const uint64_t* etab) {
  if (t >= 0.0) {
    const double e = glibc_exp(-t, etab);
    return 1.0 / (1.0 + e);
  }
  const double e = glibc_exp(t, etab);
  return e / (1.0 + e);
}

// logistic_loss_block (sobench/_kernels.py:193-201), one sample.
SIMOPT_HD double glibc_logistic_loss_term(double t, double z, const uint64_t* etab) {
  if (t >= 0.0) return glibc_log1p(glibc_exp(-t, etab)) + (1.0 - z) * t;
  return glibc_log1p(glibc_exp(t, etab)) - z * t;
}

// ---------------------------------------------------------------------------
// Divergence-free Box-Muller for the device: the same glibc arithmetic as
// glibc_boxmuller(), restructured so that every lane of a warp executes one
// instruction stream.  sin and cos of theta in [0, 2pi) always need exactly one
// do_sin-type and one do_cos-type evaluation (glibc s_sin.c, per region):
//   theta < 0.855469 : sin = do_sin(x,0)          cos = do_cos(x,0)
//   theta < 2.426265 : sin = do_cos(y,hp1)        cos = do_sin(y+hp1, (y-a)+hp1),  y = hp0-x
//   otherwise        : (a,da,n) = reduce_sincos(x); sin/cos pick do_sin/do_cos(a,da) by n
// Region arguments are selected, both evaluations run unconditionally, and the
// Taylor branch of do_sin (|a| < 0.126) is evaluated and selected.  log1p's two
// prologues (k = 0 / k != 0) are likewise both computed and selected.
// Bit-identity with glibc_boxmuller() is checked on the CPU (tools/) and on the GPU.
// ---------------------------------------------------------------------------
SIMOPT_HD double gm_do_sin_nb(double x, double dx, const double* tab) {
  const double xold = x;
  const double ax = gm_abs(x);
  const double tay = gm_taylor_sin(x, dx);
  const double dxs = (x <= 0) ? -dx : dx;
  const double ux = GM_BIG + ax;
  const double xr = ax - (ux - GM_BIG);
  const int k = (int)(gm_lo(ux) << 2);
  const double xx = xr * xr;
  const double s = xr + gm_fma(xr * xx, gm_fma(xx, GM_SN5, GM_SN3), dxs);
  const double c = gm_fma(xr, dxs, xx * gm_fma(xx, gm_fma(xx, GM_CS6, GM_CS4), GM_CS2));
  const double sn = tab[k], ssn = tab[k + 1], cs = tab[k + 2], ccs = tab[k + 3];
  double cor = gm_fma(s, ccs, ssn);
  cor = gm_fma(-c, sn, cor);
  cor = gm_fma(s, cs, cor);
  const double big = gm_copysign(sn + cor, xold);
  return (ax < 0.126) ? tay : big;
}

SIMOPT_HD void glibc_sincos_pos(double x, const double* tab, double* sin_out, double* cos_out) {
  // x >= 0, x < 105414350 (Box-Muller theta)
  const int32_t kx = gm_hi(x) & 0x7fffffff;
  const bool r2 = kx < 0x3feb6000;
  const bool r3 = !r2 && kx < 0x400368fd;
  // region 3 arguments
  const double y = GM_HP0 - x;
  const double a3 = y + GM_HP1;
  const double da3 = (y - a3) + GM_HP1;
  // region 4 arguments
  double a4, da4;
  const int n = gm_reduce_sincos(x, &a4, &da4);
  const double as = r2 ? x : (r3 ? a3 : a4);
  const double das = r2 ? 0.0 : (r3 ? da3 : da4);
  const double ac = r2 ? x : (r3 ? y : a4);
  const double dac = r2 ? 0.0 : (r3 ? GM_HP1 : da4);
  const double S = gm_do_sin_nb(as, das, tab);
  const double C = gm_do_cos(ac, dac, tab);
  double sv, cv;
  if (r2) {
    sv = S;
    cv = C;
  } else if (r3) {
    sv = gm_copysign(C, x);
    cv = S;
  } else {
    const double s4 = (n & 1) ? C : S;
    sv = (n & 2) ? -s4 : s4;
    const int m = n + 1;
    const double c4 = (m & 1) ? C : S;
    cv = (m & 2) ? -c4 : c4;
  }
  if (kx < 0x3e500000) sv = x;
  if (kx < 0x3e400000) cv = 1.0;
  *sin_out = sv;
  *cos_out = cv;
}

// log1p for x in (-1, 0] (Box-Muller's -u1) with both prologues computed.
SIMOPT_HD double glibc_log1p_neg(double x) {
  const int32_t hx = gm_hi(x);
  const int32_t ax = hx & 0x7fffffff;
  if (ax < 0x3e200000) {                   // |x| < 2**-29 (rare)
    if (ax < 0x3c900000) return x;
    return gm_fma(-(x * x), 0.5, x);
  }
  const bool k0 = (uint32_t)hx + 0x402d413cu > 0x402d413cu;
  // k != 0 prologue (x <= -0.2929): u = 1 + x in (0, 0.71]; k <= 0 so c = x - (u - 1)
  double u = 1.0 + x;
  int32_t hu = gm_hi(u);
  int32_t k = (hu >> 20) - 1023;
  double c = (x - (u - 1.0)) / u;
  hu &= 0x000fffff;
  if (hu < 0x6a09e) {
    u = gm_set_hi(u, hu | 0x3ff00000);
  } else {
    k += 1;
    u = gm_set_hi(u, hu | 0x3fe00000);
    hu = (0x00100000 - hu) >> 2;
  }
  double f = u - 1.0;
  if (k0) { k = 0; f = x; hu = 1; c = 0.0; }
  const double hfsq = (f * 0.5) * f;
  if (hu == 0) {                           // |f| < 2**-20 (rare)
    if (f == 0.0) {
      if (k == 0) return 0.0;
      const double kd = (double)k;
      return gm_fma(kd, GM_LN2_HI, gm_fma(kd, GM_LN2_LO, c));
    }
    const double R = gm_fma(-f, 0x1.5555555555555p-1, 1.0) * hfsq;
    if (k == 0) return f - R;
    const double kd = (double)k;
    return gm_fma(kd, GM_LN2_HI, -((R - gm_fma(kd, GM_LN2_LO, c)) - f));
  }
  const double s = f / (f + 2.0);
  const double z = s * s;
  const double R2 = gm_fma(z, GM_LP3, GM_LP2);
  const double R3 = gm_fma(z, GM_LP5, GM_LP4);
  const double R4 = gm_fma(z, GM_LP7, GM_LP6);
  const double z2 = z * z;
  const double z4 = z2 * z2;
  const double z6 = z2 * z4;
  double R = gm_fma(z, GM_LP1, z2 * R2);
  R = gm_fma(z4, R3, R);
  R = gm_fma(z6, R4, R);
  const double shr = s * (R + hfsq);
  const double kd = (double)k;
  const double tk = (hfsq - (gm_fma(kd, GM_LN2_LO, c) + shr)) - f;
  return k0 ? f - (hfsq - shr) : gm_fma(kd, GM_LN2_HI, -tk);
}

SIMOPT_HD void glibc_boxmuller_fast(double u1, double u2, const double* tab, double* z0,
                                    double* z1) {
  const double r = sqrt(-2.0 * glibc_log1p_neg(-u1));
  const double th = GM_TAU * u2;
  double sv, cv;
  glibc_sincos_pos(th, tab, &sv, &cv);
  *z0 = r * cv;
  *z1 = r * sv;
}
