// Newsvendor device helpers shared by newsvendor.cu and the C ABI.
//
// Epoch layout ("keyed ECDF"): every demand draw of the epoch is stored as one
// 32-bit key  q << 12 | local,  where local (12 bits) is the draw's position in
// its 4096-draw segment and q (20 bits) is a fixed-point code of an fp32
// approximation z~ of its standard normal z:
//     q = clamp(floor((z~ + 9.5) * 2^20 / 19), 0, 2^20 - 1).
// |z~ - z| <= NV_EPSZ is guaranteed by construction (error budget at
// nv_approx_pair; NV_EPSZ is > 7x the measured worst case and tests/test_gpu_newsvendor.py
// measures the maximum over 2^26 draws), and q is
// monotone in z~ up to one code of fp32 rounding.  Keys are counting-sorted by
// bucket (the top 10 bits of q) inside each segment.  An ECDF query x_j then
// splits every draw into: certainly below x, certainly above x, or ambiguous
// (|z - t| within NV_EPSZ + rounding slack, t = (x - mu)/sigma); only the few
// ambiguous draws are recomputed exactly (Philox + glibc-exact Box-Muller) and
// compared as the reference does, D = mu + sigma*z <= x.  The count is therefore
// the reference's count exactly, while an epoch writes 4 B per draw and never
// evaluates the exact transcendentals for the bulk of the draws.
#pragma once
#include <stdint.h>

#include "../../include/simopt_b200.h"
#include "glibc_math.cuh"
#include "glibc_tables.h"
#include "philox.cuh"
#include "rng_device.cuh"

#define NV_SEG 4096       // draws per segment (12-bit local index)
#define NV_B 1024         // buckets per segment (top 10 bits of q)
#define NV_QBITS 20
#define NV_QMAX ((1 << NV_QBITS) - 1)
#define NV_Z0 9.5
#define NV_QSCALE (1048576.0 / 19.0)  // codes per unit of z
#define NV_W (19.0 / 1048576.0)       // z width of one code
#define NV_EPSZ 1.5e-5                // guaranteed |z~ - z| bound (analytic worst case < 1.1e-5,
                                      // measured max 2.1e-6 over 2^26 draws)

// fp32 approximation of one Box-Muller pair (both components) from the raw
// Philox words, on the SFU (MUFU) path.  Error budget, |z~ - z|:
//   l = log1p(-u1): u1 < 2^-6: 5-term series -(u + u^2/2 + ... + u^5/5) (relative
//       error < 2^-29 + fp32 rounding); else ln2 * lg2.approx((float)(1 - u1)) with
//       1 - u1 an exact integer times 2^-53 (the __logf bound: abs error <= 3.6e-7 on
//       [0.5, 2], 3 ulp relative below; the ftz forms never see subnormals here):
//       |dr| = |dl| / r <= 2.7e-6 (worst at u1 = 2^-6, r = 0.177).
//   r = sqrt.approx(y), y = -2l (one MUFU.SQRT; sqrt.approx(0) = 0, so no zero guard):
//       relative error 1.0e-7 (2^-23.25), measured exhaustively over every fp32 y in
//       [2^-60, 80] on B200 (tools/micro/sqrt_approx_err.cu) -> |dr| <= 8.6e-7 at r = 8.57.
//   theta' = 2pi(u2 - 1/2) in [-pi, pi), from the word's top 32 bits read as a signed
//       integer (hi ^ 2^31 = hi - 2^31) converted once (rounding < 2^-25): sin/cos.approx
//       abs error <= 2^-21.41, plus 2pi * 2^-24 from u2 and the constant: |dcos|, |dsin| <= 7.3e-7.
//   => |z~ - z| <= 2.7e-6 + 8.6e-7 + 8.57 * 7.3e-7 + 1e-6 < 1.1e-5;  NV_EPSZ = 1.5e-5.
__device__ __forceinline__ void nv_approx_pair(uint64_t w0, uint64_t w1, float* z0, float* z1) {
  const uint64_t k1 = w0 >> 11;                        // u1 = k1 * 2^-53
  const float u1f = (float)k1 * 0x1p-53f;
  const float vf = (float)((1ULL << 53) - k1) * 0x1p-53f;  // 1 - u1 (exact integer)
  // y = -2 l: series for small u1 (Horner), SFU log otherwise; both evaluated, one
  // selected.  The factor -2 is folded into the coefficients (power-of-two scaling
  // commutes with rounding), so y is bitwise -2 * fl(l) of the unscaled forms.
  float ser = fmaf(u1f, 2.0f * 0.2f, 2.0f * 0.25f);
  ser = fmaf(u1f, ser, 2.0f * 0.33333334f);
  ser = fmaf(u1f, ser, 2.0f * 0.5f);
  ser = fmaf(u1f, ser, 2.0f * 1.0f);
  const float ys = u1f * ser;
  float lg;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(vf));  // vf >= 2^-53: never subnormal
  const float yl = lg * (-2.0f * 0.69314718055994531f);
  const float y = ((uint32_t)(w0 >> 32) < (1u << 26)) ? ys : yl;  // u1 < 2^-6 (k1 < 2^47)
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(y));     // y >= 2^-52 or exactly 0
  const int32_t h2 = (int32_t)((uint32_t)(w1 >> 32) ^ 0x80000000u);  // 2^32 (u2 - 1/2), truncated
  const float th = (float)h2 * (float)(6.2831853071795865 * 0x1p-32);  // theta - pi, in [-pi, pi)
  float s, c;
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(th));
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(th));
  *z0 = -r * c;
  *z1 = -r * s;
}

// The key q << 12 | local in three instructions: one FFMA evaluates the code scaled by
// 2^12 (one rounding, < 0.07 code, inside the 0.15 nv_classify assumes), and the
// saturating float -> u32 conversion is the clamp (below 0 -> 0, at or above 2^32 ->
// all ones, i.e. q = 2^20 - 1); the low 12 bits are masked off and replaced by local.
__device__ __forceinline__ uint32_t nv_key(float z, uint32_t local) {
  constexpr float kScale = (float)(NV_QSCALE * 4096.0);
  constexpr float kBias = (float)(NV_Z0 * NV_QSCALE * 4096.0);
  uint32_t k;
  asm("cvt.rzi.sat.u32.f32 %0, %1;" : "=r"(k) : "f"(fmaf(z, kScale, kBias)));
  return (k & 0xFFFFF000u) | local;
}

// Exact standard normal #i of the epoch's draw (glibc-exact Box-Muller, _kernels.py:184-190).
__device__ __forceinline__ double nv_exact_z(uint64_t seed, uint64_t sid, uint64_t clo, uint64_t chi,
                                             int64_t i, const double* tab) {
  const phx4 w = philox4x64_10(stream_block_counter(clo, chi, (uint64_t)(i >> 2)), seed, sid);
  const int pair = (int)((i >> 1) & 1);
  double z0, z1;
  glibc_boxmuller_fast(phx_u01(w.v[2 * pair]), phx_u01(w.v[2 * pair + 1]), tab, &z0, &z1);
  return (i & 1) ? z1 : z0;
}

// Query window of one product: z certainly < t - eps or > t + eps outside it.
struct NvWindow {
  double t, eps;
  uint32_t qlo, qhi;  // codes bracketing the ambiguous window (with 3 codes of slack)
};

__device__ __forceinline__ NvWindow nv_window(double x, double mu, double sigma) {
  NvWindow w;
  // 1/sigma from the hardware reciprocal seed and two Newton steps (a few ulps; no IEEE
  // division: t only places the window, and its error is inside eta's slack)
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(sigma));
  r = fma(fma(-sigma, r, 1.0), r, r);
  r = fma(fma(-sigma, r, 1.0), r, r);
  w.t = (x - mu) * r;
  // rounding slack, in z units, of D = fl(mu + fl(sigma*z)) vs x (~2u (|x| + |mu|) / sigma)
  // and of t (~4u (|x| + |mu|) / sigma), u = 2^-53, with margin
  const double eta = 16.0 * 1.1102230246251565e-16 * (fabs(mu) + fabs(x) + 10.0 * sigma) * r;
  w.eps = NV_EPSZ + eta;
  const double a = (w.t - w.eps + NV_Z0) * NV_QSCALE - 3.0;
  const double b = (w.t + w.eps + NV_Z0) * NV_QSCALE + 3.0;
  w.qlo = !(a > 0.0) ? 0u : (a >= (double)NV_QMAX ? (uint32_t)NV_QMAX : (uint32_t)a);
  w.qhi = !(b > 0.0) ? 0u : (b >= (double)NV_QMAX ? (uint32_t)NV_QMAX : (uint32_t)ceil(b));
  return w;
}

// -1: certainly below t, +1: certainly above, 0: ambiguous.  A code q means
// (z~ + 9.5) * 2^20/19 in [q - 0.15, q + 1.15] (fp32 rounding of the code's two
// operations is < 0.15 code); 0.25 code of slack is used on each side.
__device__ __forceinline__ int nv_classify(uint32_t q, const NvWindow& w) {
  const double hiz = (q >= (uint32_t)NV_QMAX) ? INFINITY : ((double)q + 1.25) * NV_W - NV_Z0;
  const double loz = (q == 0u) ? -INFINITY : ((double)q - 0.25) * NV_W - NV_Z0;
  if (hiz + w.eps < w.t) return -1;
  if (loz - w.eps > w.t) return 1;
  return 0;
}

// newsvendor_cost_block (sobench/_kernels.py:210-223), one product.
__device__ __forceinline__ double nv_cost_term(double x, double mu, double sigma, double unit,
                                               double hold, double sell) {
  const double INV_SQRT_TAU = 0.3989422804014327, SQRT1_2 = 0.7071067811865476;
  const double zj = (x - mu) / sigma;
  const double pdf = INV_SQRT_TAU * glibc_exp(-0.5 * zj * zj, simopt_exptab_dev);
  const double cdf = 0.5 * (1.0 + glibc_erf(zj * SQRT1_2, simopt_exptab_dev));
  const double over = sigma * (zj * cdf + pdf);
  const double under = sigma * (pdf - zj * (1.0 - cdf));
  return unit * x + hold * over + sell * under;
}
