// Newsvendor device helpers shared by newsvendor.cu and the C ABI.
//
// Epoch layout ("keyed ECDF"): every demand draw of the epoch is stored as one
// 32-bit key  q << 12 | local,  where local (12 bits) is the draw's position in
// its 4096-draw segment and q (20 bits) is a fixed-point code of an fp32
// approximation z~ of its standard normal z:
//     q = clamp(floor((z~ + 9.5) * 2^20 / 19), 0, 2^20 - 1).
// |z~ - z| <= NV_EPSZ is guaranteed by construction (fp32 log1pf/logf/sqrtf/
// sincospif are <= 2 ulp; the bound used is ~20x the worst case), and q is
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
#define NV_EPSZ 1e-4                  // guaranteed |z~ - z| bound (actual < 6e-6)

// fp32 approximation of one Box-Muller pair (both components).
__device__ __forceinline__ void nv_approx_pair(double u1, double u2, float* z0, float* z1) {
  // -2*log1p(-u1): log1pf for small u1, logf(1 - u1) (1 - u1 exact in double) near 1
  const float l = (u1 < 0.5) ? log1pf(-(float)u1) : logf((float)(1.0 - u1));
  const float r = sqrtf(-2.0f * l);
  float s, c;
  sincospif(2.0f * (float)u2, &s, &c);
  *z0 = r * c;
  *z1 = r * s;
}

__device__ __forceinline__ uint32_t nv_code(float z) {
  const float t = (z + (float)NV_Z0) * (float)NV_QSCALE;
  if (!(t >= 0.0f)) return 0u;
  if (t >= (float)NV_QMAX) return (uint32_t)NV_QMAX;
  return (uint32_t)t;
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
  w.t = (x - mu) / sigma;
  // rounding slack of D = fl(mu + fl(sigma*z)) vs x and of t, in z units
  const double eta = 8.0 * 1.1102230246251565e-16 * (fabs(mu) + fabs(x) + 10.0 * sigma) / sigma;
  w.eps = NV_EPSZ + eta;
  const double a = (w.t - w.eps + NV_Z0) * NV_QSCALE - 3.0;
  const double b = (w.t + w.eps + NV_Z0) * NV_QSCALE + 3.0;
  w.qlo = !(a > 0.0) ? 0u : (a >= (double)NV_QMAX ? (uint32_t)NV_QMAX : (uint32_t)a);
  w.qhi = !(b > 0.0) ? 0u : (b >= (double)NV_QMAX ? (uint32_t)NV_QMAX : (uint32_t)ceil(b));
  return w;
}

// -1: certainly below t, +1: certainly above, 0: ambiguous.
__device__ __forceinline__ int nv_classify(uint32_t q, const NvWindow& w) {
  const double hiz = (q >= (uint32_t)NV_QMAX) ? INFINITY : ((double)q + 2.0) * NV_W - NV_Z0;
  const double loz = (q == 0u) ? -INFINITY : ((double)q - 1.0) * NV_W - NV_Z0;
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
  const double cdf = 0.5 * (1.0 + erf(zj * SQRT1_2));
  const double over = sigma * (zj * cdf + pdf);
  const double under = sigma * (pdf - zj * (1.0 - cdf));
  return unit * x + hold * over + sell * under;
}
