// Newsvendor device helpers shared by newsvendor.cu and the C ABI.
#pragma once
#include <stdint.h>

#include "../../include/simopt_b200.h"
#include "glibc_math.cuh"
#include "glibc_tables.h"

#define NV_SEG 2048  // demand draws per bucket-partitioned segment
#define NV_B 512     // buckets per segment

// Monotone bucket map (see newsvendor.cu header).
__device__ __forceinline__ int nv_bucket(double v, double mu, double kappa) {
  const double t = (v - mu) * kappa + (double)(NV_B / 2);
  if (!(t >= 0.0)) return 0;  // also NaN -> 0 (never produced by finite draws)
  if (t >= (double)NV_B) return NV_B - 1;
  return (int)t;
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
