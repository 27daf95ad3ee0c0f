// Device building blocks of the fixed reduction tree and the glibc-exact maps.
#pragma once
#include "glibc_math.cuh"
#include "glibc_tables.h"

// Strictly sequential chunk sums (dot_partials / sum_partials, _kernels.py:45-68).
// Loads are batched 8 ahead for memory-level parallelism; the adds stay a single
// dependent chain in index order.
__device__ __forceinline__ double seq_dot(const double* __restrict__ x,
                                          const double* __restrict__ y, int64_t lo, int64_t hi) {
  double s = 0.0;
  int64_t i = lo;
  for (; i + 8 <= hi; i += 8) {
    double xv[8], yv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { xv[k] = x[i + k]; yv[k] = y[i + k]; }
#pragma unroll
    for (int k = 0; k < 8; ++k) s = s + xv[k] * yv[k];
  }
  for (; i < hi; ++i) s = s + x[i] * y[i];
  return s;
}

__device__ __forceinline__ double seq_sum(const double* __restrict__ x, int64_t lo, int64_t hi) {
  double s = 0.0;
  int64_t i = lo;
  for (; i + 8 <= hi; i += 8) {
    double xv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) xv[k] = x[i + k];
#pragma unroll
    for (int k = 0; k < 8; ++k) s = s + xv[k];
  }
  for (; i < hi; ++i) s = s + x[i];
  return s;
}

__device__ __forceinline__ double dev_exp(double x) { return glibc_exp(x, simopt_exptab_dev); }
__device__ __forceinline__ double dev_sigmoid(double t) { return glibc_sigmoid(t, simopt_exptab_dev); }
