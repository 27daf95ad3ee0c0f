// Euclidean projections onto the two feasible sets of the benchmark (north star:
// "a projection / Frank-Wolfe linear-minimisation step kernel for simplex/box
// feasibility"), used by the projected-SGD driver (psgd.py).  No reference
// counterpart exists (the reference only ships Frank-Wolfe), so parity is against
// the exact sort-based numpy restatement in oracle/oracle.py (tolerance).
//
//   budget set  {x : x >= 0, c . x <= C}     (newsvendor, lmo.py:68-89's polytope;
//                                             c = 1, C = 1 gives the mean-variance
//                                             simplex-with-slack of lmo.py:20-24)
//   box         {x : lo <= x <= hi}
//
// Budget projection: x = max(y - theta c, 0) with theta >= 0 the root of
// f(theta) = sum_j c_j max(y_j - theta c_j, 0) = C (theta = 0 when c . max(y,0) <= C).
// f is continuous, piecewise linear and decreasing: one CTA bisects theta on
// [0, max_j y_j / c_j] with block reductions, then the root is recomputed exactly on
// the active set A = {j : y_j > theta c_j}: theta = (sum_A c y - C) / sum_A c^2, and
// a few Michelot fixed-point passes (recompute A at the new theta) settle the
// breakpoint ties.  Sums over the active set are fixed-order (deterministic).
#include "common.cuh"

namespace {

constexpr int kPT = 1024;

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < kPT / 32; ++w) t += sh[w];
  return t;
}

__device__ __forceinline__ double block_max(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = sh[0];
  for (int w = 1; w < kPT / 32; ++w) t = fmax(t, sh[w]);
  return t;
}

__global__ void __launch_bounds__(kPT) k_project_budget(const double* __restrict__ y,
                                                        const double* __restrict__ c, double C,
                                                        int64_t d, double* __restrict__ out,
                                                        int* __restrict__ status) {
  __shared__ double sh[kPT / 32];
  auto cj = [&](int64_t j) { return c ? c[j] : 1.0; };
  // feasible after clipping at zero?
  double s = 0.0, tmax = 0.0, nan = 0.0;
  for (int64_t j = threadIdx.x; j < d; j += kPT) {
    const double yj = y[j];
    if (yj != yj) nan = 1.0;
    if (yj > 0.0) s += cj(j) * yj;
    tmax = fmax(tmax, yj / cj(j));
  }
  s = block_sum(s, sh);
  tmax = block_max(tmax, sh);
  if (block_sum(nan, sh) > 0.0) {
    if (threadIdx.x == 0 && status) *status = 1;
    return;
  }
  double theta = 0.0;
  if (s > C) {
    double lo = 0.0, hi = tmax;  // f(lo) > C >= f(hi) = 0
    for (int it = 0; it < 80 && lo < hi; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (mid <= lo || mid >= hi) break;
      double f = 0.0;
      for (int64_t j = threadIdx.x; j < d; j += kPT) {
        const double r = y[j] - mid * cj(j);
        if (r > 0.0) f += cj(j) * r;
      }
      f = block_sum(f, sh);
      if (f > C) lo = mid; else hi = mid;
    }
    theta = 0.5 * (lo + hi);
    for (int pass = 0; pass < 4; ++pass) {  // exact root on the active set
      double scy = 0.0, scc = 0.0;
      for (int64_t j = threadIdx.x; j < d; j += kPT) {
        const double cc = cj(j);
        if (y[j] > theta * cc) {
          scy += cc * y[j];
          scc += cc * cc;
        }
      }
      scy = block_sum(scy, sh);
      scc = block_sum(scc, sh);
      if (scc <= 0.0) break;
      const double t2 = (scy - C) / scc;
      if (t2 == theta) break;
      theta = t2;
    }
    if (theta < 0.0) theta = 0.0;
  }
  for (int64_t j = threadIdx.x; j < d; j += kPT) {
    const double r = y[j] - theta * cj(j);
    out[j] = r > 0.0 ? r : 0.0;
  }
}

__global__ void k_project_box(const double* __restrict__ y, double lo, double hi, int64_t d,
                              double* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < d;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = fmin(fmax(y[j], lo), hi);
}

}  // namespace

extern "C" int simopt_project_budget(void* stream, const double* y, const double* c, double budget,
                                     int64_t d, double* out, int* status) {
  SIMOPT_REQUIRE(d >= 0, SIMOPT_E_DIMENSION, "negative dimension");
  SIMOPT_REQUIRE(budget > 0.0, SIMOPT_E_INVALID_CONSTRAINT, "budget must be > 0");
  if (d == 0) return SIMOPT_OK;
  k_project_budget<<<1, kPT, 0, as_stream(stream)>>>(y, c, budget, d, out, status);
  SIMOPT_CHECK_LAUNCH("k_project_budget");
  return SIMOPT_OK;
}

extern "C" int simopt_project_box(void* stream, const double* y, double lo, double hi, int64_t d,
                                  double* out) {
  SIMOPT_REQUIRE(lo <= hi, SIMOPT_E_INVALID_CONSTRAINT, "empty box");
  if (d == 0) return SIMOPT_OK;
  const int64_t g = ceil_div(d, 256);
  k_project_box<<<(int)(g < 2048 ? g : 2048), 256, 0, as_stream(stream)>>>(y, lo, hi, d, out);
  SIMOPT_CHECK_LAUNCH("k_project_box");
  return SIMOPT_OK;
}
