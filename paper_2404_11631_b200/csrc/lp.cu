// lmo_general (sobench/lmo.py:92-160): argmin of s.g over {A s <= C, s >= 0} by the
// reference's dense primal simplex -- slack basis start, Bland's rule (lowest-index
// entering column; minimum-ratio leaving row with ties to the lowest basic index).
//
// One CTA runs the whole solve on the device: the tableau [A | I | C] (m x (n+m+1)
// doubles) and the reduced-cost row live in L2-resident scratch, every pivot is a
// parallel first-index search for the entering column, a sequential ratio test (the
// reference's comparison chain, same tolerances), and the row operations spread over
// all threads.  Every arithmetic step is the reference's numpy expression with the
// same rounding (row /= piv; row_i -= f_i * row_leave; cost -= c_e * row_leave; no
// FMA), so the vertex is the reference's bit for bit.  Intended, like the reference,
// for the small multi-resource instances (m <= 64, n <= 1e4); the single-budget
// benchmark path never calls it.
#include <math.h>

#include "common.cuh"

namespace {

constexpr int kLpThreads = 1024;

__device__ __forceinline__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  v = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
  if (warp == 0)
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (threadIdx.x == 0) red[0] = v;
  __syncthreads();
  return red[0];
}

__device__ __forceinline__ int64_t block_min_i64(int64_t v, int64_t* red) {
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t t = __shfl_xor_sync(0xffffffffu, v, o);
    v = t < v ? t : v;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  v = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : INT64_MAX;
  if (warp == 0)
    for (int o = 16; o > 0; o >>= 1) {
      const int64_t t = __shfl_xor_sync(0xffffffffu, v, o);
      v = t < v ? t : v;
    }
  if (threadIdx.x == 0) red[0] = v;
  __syncthreads();
  return red[0];
}

// status: 0 ok, SIMOPT_E_INVALID_GRADIENT (NaN in g), SIMOPT_E_SOLVER_STALL (unbounded),
// -SIMOPT_E_SOLVER_STALL (iteration cap reached)
__global__ void __launch_bounds__(kLpThreads)
    k_lmo_general(const double* __restrict__ A, const double* __restrict__ C, int64_t m, int64_t n,
                  const double* __restrict__ g, int64_t cap, double* __restrict__ tab,
                  double* __restrict__ cost, int64_t* __restrict__ basis, double* __restrict__ fac,
                  double* __restrict__ s, int* __restrict__ status) {
  __shared__ double redd[32];
  __shared__ int64_t redi[32];
  __shared__ int nan_seen;
  __shared__ int64_t leave_s;
  __shared__ double piv_s, cc_s;
  const int tid = threadIdx.x, bs = blockDim.x;
  const int64_t W = n + m + 1, nm = n + m;
  if (tid == 0) nan_seen = 0;
  __syncthreads();
  double amax = 0.0;
  for (int64_t j = tid; j < n; j += bs) {
    const double gj = g[j];
    if (gj != gj) nan_seen = 1;
    amax = fmax(amax, fabs(gj));
  }
  amax = block_max(amax, redd);  // also orders nan_seen
  if (nan_seen) {
    if (tid == 0) *status = SIMOPT_E_INVALID_GRADIENT;
    return;
  }
  const double scale = 1.0 + amax;       // lmo.py:120
  const double enter_tol = 1e-12 * scale;
  const double pivot_tol = 1e-12;
  // tableau rows [A | I | rhs], reduced costs [g | 0], slack basis (lmo.py:110-117)
  for (int64_t i = 0; i < m; ++i) {
    double* row = tab + i * W;
    for (int64_t j = tid; j < W; j += bs)
      row[j] = j < n ? A[i * n + j] : (j < nm ? (j - n == i ? 1.0 : 0.0) : C[i]);
  }
  for (int64_t j = tid; j < nm; j += bs) cost[j] = j < n ? g[j] : 0.0;
  for (int64_t i = tid; i < m; i += bs) basis[i] = n + i;
  __syncthreads();
  bool optimal = false;
  for (int64_t it = 0; it < cap; ++it) {
    // entering: the lowest index with a reduced cost below -enter_tol
    int64_t cand = INT64_MAX;
    for (int64_t j = tid; j < nm; j += bs)
      if (cost[j] < -enter_tol) { cand = j; break; }
    const int64_t e = block_min_i64(cand, redi);
    if (e == INT64_MAX) { optimal = true; break; }
    if (tid == 0) {  // ratio test, the reference's sequential comparison chain
      double best = INFINITY;
      int64_t lr = -1;
      for (int64_t i = 0; i < m; ++i) {
        const double ci = tab[i * W + e];
        if (ci > pivot_tol) {
          const double ratio = tab[i * W + W - 1] / ci;
          if (ratio < best - 1e-15 ||
              (fabs(ratio - best) <= 1e-15 && (lr < 0 || basis[i] < basis[lr]))) {
            best = ratio;
            lr = i;
          }
        }
      }
      leave_s = lr;
      piv_s = lr >= 0 ? tab[lr * W + e] : 0.0;
      cc_s = cost[e];
    }
    __syncthreads();
    const int64_t lr = leave_s;
    if (lr < 0) {
      if (tid == 0) *status = SIMOPT_E_SOLVER_STALL;
      return;
    }
    double* prow = tab + lr * W;
    const double piv = piv_s;
    for (int64_t j = tid; j < W; j += bs) prow[j] = prow[j] / piv;
    for (int64_t i = tid; i < m; i += bs) fac[i] = (i == lr) ? 0.0 : tab[i * W + e];
    __syncthreads();
    for (int64_t i = 0; i < m; ++i) {
      const double f = fac[i];
      if (i == lr || f == 0.0) continue;
      double* row = tab + i * W;
      for (int64_t j = tid; j < W; j += bs) row[j] = row[j] - f * prow[j];
    }
    const double cc = cc_s;
    if (cc != 0.0)
      for (int64_t j = tid; j < nm; j += bs) cost[j] = cost[j] - cc * prow[j];
    if (tid == 0) basis[lr] = e;
    __syncthreads();
  }
  if (!optimal) {
    if (tid == 0) *status = -SIMOPT_E_SOLVER_STALL;
    return;
  }
  for (int64_t j = tid; j < n; j += bs) s[j] = 0.0;
  __syncthreads();
  for (int64_t i = tid; i < m; i += bs) {
    const int64_t b = basis[i];
    if (b < n) s[b] = tab[i * W + W - 1];
  }
  if (tid == 0) *status = 0;
}

}  // namespace

extern "C" int simopt_lmo_general(void* stream, const double* A, const double* C, int64_t m,
                                  int64_t n, const double* g, int64_t max_iters, double* s_out,
                                  int* status) {
  SIMOPT_REQUIRE(m >= 1 && n >= 1, SIMOPT_E_DIMENSION, "empty polytope (%lld x %lld)",
                 (long long)m, (long long)n);
  SIMOPT_REQUIRE(max_iters >= 0, SIMOPT_E_CONFIG, "max_iters must be >= 0");
  cudaStream_t st = as_stream(stream);
  const int64_t W = n + m + 1;
  const size_t bytes = sizeof(double) * (size_t)(m * W + (n + m) + m) + sizeof(int64_t) * (size_t)m;
  double* tab = static_cast<double*>(simopt_scratch(st, bytes));
  SIMOPT_REQUIRE(tab != nullptr, SIMOPT_E_CUDA, "%s", simopt_last_error());
  double* cost = tab + m * W;
  double* fac = cost + (n + m);
  int64_t* basis = reinterpret_cast<int64_t*>(fac + m);
  k_lmo_general<<<1, kLpThreads, 0, st>>>(A, C, m, n, g, max_iters, tab, cost, basis, fac, s_out,
                                          status);
  SIMOPT_CHECK_LAUNCH("k_lmo_general");
  return SIMOPT_OK;
}
