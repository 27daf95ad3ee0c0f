// Frank-Wolfe linear-minimisation oracles on the device (reference: sobench/lmo.py:56-89).
// Both oracles are a first-argmin scan plus a one-hot vertex; NaN in g raises
// InvalidGradient (reported through *status so the call stays asynchronous).
#include "common.cuh"
#include "fw.cuh"

namespace {

constexpr int kThreads = 256;

// mode 0: lmo_simplex_slack  vals = g            vertex value 1.0
// mode 1: lmo_single_budget  vals = g*(C/c_j)    vertex value C/c_j*
__global__ void __launch_bounds__(kThreads)
    k_lmo(int mode, const double* __restrict__ g, const double* __restrict__ c, double budget,
          int64_t n, double* __restrict__ part_v, int64_t* __restrict__ part_i,
          unsigned* __restrict__ done, int* __restrict__ status, double* __restrict__ s_out,
          int64_t* __restrict__ jstar_out) {
  __shared__ ArgMin wb[kThreads / 32];
  __shared__ int nan_seen;
  __shared__ bool last;
  if (threadIdx.x == 0) nan_seen = 0;
  __syncthreads();
  ArgMin b{INFINITY, INT64_MAX};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double gi = g[i];
    if (gi != gi) nan_seen = 1;
    const double v = mode == 0 ? gi : gi * (budget / c[i]);
    b = amin(b, ArgMin{v, i});
    s_out[i] = 0.0;
  }
  b = warp_amin(b);
  if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kThreads / 32; ++w) b = amin(wb[0], wb[w]), wb[0] = b;
    b = wb[0];
    part_v[blockIdx.x] = b.v;
    part_i[blockIdx.x] = b.i;
    if (nan_seen) atomicOr(status, SIMOPT_E_INVALID_GRADIENT);
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  ArgMin r{INFINITY, INT64_MAX};
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x)
    r = amin(r, ArgMin{((volatile double*)part_v)[i], ((volatile int64_t*)part_i)[i]});
  r = warp_amin(r);
  if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = r;
  __syncthreads();
  if (threadIdx.x == 0) {
    r = wb[0];
    for (int w = 1; w < kThreads / 32; ++w) r = amin(r, wb[w]);
    *done = 0;
    if (jstar_out) *jstar_out = r.i;
    if (r.i < n && g[r.i] < 0.0) s_out[r.i] = mode == 0 ? 1.0 : budget / c[r.i];
  }
}

}  // namespace

static int lmo(void* stream, int mode, const double* g, const double* c, double budget, int64_t n,
               double* s_out, int* status) {
  SIMOPT_REQUIRE(n >= 1, SIMOPT_E_DIMENSION, "empty gradient");
  cudaStream_t st = as_stream(stream);
  const int grid = (int)(ceil_div(n, kThreads) < 2 * SIMOPT_NUM_SMS ? ceil_div(n, kThreads)
                                                                      : 2 * SIMOPT_NUM_SMS);
  const size_t bytes = grid * (sizeof(double) + sizeof(int64_t)) + 64;
  unsigned char* ws = static_cast<unsigned char*>(simopt_scratch(st, bytes));
  SIMOPT_REQUIRE(ws != nullptr, SIMOPT_E_CUDA, "%s", simopt_last_error());
  double* pv = reinterpret_cast<double*>(ws);
  int64_t* pi = reinterpret_cast<int64_t*>(ws + grid * sizeof(double));
  unsigned* done = reinterpret_cast<unsigned*>(ws + grid * (sizeof(double) + sizeof(int64_t)));
  SIMOPT_CUDA(cudaMemsetAsync(done, 0, sizeof(unsigned), st));
  k_lmo<<<grid, kThreads, 0, st>>>(mode, g, c, budget, n, pv, pi, done, status, s_out, nullptr);
  SIMOPT_CHECK_LAUNCH("k_lmo");
  return SIMOPT_OK;
}

extern "C" int simopt_lmo_simplex_slack(void* stream, const double* g, int64_t n, double* s_out,
                                        int* status) {
  return lmo(stream, 0, g, nullptr, 0.0, n, s_out, status);
}

extern "C" int simopt_lmo_single_budget(void* stream, const double* g, const double* c,
                                        double budget, int64_t n, double* s_out, int* status) {
  SIMOPT_REQUIRE(budget > 0, SIMOPT_E_INVALID_CONSTRAINT, "budget must be strictly positive");
  return lmo(stream, 1, g, c, budget, n, s_out, status);
}

namespace {
// out[0] = min_i x[i] (NaN if any NaN): feasibility `all(w >= -tol)` (tasks.py:289-290).
__global__ void __launch_bounds__(kThreads) k_minval(const double* __restrict__ x, int64_t n,
                                                     double* __restrict__ out) {
  __shared__ double wm[kThreads / 32];
  double m = INFINITY;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = x[i];
    m = (v < m || v != v) ? v : m;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, m, o);
    m = (t < m || t != t) ? t : m;
  }
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kThreads / 32; ++w) m = (wm[w] < m || wm[w] != wm[w]) ? wm[w] : m;
    *out = (wm[0] != wm[0]) ? wm[0] : m;
  }
}
}  // namespace

extern "C" int simopt_min_value(void* stream, const double* x, int64_t n, double* out) {
  k_minval<<<1, kThreads, 0, as_stream(stream)>>>(x, n, out);
  SIMOPT_CHECK_LAUNCH("k_minval");
  return SIMOPT_OK;
}
