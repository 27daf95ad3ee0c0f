// Frank-Wolfe linear-minimisation oracles on the device (reference: sobench/lmo.py:56-89).
// Both oracles are a first-argmin scan plus a one-hot vertex; NaN in g raises
// InvalidGradient (reported through *status so the call stays asynchronous).
#include "common.cuh"
#include "fw.cuh"
#include "reduce_device.cuh"

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

namespace {
// One mean-variance FW step after its gradient, in ONE block (frank_wolfe.py:106-117 for
// MeanVarProblem): lmo_simplex_slack (lmo.py:56-65; first argmin, NaN -> status), the
// update dir = (-1 * w) + s, w' = (gamma * dir) + w (frank_wolfe.py:69-82, the same
// IEEE operations as simopt_axpy / simopt_axpy_ptr), min(w') for the feasibility test,
// and the exact fixed-tree sums sum(w') and dot(w', mean) (backend.py:80-111): chunk
// chains strictly in order, one thread per chunk, folded pairwise.  Replaces seven
// launches (memset, lmo, two axpys, min, two tree reductions) per step.
constexpr int kTailThreads = 1024;

__global__ void __launch_bounds__(kTailThreads)
    k_mv_fw_tail(const double* __restrict__ g, const double* __restrict__ w_in,
                 const double* __restrict__ gamma, const double* __restrict__ mean, int64_t d,
                 int64_t chunk, double* __restrict__ w_out, int* __restrict__ status,
                 double* __restrict__ wmin_out, double* __restrict__ wsum_out,
                 double* __restrict__ lin_out, double* __restrict__ part, bool use_smem,
                 bool exact) {
  __shared__ ArgMin wb[kTailThreads / 32];
  __shared__ double wm[kTailThreads / 32];
  __shared__ double rs[kTailThreads / 32], rd[kTailThreads / 32];  // fast-mode warp sums
  __shared__ int nan_seen;
  __shared__ int64_t jstar_sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) nan_seen = 0;
  __syncthreads();
  ArgMin b{INFINITY, INT64_MAX};
  for (int64_t i = tid; i < d; i += kTailThreads) {
    const double gi = g[i];
    if (gi != gi) nan_seen = 1;
    b = amin(b, ArgMin{gi, i});
  }
  b = warp_amin(b);
  if (lane == 0) wb[warp] = b;
  __syncthreads();
  if (tid == 0) {
    ArgMin r = wb[0];
    for (int w = 1; w < kTailThreads / 32; ++w) r = amin(r, wb[w]);
    if (nan_seen) atomicOr(status, SIMOPT_E_INVALID_GRADIENT);
    jstar_sh = (r.i < d && g[r.i] < 0.0) ? r.i : -1;  // vertex e_j* iff g_j* < 0, else 0
  }
  __syncthreads();
  const int64_t js = jstar_sh;
  const double gm = *gamma;
  extern __shared__ double tail_sm[];  // [d] w_out, [d] mean when they fit (chains read smem)
  const bool in_smem = use_smem;
  double m = INFINITY;
  double ps = 0.0, pd = 0.0;  // fast mode: this thread's strided share of sum(w'), dot(w', mean)
  for (int64_t i = tid; i < d; i += kTailThreads) {
    const double wi = w_in[i];
    const double si = (i == js) ? 1.0 : 0.0;
    const double dir = -1.0 * wi + si;
    const double wo = gm * dir + wi;
    w_out[i] = wo;
    if (!exact) {
      ps += wo;
      pd += wo * mean[i];
    } else if (in_smem) {
      tail_sm[i] = wo;
      tail_sm[d + i] = mean[i];
    }
    m = (wo < m || wo != wo) ? wo : m;
  }
  if (!exact) {
    // fused (tolerance) mode: block-parallel sums in a fixed order -- deterministic run to
    // run, not the reference tree; the 1000-long sequential chains are 8 us at C1's d
    for (int o = 16; o > 0; o >>= 1) {
      ps += __shfl_xor_sync(0xffffffffu, ps, o);
      pd += __shfl_xor_sync(0xffffffffu, pd, o);
    }
    if (lane == 0) { rs[warp] = ps; rd[warp] = pd; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, m, o);
    m = (t < m || t != t) ? t : m;
  }
  if (lane == 0) wm[warp] = m;
  __syncthreads();  // also publishes w_out to the whole block for the chains below
  if (tid == 0) {
    for (int w = 1; w < kTailThreads / 32; ++w) m = (wm[w] < m || wm[w] != wm[w]) ? wm[w] : m;
    *wmin_out = (wm[0] != wm[0]) ? wm[0] : m;
  }
  if (!exact) {
    if (tid == 0) {
      double a = 0.0, b2 = 0.0;
      for (int w = 0; w < kTailThreads / 32; ++w) {
        a += rs[w];
        b2 += rd[w];
      }
      *wsum_out = a;
      *lin_out = b2;
    }
    return;
  }
  if (!in_smem) return;  // large d: the host wrapper runs the exact sums as a tree kernel
  // exact chains: threads [0, nch) sum(w'), threads [nch, 2 nch) dot(w', mean)
  const int64_t nch = (d + chunk - 1) / chunk;
  if (tid < 2 * nch) {
    const int64_t c = tid < nch ? tid : tid - nch;
    const int64_t lo = c * chunk, hi = lo + chunk < d ? lo + chunk : d;
    // one in-order chain per chunk; loads batched 8 ahead (seq_sum / seq_dot), from shared
    // memory when the vectors fit (an L2 round trip per batch would dominate otherwise)
    const double* wv = in_smem ? tail_sm : w_out;
    const double* mv = in_smem ? tail_sm + d : mean;
    part[tid] = tid < nch ? seq_sum(wv, lo, hi) : seq_dot(wv, mv, lo, hi);
  }
  __syncthreads();
  if (tid < 2) {
    double* p = part + tid * nch;
    int64_t mm = nch;
    while (mm > 1) {  // fold_pairwise (_kernels.py:30-42)
      const int64_t h = mm >> 1;
      for (int64_t i = 0; i < h; ++i) p[i] = p[2 * i] + p[2 * i + 1];
      if (mm & 1) { p[h] = p[mm - 1]; mm = h + 1; } else { mm = h; }
    }
    *(tid == 0 ? wsum_out : lin_out) = nch ? p[0] : 0.0;
  }
}
}  // namespace

extern "C" int simopt_mv_fw_tail(void* stream, const double* g, const double* w_in,
                                 const double* gamma, const double* mean, int64_t d, int64_t chunk,
                                 double* w_out, int* status, double* wmin_out, double* wsum_out,
                                 double* lin_out, int exact) {
  SIMOPT_REQUIRE(d >= 1, SIMOPT_E_DIMENSION, "empty gradient");
  SIMOPT_REQUIRE(chunk >= 1, SIMOPT_E_CONFIG, "chunk_size must be >= 1");
  const int64_t nch = ceil_div(d, chunk);
  SIMOPT_REQUIRE(2 * nch <= kTailThreads, SIMOPT_E_CONFIG, "too many chunks for the fused FW tail");
  cudaStream_t st = as_stream(stream);
  double* part = static_cast<double*>(simopt_scratch(st, 2 * nch * sizeof(double)));
  SIMOPT_REQUIRE(part != nullptr, SIMOPT_E_CUDA, "%s", simopt_last_error());
  const size_t smem = exact ? (size_t)2 * d * sizeof(double) : 0;
  const bool use_smem = exact && smem <= 96 * 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_mv_fw_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr = true;
  }
  k_mv_fw_tail<<<1, kTailThreads, use_smem ? smem : 0, st>>>(g, w_in, gamma, mean, d, chunk, w_out,
                                                             status, wmin_out, wsum_out, lin_out,
                                                             part, use_smem, exact != 0);
  SIMOPT_CHECK_LAUNCH("k_mv_fw_tail");
  if (!exact) return SIMOPT_OK;
  // vectors too large for one block's shared memory: the exact sums as a warp-per-chunk
  // tree kernel (one chain per 4096-chunk in a single block would wait on L2 per batch)
  if (!use_smem)
    return simopt_tree_sums2(stream, w_out, mean, d, lin_out, w_out, nullptr, d, wsum_out, chunk);
  return SIMOPT_OK;
}
