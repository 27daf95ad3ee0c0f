// Logistic-regression task and SQN building blocks on sm_100a.
//
// Reference: sobench/tasks.py:205-253 (logistic loss / gradient / HVP),
// _kernels.py:159-201 (sigmoid, logistic_loss_block), _kernels.py:226-242
// (bfgs_rank2_block), sqn.py:75-110 (hessian_update), sampling.py:196-209
// (sample_indices), sampling.py:229-265 (synth_classification).
// The reductions themselves are the exact-tree matvec/matvec_t kernels of
// reduce.cu (with row gather for mini-batches); this file holds the elementwise
// epilogues, the BFGS rank-2 update and the counter-driven index sampler.
#include "common.cuh"
#include "glibc_math.cuh"
#include "glibc_tables.h"
#include "philox.cuh"
#include "reduce_device.cuh"
#include "rng_device.cuh"

namespace {

int egrid(int64_t n) {
  const int64_t g = ceil_div(n, 256);
  const int64_t cap = (int64_t)SIMOPT_NUM_SMS * 16;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

// c - z_b (tasks.py:236: backend.matvec_t(xb, c - zb)), c = sigmoid(t)
__global__ void k_resid(const double* __restrict__ t, const double* __restrict__ z,
                        const int64_t* __restrict__ idx, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double zi = z[idx ? idx[i] : i];
    out[i] = dev_sigmoid(t[i]) - zi;
  }
}

// weighted = c * (1.0 - c) * tv (tasks.py:252), c = sigmoid(t)
__global__ void k_hvp_weights(const double* __restrict__ t, const double* __restrict__ tv, int64_t n,
                              double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double c = dev_sigmoid(t[i]);
    out[i] = (c * (1.0 - c)) * tv[i];
  }
}

// logistic_loss_block (_kernels.py:193-201)
__global__ void k_loss_terms(const double* __restrict__ t, const double* __restrict__ z,
                             const int64_t* __restrict__ idx, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = glibc_logistic_loss_term(t[i], z[idx ? idx[i] : i], simopt_exptab_dev);
}

// bfgs_rank2_block (_kernels.py:226-242):
// h[i,j] += coef_su*(s_i*u_j) + coef_su*(u_i*s_j) + coef_ss*(s_i*s_j)
// Row per block (grid-stride), columns across threads.  kappa != nullptr: coef_ss is
// formed on the device as (rho*rho)*kappa + rho (sqn.py:108, left to right, no FMA), so
// hessian_update needs no host read of kappa between pairs.
__global__ void k_bfgs_rank2(double* __restrict__ h, const double* __restrict__ s,
                             const double* __restrict__ u, double a, double b,
                             const double* __restrict__ kappa, double rho, int64_t n) {
  if (kappa) b = __dadd_rn(__dmul_rn(__dmul_rn(rho, rho), *kappa), rho);
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const double si = s[i], ui = u[i];
    double* row = h + i * n;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
      const double sj = s[j], uj = u[j];
      const double inc = ((a * (si * uj)) + (a * (ui * sj))) + (b * (si * sj));
      row[j] = row[j] + inc;
    }
  }
}

__global__ void k_diag_fill(double* __restrict__ h, int64_t n, double v) {
  const int64_t total = n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    h[e] = (e / n == e % n) ? v : 0.0;
}

// Elementwise vector ops of the SQN driver (sqn.py:143-149, :154-157), numpy order.
__global__ void k_vec_op(int op, double alpha, const double* __restrict__ x,
                         const double* __restrict__ y, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double r;
    switch (op) {
      case SIMOPT_VEC_SUB_SCALED: r = x[i] - alpha * y[i]; break;  // x - alpha*y
      case SIMOPT_VEC_ADD: r = x[i] + y[i]; break;
      case SIMOPT_VEC_SUB: r = x[i] - y[i]; break;
      case SIMOPT_VEC_MUL: r = x[i] * y[i]; break;
      default: r = x[i] * alpha; break;                             // SCALE
    }
    out[i] = r;
  }
}

// sample_indices (sampling.py:196-209): partial Fisher-Yates over an implicit
// arange(n), one uniform per selected index, j = i + int(u[i] * (n - i)).
// One thread walks the swaps (they are a dependent chain); the displaced
// entries of the permutation live in an open-addressing table in shared memory.
constexpr int kFyCap = 8192;  // table slots (b <= kFyCap/2)

__device__ __forceinline__ int fy_slot(const int64_t* keys, int64_t key) {
  uint64_t hsh = (uint64_t)key * 0x9E3779B97F4A7C15ULL;
  int s = (int)(hsh >> 51);  // 13 bits
  while (keys[s] != -1 && keys[s] != key) s = (s + 1) & (kFyCap - 1);
  return s;
}

__global__ void k_sample_indices(uint64_t seed, uint64_t sid, uint64_t clo, uint64_t chi,
                                 int64_t n, int64_t b, int64_t* __restrict__ out,
                                 uint64_t* __restrict__ words) {
  extern __shared__ int64_t fy[];
  if (words) {  // device-resident stream position (CUDA-graph replay), advanced below
    seed = words[0]; sid = words[1]; clo = words[2]; chi = words[3];
  }
  int64_t* keys = fy;
  int64_t* vals = fy + kFyCap;
  __shared__ double u[kFyCap / 2];
  for (int i = threadIdx.x; i < kFyCap; i += blockDim.x) keys[i] = -1;
  for (int64_t q = threadIdx.x; q < (b + 3) / 4; q += blockDim.x) {
    const phx4 w = philox4x64_10(stream_block_counter(clo, chi, (uint64_t)q), seed, sid);
    for (int k = 0; k < 4; ++k)
      if (4 * q + k < b) u[4 * q + k] = phx_u01(w.v[k]);
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (words) {  // RngStream.advance(b): the 128-bit counter moves ceil(b/4) blocks
    const uint64_t lo = clo + (uint64_t)((b + 3) / 4);
    words[2] = lo;
    words[3] = chi + (lo < clo ? 1ULL : 0ULL);
  }
  for (int64_t i = 0; i < b; ++i) {
    const int64_t j = i + (int64_t)(u[i] * (double)(n - i));
    const int si = fy_slot(keys, i);
    const int64_t vi = keys[si] == -1 ? i : vals[si];
    const int sj = fy_slot(keys, j);
    const int64_t vj = keys[sj] == -1 ? j : vals[sj];
    keys[si] = i; vals[si] = vj;                     // idx[i] <- idx[j]
    const int sj2 = fy_slot(keys, j);
    keys[sj2] = j; vals[sj2] = vi;                   // idx[j] <- old idx[i]
    out[i] = vj;
  }
}

}  // namespace

extern "C" int simopt_logistic_resid(void* stream, const double* t, const double* z,
                                     const int64_t* idx, int64_t n, double* out) {
  if (n == 0) return SIMOPT_OK;
  k_resid<<<egrid(n), 256, 0, as_stream(stream)>>>(t, z, idx, n, out);
  SIMOPT_CHECK_LAUNCH("k_resid");
  return SIMOPT_OK;
}

extern "C" int simopt_logistic_hvp_weights(void* stream, const double* t, const double* tv,
                                           int64_t n, double* out) {
  if (n == 0) return SIMOPT_OK;
  k_hvp_weights<<<egrid(n), 256, 0, as_stream(stream)>>>(t, tv, n, out);
  SIMOPT_CHECK_LAUNCH("k_hvp_weights");
  return SIMOPT_OK;
}

extern "C" int simopt_logistic_loss_terms(void* stream, const double* t, const double* z,
                                          const int64_t* idx, int64_t n, double* out) {
  if (n == 0) return SIMOPT_OK;
  k_loss_terms<<<egrid(n), 256, 0, as_stream(stream)>>>(t, z, idx, n, out);
  SIMOPT_CHECK_LAUNCH("k_loss_terms");
  return SIMOPT_OK;
}

extern "C" int simopt_bfgs_rank2(void* stream, double* h, const double* s, const double* u,
                                 double coef_su, double coef_ss, int64_t n) {
  if (n == 0) return SIMOPT_OK;
  const int grid = (int)(n < 16 * SIMOPT_NUM_SMS ? n : 16 * SIMOPT_NUM_SMS);
  k_bfgs_rank2<<<grid, 256, 0, as_stream(stream)>>>(h, s, u, coef_su, coef_ss, nullptr, 0.0, n);
  SIMOPT_CHECK_LAUNCH("k_bfgs_rank2");
  return SIMOPT_OK;
}

extern "C" int simopt_bfgs_rank2_dev(void* stream, double* h, const double* s, const double* u,
                                     double rho, const double* kappa, int64_t n) {
  if (n == 0) return SIMOPT_OK;
  const int grid = (int)(n < 16 * SIMOPT_NUM_SMS ? n : 16 * SIMOPT_NUM_SMS);
  k_bfgs_rank2<<<grid, 256, 0, as_stream(stream)>>>(h, s, u, -rho, 0.0, kappa, rho, n);
  SIMOPT_CHECK_LAUNCH("k_bfgs_rank2");
  return SIMOPT_OK;
}

extern "C" int simopt_diag_fill(void* stream, double* h, int64_t n, double v) {
  if (n == 0) return SIMOPT_OK;
  k_diag_fill<<<egrid(n * n), 256, 0, as_stream(stream)>>>(h, n, v);
  SIMOPT_CHECK_LAUNCH("k_diag_fill");
  return SIMOPT_OK;
}

extern "C" int simopt_vec_op(void* stream, int op, double alpha, const double* x, const double* y,
                             int64_t n, double* out) {
  SIMOPT_REQUIRE(op >= 0 && op <= 4, SIMOPT_E_CONFIG, "unknown vector op %d", op);
  if (n == 0) return SIMOPT_OK;
  k_vec_op<<<egrid(n), 256, 0, as_stream(stream)>>>(op, alpha, x, y, n, out);
  SIMOPT_CHECK_LAUNCH("k_vec_op");
  return SIMOPT_OK;
}

extern "C" int simopt_sample_indices(void* stream, uint64_t seed, uint64_t sid, uint64_t clo,
                                     uint64_t chi, int64_t n, int64_t b, int64_t* out) {
  SIMOPT_REQUIRE(b >= 1 && b <= n, SIMOPT_E_CONFIG, "need 1 <= b <= n, got b=%lld, n=%lld",
                 (long long)b, (long long)n);
  SIMOPT_REQUIRE(b <= kFyCap / 2, SIMOPT_E_CONFIG, "device sample_indices supports b <= %d",
                 kFyCap / 2);
  static bool attr = false;
  const int smem = 2 * kFyCap * (int)sizeof(int64_t);
  if (!attr) {
    SIMOPT_CUDA(cudaFuncSetAttribute(k_sample_indices, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     smem));
    attr = true;
  }
  k_sample_indices<<<1, 256, smem, as_stream(stream)>>>(seed, sid, clo, chi, n, b, out, nullptr);
  SIMOPT_CHECK_LAUNCH("k_sample_indices");
  return SIMOPT_OK;
}

extern "C" int simopt_sample_indices_dev(void* stream, uint64_t* words, int64_t n, int64_t b,
                                         int64_t* out) {
  SIMOPT_REQUIRE(b >= 1 && b <= n, SIMOPT_E_CONFIG, "need 1 <= b <= n, got b=%lld, n=%lld",
                 (long long)b, (long long)n);
  SIMOPT_REQUIRE(b <= kFyCap / 2, SIMOPT_E_CONFIG, "device sample_indices supports b <= %d",
                 kFyCap / 2);
  static bool attr = false;  // set by the eager warm-up call, not during graph capture
  const int smem = 2 * kFyCap * (int)sizeof(int64_t);
  if (!attr) {
    SIMOPT_CUDA(cudaFuncSetAttribute(k_sample_indices, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     smem));
    attr = true;
  }
  k_sample_indices<<<1, 256, smem, as_stream(stream)>>>(0, 0, 0, 0, n, b, out, words);
  SIMOPT_CHECK_LAUNCH("k_sample_indices");
  return SIMOPT_OK;
}

namespace {
// w <- w - (beta / k) * y with k, beta from the device control block (sqn.py:160-165:
// alpha = beta / k, a true IEEE division of the same operands as the host's)
__global__ void k_sqn_step(const SqnCtl* __restrict__ ctl, const double* __restrict__ x,
                           const double* __restrict__ y, int64_t n, double* __restrict__ out) {
  const double alpha = ctl->beta / (double)ctl->k;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[i] - alpha * y[i];
}

__global__ void k_sqn_record(SqnCtl* ctl, const double* __restrict__ val, double* __restrict__ sums,
                             int64_t* __restrict__ stamps) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const int64_t r = ctl->rec;
  sums[r] = *val;
  stamps[r] = (int64_t)t;
  ctl->rec = r + 1;
  ctl->k += 1;
}
}  // namespace

extern "C" int simopt_sqn_step(void* stream, const SqnCtl* ctl, const double* x, const double* y,
                               int64_t n, double* out) {
  if (n == 0) return SIMOPT_OK;
  k_sqn_step<<<egrid(n), 256, 0, as_stream(stream)>>>(ctl, x, y, n, out);
  SIMOPT_CHECK_LAUNCH("k_sqn_step");
  return SIMOPT_OK;
}

extern "C" int simopt_sqn_record(void* stream, SqnCtl* ctl, const double* val, double* sums,
                                 int64_t* stamps) {
  k_sqn_record<<<1, 1, 0, as_stream(stream)>>>(ctl, val, sums, stamps);
  SIMOPT_CHECK_LAUNCH("k_sqn_record");
  return SIMOPT_OK;
}

// Host-side partial Fisher-Yates for large b (instance label flips, sampling.py:262-264):
// u = the b uniforms of the draw (host copy).  Native runtime helper, O(b).
#include <unordered_map>
extern "C" int simopt_fisher_yates_host(int64_t n, int64_t b, const double* u, int64_t* out) {
  SIMOPT_REQUIRE(b >= 1 && b <= n, SIMOPT_E_CONFIG, "need 1 <= b <= n");
  std::unordered_map<int64_t, int64_t> moved;
  moved.reserve((size_t)(2 * b));
  auto get = [&](int64_t k) {
    auto it = moved.find(k);
    return it == moved.end() ? k : it->second;
  };
  for (int64_t i = 0; i < b; ++i) {
    const int64_t j = i + (int64_t)(u[i] * (double)(n - i));
    const int64_t vi = get(i), vj = get(j);
    moved[i] = vj;
    moved[j] = vi;
    out[i] = vj;
  }
  return SIMOPT_OK;
}

namespace {
// One CG step on device scalars (oracle.newton_cg; no host round trip):
//   alpha = rr / dHd; p = p + alpha*d; r = r - alpha*Hd       (skipped when rr == 0: `break`)
__global__ void k_cg_step1(double* __restrict__ p, double* __restrict__ r, const double* __restrict__ d,
                           const double* __restrict__ hd, const double* __restrict__ rr,
                           const double* __restrict__ dhd, int64_t n) {
  const double rrv = *rr;
  if (rrv == 0.0) return;
  const double alpha = rrv / *dhd;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    p[i] = p[i] + alpha * d[i];
    r[i] = r[i] - alpha * hd[i];
  }
}
//   beta = rr_new / rr; d = r + beta*d                           (skipped when rr == 0)
__global__ void k_cg_step2(double* __restrict__ d, const double* __restrict__ r,
                           const double* __restrict__ rr_new, const double* __restrict__ rr, int64_t n) {
  const double rrv = *rr;
  if (rrv == 0.0) return;
  const double beta = *rr_new / rrv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    d[i] = r[i] + beta * d[i];
}
}  // namespace

extern "C" int simopt_cg_step1(void* stream, double* p, double* r, const double* d, const double* hd,
                               const double* rr, const double* dhd, int64_t n) {
  k_cg_step1<<<egrid(n), 256, 0, as_stream(stream)>>>(p, r, d, hd, rr, dhd, n);
  SIMOPT_CHECK_LAUNCH("k_cg_step1");
  return SIMOPT_OK;
}

extern "C" int simopt_cg_step2(void* stream, double* d, const double* r, const double* rr_new,
                               const double* rr, int64_t n) {
  k_cg_step2<<<egrid(n), 256, 0, as_stream(stream)>>>(d, r, rr_new, rr, n);
  SIMOPT_CHECK_LAUNCH("k_cg_step2");
  return SIMOPT_OK;
}
