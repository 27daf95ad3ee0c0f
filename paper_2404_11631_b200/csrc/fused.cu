// Fused single-pass "row dot -> per-row weight -> column accumulate" kernels.
//
// Every big streaming pass of the three tasks has the same shape
//     t_r  = x_r . v                     (row dot over d columns)
//     wt_r = f(t_r, aux_r)               (per-row epilogue)
//     g_j  = sum_r x_rj * wt_r           (column accumulation over N rows)
// with, in reference terms,
//   MV       mean-variance gradient  tasks.py:78-85   x = X - mean, f = identity;
//            the recorded objective's |Xc w|^2 (tasks.py:67-75) is the side sum
//   LR_GRAD  logistic gradient       tasks.py:228-236 f = sigmoid(t) - z; the side
//            sum is the loss of tasks.py:216-225, and c(1-c) (tasks.py:252) is
//            written for the following HVPs
//   LR_HVP   logistic HVP            tasks.py:239-253 f = dw_r * t_r
// The reference evaluates each as matvec + matvec_t, two passes over X.  Here a
// row tile is loaded once into registers, its dots are reduced (warp shuffles,
// then across the CTA, then -- for wide rows -- across a thread-block cluster
// through distributed shared memory), and the same registers feed the column
// accumulation: one HBM pass per evaluation.
//
// Summation order is NOT the reference's fixed 4096-chunk tree (that is the
// exact mode, reduce.cu); results agree to ~1e-15 relative, inside the
// north-star gradient tolerance (1e-10).  The order is fixed by the grid
// (static tile striding, per-cluster partials folded in cluster order), so a
// pass is deterministic run to run.
//
// Layout: X row-major N x d fp64.  A cluster of C CTAs splits the columns into
// C bands (even width); each CTA's 256 threads own column pairs
// (16-byte loads) p = tid + k*256, k < K.  A tile is R rows; one thread holds
// R*K double2 of it.
#include <cooperative_groups.h>

#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"
#include "reduce_device.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int kNT = 256;
constexpr int kNW = kNT / 32;

struct FusedArgs {
  const double* X;
  int64_t N, d;
  const double* v;       // d
  const double* mean;    // d (MV)
  const double* rowaux;  // N: labels z (LR_GRAD) or c(1-c) (LR_HVP)
  double* t_out;         // N, optional
  double* dw_out;        // N, optional (LR_GRAD)
  double* col_part;      // [ncl][d]
  double* scal_part;     // [ncl]
  int accumulate;
};

__device__ __forceinline__ double2 ld2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

// Bulk L2 prefetch of one contiguous row band (TMA engine; no registers, no smem).
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <int MODE, int C, int K, bool VEC>
__global__ void __launch_bounds__(kNT, 2) k_fused_rows(FusedArgs a) {
  constexpr int R = (16 / K) < 1 ? 1 : 16 / K;
  extern __shared__ __align__(16) double vs[];  // [band] v, then [band] mean (MV)
  __shared__ double red[2][R][kNW];
  __shared__ double part[2][R];
  __shared__ double wts[2][R];
  __shared__ double sred[kNW];
  const int tid = threadIdx.x;
  int rank = 0;
  if constexpr (C > 1) rank = (int)cg::this_cluster().block_rank();
  const int64_t cl = blockIdx.x / C, ncl = gridDim.x / C;
  const int64_t d = a.d, N = a.N;
  int64_t band = (d + C - 1) / C;
  band += band & 1;
  const int64_t b0 = rank * band;
  const int64_t b1 = b0 + band < d ? b0 + band : d;
  // v (and the mean) of this band, zero-padded to K*256 pairs
  double* ms = vs + 2 * K * kNT;
  for (int i = tid; i < 2 * K * kNT; i += kNT) {
    const int64_t c = b0 + i;
    vs[i] = c < b1 ? a.v[c] : 0.0;
    if (MODE == SIMOPT_FUSED_MV) ms[i] = c < b1 ? a.mean[c] : 0.0;
  }
  __syncthreads();
  const double2* v2 = reinterpret_cast<const double2*>(vs);
  const double2* m2 = reinterpret_cast<const double2*>(ms);
#define COL(k) (b0 + 2 * (int64_t)(tid + (k) * kNT))
  double2 acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = make_double2(0.0, 0.0);
  double sc = 0.0;
  const int64_t ntiles = (N + R - 1) / R;
  int par = 0;
  const uint32_t band_bytes = (uint32_t)(((b1 - b0) * 8 + 15) & ~15LL);
  for (int64_t tile = cl; tile < ntiles; tile += ncl, par ^= 1) {
    const int64_t r0 = tile * R;
    // keep HBM busy through this tile's reductions: the next tile's rows go to L2 now
    if (VEC && tid < R && b1 > b0) {
      const int64_t rn = r0 + ncl * R + tid;
      if (rn < N) prefetch_l2(a.X + rn * d + b0, band_bytes);
    }
    double2 x[R][K];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const bool rv = r0 + i < N;
      const double* row = a.X + (rv ? r0 + i : 0) * d;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int64_t c = COL(k);
        if (VEC) {
          x[i][k] = (rv && c < b1) ? ld2(row + c) : make_double2(0.0, 0.0);
        } else {
          x[i][k].x = (rv && c < b1) ? __ldg(row + c) : 0.0;
          x[i][k].y = (rv && c + 1 < b1) ? __ldg(row + c + 1) : 0.0;
        }
      }
    }
    double s[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      double acc_s = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const double2 vk = v2[tid + k * kNT];
        if (MODE == SIMOPT_FUSED_MV) {
          // Xc = X - mean (tasks.py:63); out-of-range rows are discarded (wt = 0)
          const double2 mk = m2[tid + k * kNT];
          x[i][k].x = x[i][k].x - mk.x;
          x[i][k].y = x[i][k].y - mk.y;
        }
        acc_s = fma(x[i][k].x, vk.x, acc_s);
        acc_s = fma(x[i][k].y, vk.y, acc_s);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc_s += __shfl_xor_sync(0xffffffffu, acc_s, o);
      s[i] = acc_s;
    }
    if ((tid & 31) == 0) {
#pragma unroll
      for (int i = 0; i < R; ++i) red[par][i][tid >> 5] = s[i];
    }
    __syncthreads();
    if (tid < R) {
      double p = 0.0;
#pragma unroll
      for (int w = 0; w < kNW; ++w) p += red[par][tid][w];
      part[par][tid] = p;
    }
    if constexpr (C > 1) {
      cg::this_cluster().sync();
    } else {
      __syncthreads();
    }
    if (tid < R) {
      double t = 0.0;
      if constexpr (C > 1) {
        cg::cluster_group cluster = cg::this_cluster();
#pragma unroll
        for (int q = 0; q < C; ++q) t += *cluster.map_shared_rank(&part[par][tid], q);
      } else {
        t = part[par][tid];
      }
      const int64_t r = r0 + tid;
      double wt = 0.0;
      if (r < N) {
        if (MODE == SIMOPT_FUSED_MV) {
          wt = t;
          sc = fma(t, t, sc);
        } else if (MODE == SIMOPT_FUSED_LR_GRAD) {
          const double z = a.rowaux[r];
          const double c = dev_sigmoid(t);
          wt = c - z;
          if (rank == 0) {
            if (a.dw_out) a.dw_out[r] = c * (1.0 - c);
            sc += glibc_logistic_loss_term(t, z, simopt_exptab_dev);
          }
        } else {
          wt = a.rowaux[r] * t;
        }
        if (rank == 0 && a.t_out) a.t_out[r] = t;
      }
      wts[par][tid] = wt;
    }
    __syncthreads();
    if (a.accumulate) {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const double wt = wts[par][i];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          acc[k].x = fma(x[i][k].x, wt, acc[k].x);
          acc[k].y = fma(x[i][k].y, wt, acc[k].y);
        }
      }
    }
  }
  if (a.accumulate) {
    double* out = a.col_part + cl * d;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int64_t c = COL(k);
      if (c < b1) out[c] = acc[k].x;
      if (c + 1 < b1) out[c + 1] = acc[k].y;
    }
  }
  if (rank == 0) {
    // scalar side sum: only threads < R carry one; reduce in thread order
    double v = sc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) sred[tid >> 5] = v;
    __syncthreads();
    if (tid == 0) {
      double p = 0.0;
      for (int w = 0; w < kNW; ++w) p += sred[w];
      a.scal_part[cl] = p;
    }
  }
  if constexpr (C > 1) cg::this_cluster().sync();  // keep smem alive for remote readers
#undef COL
}

// out[j] = (sum_cl part[cl][j]) * scale - center[j];  scalar = sum_cl spart[cl]
// Block = 32 columns x 8 warps; warp w sums clusters w, w+8, ... (independent loads),
// then the 8 warp partials are added in warp order (fixed order: deterministic).
__global__ void __launch_bounds__(256) k_fused_finish(const double* __restrict__ part,
                                                      const double* __restrict__ spart, int64_t ncl,
                                                      int64_t d, double scale,
                                                      const double* __restrict__ center,
                                                      double* __restrict__ out,
                                                      double* __restrict__ scalar_out) {
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (out) {
    const int64_t j = blockIdx.x * 32LL + lane;
    double s = 0.0;
    if (j < d) {
      for (int64_t c = w; c < ncl; c += 8) s += part[c * d + j];
    }
    red[w][lane] = s;
    __syncthreads();
    if (w == 0 && j < d) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) t += red[k][lane];
      t = t * scale;
      out[j] = center ? t - center[j] : t;
    }
  }
  if (scalar_out && blockIdx.x == 0 && threadIdx.x == 0) {
    double s = 0.0;
    for (int64_t c = 0; c < ncl; ++c) s += spart[c];
    *scalar_out = s;
  }
}

using KernelFn = void (*)(FusedArgs);

template <int MODE, int C, int K>
KernelFn pick_vec(bool vec) {
  return vec ? k_fused_rows<MODE, C, K, true> : k_fused_rows<MODE, C, K, false>;
}

template <int MODE, int C>
KernelFn pick_k(int K, bool vec) {
  switch (K) {
    case 1: return pick_vec<MODE, C, 1>(vec);
    case 2: return pick_vec<MODE, C, 2>(vec);
    case 3: return pick_vec<MODE, C, 3>(vec);
    case 4: return pick_vec<MODE, C, 4>(vec);
    case 5: return pick_vec<MODE, C, 5>(vec);
    case 6: return pick_vec<MODE, C, 6>(vec);
    default: return pick_vec<MODE, C, 8>(vec);
  }
}

template <int MODE>
KernelFn pick_c(int C, int K, bool vec) {
  switch (C) {
    case 1: return pick_k<MODE, 1>(K, vec);
    case 2: return pick_k<MODE, 2>(K, vec);
    case 4: return pick_k<MODE, 4>(K, vec);
    default: return pick_k<MODE, 8>(K, vec);
  }
}

KernelFn pick(int mode, int C, int K, bool vec) {
  switch (mode) {
    case SIMOPT_FUSED_MV: return pick_c<SIMOPT_FUSED_MV>(C, K, vec);
    case SIMOPT_FUSED_LR_GRAD: return pick_c<SIMOPT_FUSED_LR_GRAD>(C, K, vec);
    default: return pick_c<SIMOPT_FUSED_LR_HVP>(C, K, vec);
  }
}

// Column split: the smallest cluster size C in {1,2,4,8} and pairs-per-thread K
// in {1..6,8} such that a band of ceil(d/C) columns fits K*256 column pairs.
bool geometry(int64_t d, int* C, int* K) {
  for (int c : {1, 2, 4, 8}) {
    int64_t band = (d + c - 1) / c;
    band += band & 1;
    const int64_t pairs = band / 2;
    const int64_t k = (pairs + kNT - 1) / kNT;
    const int64_t kmax = (c == 8) ? 8 : 4;  // prefer wider clusters over very long rows
    if (k <= kmax) {
      *C = c;
      *K = (int)(k == 7 ? 8 : (k < 1 ? 1 : k));
      return true;
    }
  }
  return false;
}

size_t dyn_smem(int mode, int K) {
  return (size_t)(mode == SIMOPT_FUSED_MV ? 2 : 1) * 2 * K * kNT * sizeof(double);
}

int grid_for(KernelFn fn, int C, size_t smem) {
  static std::mutex mu;
  static std::vector<std::pair<KernelFn, int>> cache;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : cache)
    if (e.first == fn) return e.second;
  int grid = 0;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (C == 1) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kNT, smem) != cudaSuccess || per_sm < 1)
      per_sm = 1;
    grid = per_sm * SIMOPT_NUM_SMS;
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C * SIMOPT_NUM_SMS);
    cfg.blockDim = dim3(kNT);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = C;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg) != cudaSuccess || ncl < 1) {
      cudaGetLastError();
      ncl = SIMOPT_NUM_SMS / C;
    }
    grid = ncl * C;
  }
  cache.emplace_back(fn, grid);
  return grid;
}

}  // namespace

extern "C" int simopt_fused_rows(void* stream, int mode, const double* X, int64_t rows, int64_t cols,
                                 const double* v, const double* center, const double* rowaux,
                                 double col_scale, int accumulate, int raw, double* t_out,
                                 double* dw_out, double* col_out, double* scalar_out) {
  cudaStream_t st = as_stream(stream);
  SIMOPT_REQUIRE(mode == SIMOPT_FUSED_MV || mode == SIMOPT_FUSED_LR_GRAD || mode == SIMOPT_FUSED_LR_HVP,
                 SIMOPT_E_CONFIG, "unknown fused mode %d", mode);
  SIMOPT_REQUIRE(rows >= 0 && cols >= 0, SIMOPT_E_DIMENSION, "negative extent");
  SIMOPT_REQUIRE(mode != SIMOPT_FUSED_MV || center != nullptr, SIMOPT_E_CONFIG, "MV needs the mean");
  SIMOPT_REQUIRE(mode == SIMOPT_FUSED_MV || rowaux != nullptr, SIMOPT_E_CONFIG, "row weights missing");
  if (cols == 0 || rows == 0) {  // empty sums: col_out = 0 * scale [- center], scalar 0
    k_fused_finish<<<(int)(cols > 0 ? ceil_div(cols, 32) : 1), 256, 0, st>>>(
        nullptr, nullptr, 0, cols, col_scale, (mode == SIMOPT_FUSED_MV && !raw) ? center : nullptr,
        (accumulate && cols) ? col_out : nullptr, scalar_out);
    SIMOPT_CHECK_LAUNCH("k_fused_finish");
    return SIMOPT_OK;
  }
  int C = 1, K = 1;
  SIMOPT_REQUIRE(geometry(cols, &C, &K), SIMOPT_E_CONFIG,
                 "fused pass supports up to %d columns (got %lld)", 8 * 8 * 2 * kNT, (long long)cols);
  const bool vec = (cols % 2 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  KernelFn fn = pick(mode, C, K, vec);
  const int grid = grid_for(fn, C, dyn_smem(mode, K));
  const int64_t ncl = grid / C;
  double* part = static_cast<double*>(simopt_scratch(st, (ncl * cols + ncl) * sizeof(double)));
  SIMOPT_REQUIRE(part != nullptr, SIMOPT_E_CUDA, "%s", simopt_last_error());
  FusedArgs a;
  a.X = X;
  a.N = rows;
  a.d = cols;
  a.v = v;
  a.mean = center;
  a.rowaux = rowaux;
  a.t_out = t_out;
  a.dw_out = dw_out;
  a.col_part = part;
  a.scal_part = part + ncl * cols;
  a.accumulate = (accumulate && col_out) ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kNT);
  cfg.stream = st;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = C;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  cfg.dynamicSmemBytes = dyn_smem(mode, K);
  SIMOPT_CUDA(cudaLaunchKernelEx(&cfg, fn, a));
  const int fgrid = (int)(a.accumulate ? ceil_div(cols, 32) : 1);
  k_fused_finish<<<fgrid < 1 ? 1 : fgrid, 256, 0, st>>>(
      part, a.scal_part, ncl, cols, raw ? 1.0 : col_scale,
      (mode == SIMOPT_FUSED_MV && !raw) ? center : nullptr, a.accumulate ? col_out : nullptr,
      scalar_out);
  SIMOPT_CHECK_LAUNCH("k_fused_finish");
  return SIMOPT_OK;
}
