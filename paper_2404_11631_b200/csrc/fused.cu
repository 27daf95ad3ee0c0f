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
#include <stdlib.h>

#include <algorithm>

#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"
#include "fw.cuh"
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

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t peer_addr(uint32_t local, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}

// Wide rows (C > 1): ASYNC exchanges each tile's per-CTA row-dot partials by pushing them
// into every peer's receive slots with st.async (DSMEM) completing on the peer's mbarrier,
// instead of a cluster-wide barrier per tile; a CTA waits only for its peers' partials of
// the tile it is on.  Slots and barriers are double-buffered by tile parity: a CTA can be
// at most one tile ahead of its slowest peer (each tile needs every peer's previous one).
template <int MODE, int C, int K, bool VEC, bool ASYNC = false>
__global__ void __launch_bounds__(kNT, 2) k_fused_rows(FusedArgs a) {
  constexpr int R = (16 / K) < 1 ? 1 : 16 / K;
  extern __shared__ __align__(16) double vs[];  // [band] v, then [band] mean (MV)
  __shared__ double red[2][R][kNW];
  __shared__ double part[2][R];
  __shared__ double wts[2][R];
  __shared__ double sred[kNW];
  __shared__ __align__(8) double rcv[2][C][R];  // ASYNC: partials pushed by every peer
  __shared__ __align__(8) uint64_t rbar[2];     // ASYNC: full barriers of rcv[par]
  const int tid = threadIdx.x;
  int rank = 0;
  if constexpr (C > 1) rank = (int)cg::this_cluster().block_rank();
  if constexpr (ASYNC) {
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&rbar[0])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&rbar[1])));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cg::this_cluster().sync();  // peers' barriers initialised before the first push
  }
  uint32_t phase = 0;  // ASYNC: bit par = the parity of rbar[par]'s current phase
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
  for (int64_t tile = cl; tile < ntiles; tile += ncl, par ^= 1) {
    const int64_t r0 = tile * R;
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
    if constexpr (ASYNC) {
      if (tid == 0)  // this phase completes once all C*R partials have landed
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&rbar[par])),
                     "r"((uint32_t)(C * R * sizeof(double))) : "memory");
      if (tid < R) {
        const double pv = part[par][tid];
        const uint32_t la = smem_addr(&rcv[par][rank][tid]), lb = smem_addr(&rbar[par]);
#pragma unroll
        for (int q = 0; q < C; ++q)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(
                           peer_addr(la, q)),
                       "l"(__double_as_longlong(pv)), "r"(peer_addr(lb, q))
                       : "memory");
      }
      // MV in 8-CTA clusters: every thread waits for the tile's partials and forms the R row
      // weights itself (wt = t), so no block barrier is needed before the accumulation
      // (C4, d = 2e4: 6.00 -> 6.25 TB/s); otherwise the R owner threads wait and publish the
      // weights through shared memory
      constexpr bool kAllWait = MODE == SIMOPT_FUSED_MV && C >= 8;
      if (kAllWait || tid < R) {
        const uint32_t want = (phase >> par) & 1u;
        asm volatile(
            "{\n\t.reg .pred P1;\n"
            "WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
            "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_addr(&rbar[par])),
            "r"(want)
            : "memory");
      }
      phase ^= 1u << par;
      if constexpr (kAllWait) {
        double wv[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
          double t = 0.0;
#pragma unroll
          for (int q = 0; q < C; ++q) t += rcv[par][q][i];
          const bool rv = r0 + i < N;
          wv[i] = rv ? t : 0.0;
          if (tid == i && rv) {
            sc = fma(t, t, sc);
            if (rank == 0 && a.t_out) a.t_out[r0 + i] = t;
          }
        }
        if (a.accumulate) {
#pragma unroll
          for (int i = 0; i < R; ++i) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
              acc[k].x = fma(x[i][k].x, wv[i], acc[k].x);
              acc[k].y = fma(x[i][k].y, wv[i], acc[k].y);
            }
          }
        }
        continue;  // next tile
      }
    } else if constexpr (C > 1) {
      cg::this_cluster().sync();
    } else {
      __syncthreads();
    }
    if (tid < R) {
      double t = 0.0;
      if constexpr (ASYNC) {
#pragma unroll
        for (int q = 0; q < C; ++q) t += rcv[par][q][tid];
      } else if constexpr (C > 1) {
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
#pragma unroll 8
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
  if (scalar_out && blockIdx.x == 0) {  // block-parallel, fixed order: deterministic
    __shared__ double ws[8];
    double s = 0.0;
    for (int64_t c = threadIdx.x; c < ncl; c += 256) s += spart[c];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) ws[w] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int k = 0; k < 8; ++k) t += ws[k];
      *scalar_out = t;
    }
  }
}

// ---------------------------------------------------------------------------
// Persistent mean-variance FW epoch (fused mode, one GPU, d <= 2*K*256 in one CTA band).
// At C1's size (N = 10^4 rows x d = 10^3, 80 MB, L2-resident) a step is ~15 us of work
// split over a pass, a fold and a tail: as separate launches it is launch- and
// latency-bound (~44 us per step).  One cooperative launch runs the epoch's M+1 passes
// with two grid barriers per step:
//   pass (all CTAs, rows striped by tile as in k_fused_rows): q = Xc w, per-CTA column
//        partials of Xc^T q and the partial |q|^2  -> barrier
//   fold (columns split over CTAs, a warp per column, lane-strided over the CTA partials
//        then a fixed xor tree; CTA 0 folds |q|^2): g = inv * sum - mean, quad  -> barrier
//   tail (every CTA, redundantly: g is 8-16 KB in L2): NaN check, argmin (lmo.py:56-65),
//        w' = (gamma * ((-1 * w) + s)) + w straight into the CTA's shared v for the next
//        pass; CTA 0 also writes the ring row, min, the block-parallel sum / dot and the
//        step's %globaltimer stamp.
// Summation orders are fixed (deterministic run to run); like every fused pass they are
// not the reference tree (trajectories within the north-star 1e-8).
struct MvEpochArgs {
  const double* X;
  int64_t N, d;
  const double* mean;
  double inv;          // 1 / (N - 1)
  double* ring;        // (M+1) x d: row 0 = the epoch's first iterate, rows 1..M written
  int64_t M;
  const double* gamma;  // M step sizes
  int* status;          // M
  double *wmin, *wsum, *lin, *quad;  // M each
  int64_t* stamps;      // M
  double* col_part;     // [G][d]
  double* scal_part;    // [G]
  double* g;            // d
  unsigned* bar;        // grid barrier counter, zero at launch
};

__device__ __forceinline__ void mv_grid_sync(unsigned* bar, unsigned& target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += gridDim.x;
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// Between two passes (both epoch kernels): barrier, fold the CTA partials into g (columns
// split over CTAs, a warp per column lane-strided over the partials then an xor tree; CTA 0
// folds |q|^2 into quad[it-1]), barrier, then every CTA runs step it's tail: NaN check,
// argmin (lmo.py:56-65), w' = (gamma * ((-1 * w) + s)) + w into vs[0..d); CTA 0 writes the
// ring row, min, the block-parallel sum / dot and the step's %globaltimer stamp.  Returns
// false after the last pass (it == M).
__device__ __noinline__ bool mv_epoch_fold_tail(const MvEpochArgs& a, int64_t it, bool cols,
                                                double* vs, const double* ms, unsigned& target) {
  __shared__ ArgMin wb[32];
  __shared__ double wm[32], rs[32], rd[32];
  __shared__ int nan_seen;
  __shared__ int64_t js_sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int64_t d = a.d, G = gridDim.x, cta = blockIdx.x;
  mv_grid_sync(a.bar, target);
  const int64_t cpc = (d + G - 1) / G;
  const int64_t c0 = cta * cpc;
  for (int64_t j = c0 + warp; cols && j < c0 + cpc && j < d; j += nw) {
    double t = 0.0;
    for (int64_t c = lane; c < G; c += 32) t += __ldcg(a.col_part + c * d + j);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) a.g[j] = t * a.inv - ms[j];
  }
  if (cta == 0 && it > 0 && warp == nw - 1) {
    double t = 0.0;
    for (int64_t c = lane; c < G; c += 32) t += __ldcg(a.scal_part + c);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) a.quad[it - 1] = t;
  }
  if (it == a.M) return false;
  mv_grid_sync(a.bar, target);
  if (tid == 0) nan_seen = 0;
  __syncthreads();
  ArgMin b{INFINITY, INT64_MAX};
  for (int64_t i = tid; i < d; i += blockDim.x) {
    const double gi = __ldcg(a.g + i);
    if (gi != gi) nan_seen = 1;
    b = amin(b, ArgMin{gi, i});
  }
  b = warp_amin(b);
  if (lane == 0) wb[warp] = b;
  __syncthreads();
  if (tid == 0) {
    ArgMin r = wb[0];
    for (int w = 1; w < nw; ++w) r = amin(r, wb[w]);
    if (cta == 0 && nan_seen) atomicOr(a.status + it, SIMOPT_E_INVALID_GRADIENT);
    js_sh = (r.i < d && __ldcg(a.g + r.i) < 0.0) ? r.i : -1;  // vertex e_j* iff g_j* < 0
  }
  __syncthreads();
  const int64_t js = js_sh;
  const double gm = a.gamma[it];
  double mn = INFINITY, ps = 0.0, pd = 0.0;
  for (int64_t i = tid; i < d; i += blockDim.x) {
    const double wi = vs[i];
    const double si = (i == js) ? 1.0 : 0.0;
    const double dir = -1.0 * wi + si;
    const double wo = gm * dir + wi;
    vs[i] = wo;
    if (cta == 0) {
      a.ring[(it + 1) * d + i] = wo;
      ps += wo;
      pd += wo * ms[i];
      mn = (wo < mn || wo != wo) ? wo : mn;
    }
  }
  if (cta == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ps += __shfl_xor_sync(0xffffffffu, ps, o);
      pd += __shfl_xor_sync(0xffffffffu, pd, o);
      const double t = __shfl_xor_sync(0xffffffffu, mn, o);
      mn = (t < mn || t != t) ? t : mn;
    }
    if (lane == 0) {
      rs[warp] = ps;
      rd[warp] = pd;
      wm[warp] = mn;
    }
  }
  __syncthreads();  // vs holds w_{it+1} for the next pass
  if (cta == 0 && tid == 0) {
    double sa = 0.0, sb = 0.0, m = wm[0];
    for (int w = 0; w < nw; ++w) {
      sa += rs[w];
      sb += rd[w];
      if (w > 0) m = (wm[w] < m || wm[w] != wm[w]) ? wm[w] : m;
    }
    a.wsum[it] = sa;
    a.lin[it] = sb;
    a.wmin[it] = m;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.stamps[it] = (int64_t)t;
  }
  return true;
}

// Warp-per-row variant (d <= 1024): lane l holds columns 2(l + 32k), k < KW, of one row at
// a time, so a row dot is one warp's xor tree (no block barrier per tile) and the column
// accumulators stay per warp; a pass ends with the warps' partials combined in warp order
// through shared memory.  ~4.5 instructions per element instead of ~12 for the CTA-per-row
// tiles at C1's d = 1000.
template <int KW, bool VEC>
__global__ void __launch_bounds__(kNT, 1) k_mv_fw_epoch_wr(MvEpochArgs a) {
  constexpr int CW = 64 * KW;  // columns covered
  extern __shared__ __align__(16) double smw[];
  double* vs = smw;            // [CW] w (the pass's v)
  double* ms = smw + CW;       // [CW] mean
  double* wp = smw + 2 * CW;   // [kNW][CW] per-warp column partials
  __shared__ double wsc[kNW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t d = a.d, N = a.N, G = gridDim.x, cta = blockIdx.x;
  for (int i = tid; i < CW; i += kNT) {
    vs[i] = i < d ? a.ring[i] : 0.0;
    ms[i] = i < d ? a.mean[i] : 0.0;
  }
  __syncthreads();
  const double2* v2 = reinterpret_cast<const double2*>(vs);
  const double2* m2 = reinterpret_cast<const double2*>(ms);
  const int64_t gw = cta * kNW + warp, nwg = G * kNW;
  unsigned target = 0;
  for (int64_t it = 0; it <= a.M; ++it) {
    const bool cols = it < a.M;
    double2 acc[KW];
#pragma unroll
    for (int k = 0; k < KW; ++k) acc[k] = make_double2(0.0, 0.0);
    double sc = 0.0;
    for (int64_t r = gw; r < N; r += nwg) {
      const double* row = a.X + r * d;
      double2 x[KW];
#pragma unroll
      for (int k = 0; k < KW; ++k) {
        const int64_t c = 2 * (int64_t)(lane + 32 * k);
        if (VEC) {
          x[k] = c < d ? ld2(row + c) : make_double2(0.0, 0.0);
        } else {
          x[k].x = c < d ? __ldg(row + c) : 0.0;
          x[k].y = c + 1 < d ? __ldg(row + c + 1) : 0.0;
        }
      }
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < KW; ++k) {
        const double2 mk = m2[lane + 32 * k];
        const double2 vk = v2[lane + 32 * k];
        x[k].x = x[k].x - mk.x;  // Xc = X - mean (tasks.py:63); padded columns stay 0
        x[k].y = x[k].y - mk.y;
        t = fma(x[k].x, vk.x, t);
        t = fma(x[k].y, vk.y, t);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      sc = fma(t, t, sc);  // identical on every lane; lane 0's is used
      if (cols) {
#pragma unroll
        for (int k = 0; k < KW; ++k) {
          acc[k].x = fma(x[k].x, t, acc[k].x);
          acc[k].y = fma(x[k].y, t, acc[k].y);
        }
      }
    }
    if (cols) {
      double2* w2 = reinterpret_cast<double2*>(wp + warp * CW);
#pragma unroll
      for (int k = 0; k < KW; ++k) w2[lane + 32 * k] = acc[k];
    }
    if (lane == 0) wsc[warp] = sc;
    __syncthreads();
    if (cols) {
      for (int64_t c = tid; c < d; c += kNT) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < kNW; ++w) t += wp[w * CW + c];
        a.col_part[cta * d + c] = t;
      }
    }
    if (tid == 0) {
      double p = 0.0;
      for (int w = 0; w < kNW; ++w) p += wsc[w];
      a.scal_part[cta] = p;
    }
    if (!mv_epoch_fold_tail(a, it, cols, vs, ms, target)) break;
  }
}

template <int K, bool VEC>
__global__ void __launch_bounds__(kNT, 2) k_mv_fw_epoch(MvEpochArgs a) {
  constexpr int R = (16 / K) < 1 ? 1 : 16 / K;
  extern __shared__ __align__(16) double vs[];  // [2*K*256] w (the pass's v), then the mean
  __shared__ double red[2][R][kNW];
  __shared__ double part[2][R];
  __shared__ double wts[2][R];
  __shared__ double sred[kNW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t d = a.d, N = a.N, G = gridDim.x, cta = blockIdx.x;
  double* ms = vs + 2 * K * kNT;
  for (int i = tid; i < 2 * K * kNT; i += kNT) {
    vs[i] = i < d ? a.ring[i] : 0.0;
    ms[i] = i < d ? a.mean[i] : 0.0;
  }
  __syncthreads();
  const double2* v2 = reinterpret_cast<const double2*>(vs);
  const double2* m2 = reinterpret_cast<const double2*>(ms);
  unsigned target = 0;
  const int64_t ntiles = (N + R - 1) / R;
  for (int64_t it = 0; it <= a.M; ++it) {
    // ---- pass at w_it: columns for step it's gradient (it < M), |q|^2 for step it-1
    const bool cols = it < a.M;
    double2 acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = make_double2(0.0, 0.0);
    double sc = 0.0;
    int par = 0;
    for (int64_t tile = cta; tile < ntiles; tile += G, par ^= 1) {
      const int64_t r0 = tile * R;
      double2 x[R][K];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const bool rv = r0 + i < N;
        const double* row = a.X + (rv ? r0 + i : 0) * d;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int64_t c = 2 * (int64_t)(tid + k * kNT);
          if (VEC) {
            x[i][k] = (rv && c < d) ? ld2(row + c) : make_double2(0.0, 0.0);
          } else {
            x[i][k].x = (rv && c < d) ? __ldg(row + c) : 0.0;
            x[i][k].y = (rv && c + 1 < d) ? __ldg(row + c + 1) : 0.0;
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
          const double2 mk = m2[tid + k * kNT];
          x[i][k].x = x[i][k].x - mk.x;  // Xc = X - mean (tasks.py:63)
          x[i][k].y = x[i][k].y - mk.y;
          acc_s = fma(x[i][k].x, vk.x, acc_s);
          acc_s = fma(x[i][k].y, vk.y, acc_s);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc_s += __shfl_xor_sync(0xffffffffu, acc_s, o);
        s[i] = acc_s;
      }
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < R; ++i) red[par][i][warp] = s[i];
      }
      __syncthreads();
      if (tid < R) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < kNW; ++w) t += red[par][tid][w];
        const int64_t r = r0 + tid;
        double wt = 0.0;
        if (r < N) {
          wt = t;
          sc = fma(t, t, sc);
        }
        wts[par][tid] = wt;
      }
      __syncthreads();
      if (cols) {
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
    if (cols) {
      double* out = a.col_part + cta * d;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int64_t c = 2 * (int64_t)(tid + k * kNT);
        if (c < d) out[c] = acc[k].x;
        if (c + 1 < d) out[c + 1] = acc[k].y;
      }
    }
    {
      double v = sc;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) sred[warp] = v;
      __syncthreads();
      if (tid == 0) {
        double p = 0.0;
        for (int w = 0; w < kNW; ++w) p += sred[w];
        a.scal_part[cta] = p;
      }
    }
    if (!mv_epoch_fold_tail(a, it, cols, vs, ms, target)) break;
  }
}

// ---------------------------------------------------------------------------
// The same pass on bit-packed binary features (csrc/bits.cu layout, W = ceil(d/64)
// words per row): one read of N*W*8 bytes, 1/64 of the fp64 layout, so the pass is
// issue-bound and the work per element is what matters.
// Nibble-table variant for d <= 1024 (G = ceil(d/4) <= 256 four-column groups), one
// tile row per thread:
//   row dot     t_r = sum over the row's nibbles of T[c][p], T[c][p] = sum of v over the
//               set bits of pattern p in group c (built once per CTA; [G][16] layout: a
//               warp reads one 128-byte line per nibble step -- conflict-free);
//   accumulate  thread c owns group c's 16 pattern accumulators A[p][c] += wt_r over
//               the tile rows ([16][Gp] layout, Gp = 32k: conflict-free), expanded to
//               the four column sums once at the end.
// ~2.5 instructions per element instead of ~30 (per-bit loops); no atomics.
constexpr int kMaxNibG = kNT;

template <int MODE>
__global__ void __launch_bounds__(kNT) k_fused_nib(const uint64_t* __restrict__ bits, int64_t N,
                                                   int64_t d, int64_t W, int tpr,
                                                   const double* __restrict__ v,
                                                   const double* __restrict__ rowaux,
                                                   double* __restrict__ t_out,
                                                   double* __restrict__ dw_out,
                                                   double* __restrict__ col_part,
                                                   double* __restrict__ scal_part, int accumulate) {
  (void)tpr;
  extern __shared__ __align__(16) double dsm[];
  const int G = (int)((d + 3) >> 2);
  const int Gp = (G + 31) & ~31;
  const int WS = (int)W + 1;                    // padded row stride of the tile (u64 words)
  const int GT = 16 * (int)W;                   // table groups: whole words (zero past d)
  double* T = dsm;                              // [GT][16]
  double* A = T + 16 * GT;                      // [16][Gp]
  double* wts = A + 16 * Gp;                    // [kNT]
  uint64_t* tb = reinterpret_cast<uint64_t*>(wts + kNT);  // [kNT][WS]
  __shared__ double red[kNT / 32];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int e = tid; e < 16 * GT; e += kNT) {
    const int c = e >> 4, p = e & 15;
    double t = 0.0;
    for (int b = 0; b < 4; ++b) {
      const int64_t j = 4 * c + b;
      if (((p >> b) & 1) && j < d) t += v[j];
    }
    T[e] = t;
  }
  for (int e = tid; e < 16 * Gp; e += kNT) A[e] = 0.0;
  double sc = 0.0;
  const int64_t ntiles = (N + kNT - 1) / kNT;
  // the next tile's words are loaded into registers while this tile is processed
  // (coalesced: consecutive threads, consecutive words; W <= 16 words per row here)
  uint64_t pf[16];
  auto fetch = [&](int64_t tl) {
    const int64_t rb = tl * kNT;
    const int64_t nr = tl < ntiles ? (N - rb < kNT ? N - rb : kNT) : 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int e = tid + k * kNT, rr = e / (int)W, ww = e - rr * (int)W;
      pf[k] = (k < (int)W && rr < nr) ? __ldg(bits + (rb + rr) * W + ww) : 0ULL;
    }
  };
  fetch(blockIdx.x);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * kNT;
    const int64_t nrow = N - r0 < kNT ? N - r0 : kNT;
    __syncthreads();  // tables built / previous tile consumed
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int e = tid + k * kNT, rr = e / (int)W, ww = e - rr * (int)W;
      if (k < (int)W) tb[rr * WS + ww] = pf[k];
    }
    fetch(tile + gridDim.x);
    __syncthreads();
    // row dot: this thread's row, nibble by nibble
    const int64_t r = r0 + tid;
    const uint64_t* row = tb + tid * WS;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;  // 4 chains: latency, not issue, bound
    for (int ww = 0; ww < (int)W; ++ww) {
      const uint64_t m = row[ww];
      const double* Tw = T + 16 * 16 * ww;
#pragma unroll
      for (int i = 0; i < 16; i += 4) {
        s0 += Tw[16 * i + (int)((m >> (4 * i)) & 15ULL)];
        s1 += Tw[16 * (i + 1) + (int)((m >> (4 * i + 4)) & 15ULL)];
        s2 += Tw[16 * (i + 2) + (int)((m >> (4 * i + 8)) & 15ULL)];
        s3 += Tw[16 * (i + 3) + (int)((m >> (4 * i + 12)) & 15ULL)];
      }
    }
    const double s = (s0 + s1) + (s2 + s3);
    double wt = 0.0;
    if (r < N) {
      const double t = s;
      if (MODE == SIMOPT_FUSED_LR_GRAD) {
        const double z = rowaux[r];
        const double c = dev_sigmoid(t);
        wt = c - z;
        if (dw_out) dw_out[r] = c * (1.0 - c);
        sc += glibc_logistic_loss_term(t, z, simopt_exptab_dev);
      } else {
        wt = rowaux[r] * t;
      }
      if (t_out) t_out[r] = t;
    }
    wts[tid] = wt;
    __syncthreads();
    if (accumulate && tid < G) {
      // four rows per step: their four accumulators are loaded before any is stored, and
      // a pattern repeated within the step continues from the latest earlier sum -- the
      // same additions in the same order as one row at a time, but one shared-memory
      // round trip per four rows instead of a load-add-store chain per row
      const int c = tid, word = c >> 4, sh = 4 * (c & 15);
      double* Ac = A + c;
      const int nr = (int)nrow;
      int i = 0;
      for (; i + 4 <= nr; i += 4) {
        const int p0 = (int)((tb[i * WS + word] >> sh) & 15ULL);
        const int p1 = (int)((tb[(i + 1) * WS + word] >> sh) & 15ULL);
        const int p2 = (int)((tb[(i + 2) * WS + word] >> sh) & 15ULL);
        const int p3 = (int)((tb[(i + 3) * WS + word] >> sh) & 15ULL);
        const double2 wa = *reinterpret_cast<const double2*>(wts + i);
        const double2 wb = *reinterpret_cast<const double2*>(wts + i + 2);
        const double a0 = Ac[p0 * Gp], a1 = Ac[p1 * Gp], a2 = Ac[p2 * Gp], a3 = Ac[p3 * Gp];
        const double s0 = a0 + wa.x;
        const double s1 = (p1 == p0 ? s0 : a1) + wa.y;
        const double s2 = (p2 == p1 ? s1 : (p2 == p0 ? s0 : a2)) + wb.x;
        const double s3 = (p3 == p2 ? s2 : (p3 == p1 ? s1 : (p3 == p0 ? s0 : a3))) + wb.y;
        Ac[p0 * Gp] = s0;  // in row order: a repeated pattern's last store holds its sum
        Ac[p1 * Gp] = s1;
        Ac[p2 * Gp] = s2;
        Ac[p3 * Gp] = s3;
      }
      for (; i < nr; ++i) {
        const int p = (int)((tb[i * WS + word] >> sh) & 15ULL);
        Ac[p * Gp] += wts[i];
      }
    }
  }
  if (accumulate) {
    __syncthreads();
    double* out = col_part + blockIdx.x * d;
    for (int c = tid; c < G; c += kNT) {
      double col[4] = {0.0, 0.0, 0.0, 0.0};
      for (int p = 1; p < 16; ++p) {
        const double ap = A[p * Gp + c];
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if ((p >> b) & 1) col[b] += ap;
      }
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (4 * c + b < d) out[4 * c + b] = col[b];
    }
  }
  for (int o = 16; o > 0; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
  __syncthreads();
  if (lane == 0) red[tid >> 5] = sc;
  __syncthreads();
  if (tid == 0) {
    double p = 0.0;
    for (int q = 0; q < kNT / 32; ++q) p += red[q];
    scal_part[blockIdx.x] = p;
  }
}

// ---------------------------------------------------------------------------
// Banded nibble-table pass for d > 1024 (C5: d = 8192): the nibble tables of all of d do
// not fit one CTA, so the pass splits into 1024-column bands (16 words) and two sweeps of
// the bits (1/64 of the fp64 bytes each -- the sweeps are issue-bound, not HBM-bound):
//   k_nibb_rowdot  grid (x, band): band partial row dots via the band's nibble tables
//   k_nibb_rowfin  per row: t = sum of the band partials in band order, the epilogue
//                  (weight, c(1-c), loss term, t) as k_fused_nib
//   k_nibb_colsum  grid (x, band): the band's pattern accumulators A[p][c] += wt_r,
//                  expanded to column sums per CTA (col_part[x][band columns])
// and the usual finish kernel folds col_part over x.  ~3 instructions per element
// against ~32 for a per-bit walk (the earlier kernel at this width, 13x slower).
constexpr int kBandW = 16;                    // words per band (1024 columns)
constexpr int kBandWS = kBandW + 1;           // padded tile row stride (u64 words)

__device__ __forceinline__ void nibb_fetch(uint64_t (&pf)[kBandW], const uint64_t* __restrict__ bits,
                                           int64_t N, int64_t W, int64_t w0, int64_t tl,
                                           int64_t ntiles) {
  const int64_t rb = tl * kNT;
  const int64_t nr = tl < ntiles ? (N - rb < kNT ? N - rb : kNT) : 0;
#pragma unroll
  for (int k = 0; k < kBandW; ++k) {
    const int e = threadIdx.x + k * kNT, rr = e >> 4, ww = e & 15;
    pf[k] = (rr < nr && w0 + ww < W) ? __ldg(bits + (rb + rr) * W + w0 + ww) : 0ULL;
  }
}

__global__ void __launch_bounds__(kNT) k_nibb_rowdot(const uint64_t* __restrict__ bits, int64_t N,
                                                     int64_t d, int64_t W,
                                                     const double* __restrict__ v,
                                                     double* __restrict__ part) {
  extern __shared__ __align__(16) double dsm[];
  double* T = dsm;                                            // [16 words][16 groups][16]
  uint64_t* tb = reinterpret_cast<uint64_t*>(T + kBandW * 256);  // [kNT][kBandWS]
  const int tid = threadIdx.x, band = blockIdx.y;
  const int64_t w0 = (int64_t)band * kBandW;
  for (int e = tid; e < kBandW * 256; e += kNT) {
    const int c = e >> 4, p = e & 15;  // group c of the band: columns 64 w0 + 4c ..
    double t = 0.0;
    for (int b = 0; b < 4; ++b) {
      const int64_t j = 64 * w0 + 4 * c + b;
      if (((p >> b) & 1) && j < d) t += v[j];
    }
    T[e] = t;
  }
  const int64_t ntiles = (N + kNT - 1) / kNT;
  uint64_t pf[kBandW];
  nibb_fetch(pf, bits, N, W, w0, blockIdx.x, ntiles);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kBandW; ++k) {
      const int e = tid + k * kNT;
      tb[(e >> 4) * kBandWS + (e & 15)] = pf[k];
    }
    nibb_fetch(pf, bits, N, W, w0, tile + gridDim.x, ntiles);
    __syncthreads();
    const int64_t r = tile * kNT + tid;
    const uint64_t* row = tb + tid * kBandWS;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll 4
    for (int ww = 0; ww < kBandW; ++ww) {
      const uint64_t m = row[ww];
      const double* Tw = T + 256 * ww;
#pragma unroll
      for (int i = 0; i < 16; i += 4) {
        s0 += Tw[16 * i + (int)((m >> (4 * i)) & 15ULL)];
        s1 += Tw[16 * (i + 1) + (int)((m >> (4 * i + 4)) & 15ULL)];
        s2 += Tw[16 * (i + 2) + (int)((m >> (4 * i + 8)) & 15ULL)];
        s3 += Tw[16 * (i + 3) + (int)((m >> (4 * i + 12)) & 15ULL)];
      }
    }
    if (r < N) part[(int64_t)band * N + r] = (s0 + s1) + (s2 + s3);
  }
}

template <int MODE>
__global__ void __launch_bounds__(kNT) k_nibb_rowfin(const double* __restrict__ part, int64_t N,
                                                     int nb, const double* __restrict__ rowaux,
                                                     double* __restrict__ wt_out,
                                                     double* __restrict__ t_out,
                                                     double* __restrict__ dw_out,
                                                     double* __restrict__ scal_part) {
  __shared__ double red[kNT / 32];
  double sc = 0.0;
  for (int64_t r = blockIdx.x * (int64_t)kNT + threadIdx.x; r < N; r += (int64_t)gridDim.x * kNT) {
    double t = 0.0;
    for (int b = 0; b < nb; ++b) t += part[(int64_t)b * N + r];
    double wt;
    if (MODE == SIMOPT_FUSED_LR_GRAD) {
      const double z = rowaux[r];
      const double c = dev_sigmoid(t);
      wt = c - z;
      if (dw_out) dw_out[r] = c * (1.0 - c);
      sc += glibc_logistic_loss_term(t, z, simopt_exptab_dev);
    } else {
      wt = rowaux[r] * t;
    }
    if (t_out) t_out[r] = t;
    wt_out[r] = wt;
  }
  const int lane = threadIdx.x & 31;
  for (int o = 16; o > 0; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
  if (lane == 0) red[threadIdx.x >> 5] = sc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double p = 0.0;
    for (int q = 0; q < kNT / 32; ++q) p += red[q];
    scal_part[blockIdx.x] = p;
  }
}

__global__ void __launch_bounds__(kNT) k_nibb_colsum(const uint64_t* __restrict__ bits, int64_t N,
                                                     int64_t d, int64_t W,
                                                     const double* __restrict__ wt,
                                                     double* __restrict__ col_part) {
  extern __shared__ __align__(16) double dsm[];
  double* A = dsm;                                           // [16][kNT]
  double* wts = A + 16 * kNT;                                // [kNT]
  uint64_t* tb = reinterpret_cast<uint64_t*>(wts + kNT);     // [kNT][kBandWS]
  const int tid = threadIdx.x, band = blockIdx.y;
  const int64_t w0 = (int64_t)band * kBandW;
  for (int e = tid; e < 16 * kNT; e += kNT) A[e] = 0.0;
  const int64_t ntiles = (N + kNT - 1) / kNT;
  uint64_t pf[kBandW];
  nibb_fetch(pf, bits, N, W, w0, blockIdx.x, ntiles);
  const int word = tid >> 4, sh = 4 * (tid & 15);  // this thread's group: 4 columns
  double* Ac = A + tid;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * kNT;
    const int nrow = (int)(N - r0 < kNT ? N - r0 : kNT);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kBandW; ++k) {
      const int e = tid + k * kNT;
      tb[(e >> 4) * kBandWS + (e & 15)] = pf[k];
    }
    wts[tid] = tid < nrow ? wt[r0 + tid] : 0.0;
    nibb_fetch(pf, bits, N, W, w0, tile + gridDim.x, ntiles);
    __syncthreads();
    for (int i = 0; i < nrow; ++i) {
      const int p = (int)((tb[i * kBandWS + word] >> sh) & 15ULL);
      Ac[p * kNT] += wts[i];
    }
  }
  __syncthreads();
  double col[4] = {0.0, 0.0, 0.0, 0.0};
  for (int p = 1; p < 16; ++p) {
    const double ap = A[p * kNT + tid];
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if ((p >> b) & 1) col[b] += ap;
  }
  double* out = col_part + blockIdx.x * d;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int64_t j = 64 * w0 + 4 * tid + b;
    if (j < d) out[j] = col[b];
  }
}

using BitsFn = void (*)(const uint64_t*, int64_t, int64_t, int64_t, int, const double*,
                        const double*, double*, double*, double*, double*, int);

// Cross-rank finish over peer memory (SimoptPeerReduce).  kFB blocks (a layout
// constant of the flag area, the same on every rank), all resident at 256 threads
// on any sm_100 part, so the spin waits cannot starve a block another rank waits for.
constexpr int kFB = 148;

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(256) k_fused_finish_peer(const double* __restrict__ part,
                                                           const double* __restrict__ spart,
                                                           int64_t ncl, int64_t d, double scale,
                                                           const double* __restrict__ center,
                                                           double* __restrict__ out,
                                                           double* __restrict__ scalar_out,
                                                           SimoptPeerReduce pr) {
  const int64_t W = pr.world, D1 = d + 1, par = (int64_t)(pr.seq & 1ULL);
  const int b = blockIdx.x, tid = threadIdx.x;
  // layout of every rank's buffer: data [2][W][d+1] doubles, then flags [2][W][kFB] u64
  auto data = [&](int64_t q) { return reinterpret_cast<double*>(pr.peers[q]); };
  auto flags = [&](int64_t q) { return reinterpret_cast<uint64_t*>(data(q) + 2 * W * D1); };
  const int64_t jlo = out ? 0 : d;  // row pass only: just the side scalar crosses ranks
  for (int64_t j = jlo + (int64_t)b * 256 + tid; j < d; j += (int64_t)kFB * 256) {
    double s = 0.0;
#pragma unroll 8
    for (int64_t c = 0; c < ncl; ++c) s += part[c * d + j];
    for (int64_t q = 0; q < W; ++q) data(q)[(par * W + pr.rank) * D1 + j] = s;
  }
  if (b == (int)((d - jlo) / 256 % kFB)) {  // the block that owns index d: side scalar, block-parallel
    __shared__ double ws[8];
    double s = 0.0;
    for (int64_t c = tid; c < ncl; c += 256) s += spart[c];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((tid & 31) == 0) ws[tid >> 5] = s;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int k = 0; k < 8; ++k) t += ws[k];
      for (int64_t q = 0; q < W; ++q) data(q)[(par * W + pr.rank) * D1 + d] = t;
    }
  }
  __threadfence_system();
  __syncthreads();
  if (tid == 0) {
    for (int64_t q = 0; q < W; ++q) st_release_sys(flags(q) + (par * W + pr.rank) * kFB + b, pr.seq);
    const uint64_t* mine = flags(pr.rank) + par * W * kFB;
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    bool failed = pr.status && *((volatile int*)pr.status) != 0;  // sticky: fail fast
    for (int64_t q = 0; q < W && !failed; ++q) {
      while (ld_acquire_sys(mine + q * kFB + b) != pr.seq) {
        uint64_t t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > 10000000000ULL) {
          if (pr.status) atomicExch(pr.status, 1);
          failed = true;
          break;
        }
      }
    }
  }
  __syncthreads();
  const double* mine = data(pr.rank) + par * W * D1;
  for (int64_t j = jlo + (int64_t)b * 256 + tid; j < D1; j += (int64_t)kFB * 256) {
    double t = 0.0;
    for (int64_t q = 0; q < W; ++q) t += __ldcv(mine + q * D1 + j);  // rank order: same bits everywhere
    if (j < d) {
      if (out) {
        t = t * scale;
        out[j] = center ? t - center[j] : t;
      }
    } else if (scalar_out) {
      *scalar_out = t;
    }
  }
}

int finish(cudaStream_t st, const double* part, const double* spart, int64_t ncl, int64_t d,
           double scale, const double* center, double* out, double* scalar_out,
           const SimoptPeerReduce* peer) {
  if (peer == nullptr) {
    const int fgrid = (int)(out ? ceil_div(d, 32) : 1);
    k_fused_finish<<<fgrid < 1 ? 1 : fgrid, 256, 0, st>>>(part, spart, ncl, d, scale, center, out,
                                                         scalar_out);
    SIMOPT_CHECK_LAUNCH("k_fused_finish");
  } else {
    k_fused_finish_peer<<<kFB, 256, 0, st>>>(part, spart, ncl, d, scale, center, out, scalar_out, *peer);
    SIMOPT_CHECK_LAUNCH("k_fused_finish_peer");
  }
  return SIMOPT_OK;
}

using KernelFn = void (*)(FusedArgs);

template <int MODE, int C, int K>
KernelFn pick_vec(bool vec) {
  if constexpr (C >= 8) {  // measured: 8-CTA clusters gain (5.45 -> 6.26 TB/s at d = 2e4),
                           // 4-CTA clusters lose (4.58 -> 4.3 TB/s at d = 1e4)
    const char* ev = getenv("SIMOPT_FUSED_ASYNC");
    if (!(ev && atoi(ev) == 0))
      return vec ? k_fused_rows<MODE, C, K, true, true> : k_fused_rows<MODE, C, K, false, true>;
  }
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
                                 double* dw_out, double* col_out, double* scalar_out,
                                 const SimoptPeerReduce* peer) {
  cudaStream_t st = as_stream(stream);
  SIMOPT_REQUIRE(mode == SIMOPT_FUSED_MV || mode == SIMOPT_FUSED_LR_GRAD || mode == SIMOPT_FUSED_LR_HVP,
                 SIMOPT_E_CONFIG, "unknown fused mode %d", mode);
  SIMOPT_REQUIRE(rows >= 0 && cols >= 0, SIMOPT_E_DIMENSION, "negative extent");
  SIMOPT_REQUIRE(mode != SIMOPT_FUSED_MV || center != nullptr, SIMOPT_E_CONFIG, "MV needs the mean");
  if (cols == 0 || rows == 0)  // empty local sums: col_out = 0 * scale [- center], scalar 0
    return finish(st, nullptr, nullptr, 0, cols, col_scale,
                  (mode == SIMOPT_FUSED_MV && !raw) ? center : nullptr,
                  (accumulate && cols) ? col_out : nullptr, scalar_out, peer);
  SIMOPT_REQUIRE(mode == SIMOPT_FUSED_MV || rowaux != nullptr, SIMOPT_E_CONFIG, "row weights missing");
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
  return finish(st, part, a.scal_part, ncl, cols, raw ? 1.0 : col_scale,
                (mode == SIMOPT_FUSED_MV && !raw) ? center : nullptr,
                a.accumulate ? col_out : nullptr, scalar_out, peer);
}

extern "C" int simopt_fused_geometry(int mode, int64_t cols, int vec, int* cluster, int* clusters,
                                     int* grid) {
  SIMOPT_REQUIRE(mode == SIMOPT_FUSED_MV || mode == SIMOPT_FUSED_LR_GRAD || mode == SIMOPT_FUSED_LR_HVP,
                 SIMOPT_E_CONFIG, "unknown fused mode %d", mode);
  int C = 1, K = 1;
  SIMOPT_REQUIRE(cols >= 1 && geometry(cols, &C, &K), SIMOPT_E_CONFIG, "unsupported column count %lld",
                 (long long)cols);
  const int g = grid_for(pick(mode, C, K, vec != 0), C, dyn_smem(mode, K));
  if (cluster) *cluster = C;
  if (clusters) *clusters = g / C;
  if (grid) *grid = g;
  return SIMOPT_OK;
}

extern "C" int simopt_fused_rows_bits(void* stream, int mode, const uint64_t* bits, int64_t rows,
                                      int64_t cols, const double* v, const double* rowaux,
                                      double col_scale, int accumulate, int raw, double* t_out,
                                      double* dw_out, double* col_out, double* scalar_out,
                                      const SimoptPeerReduce* peer) {
  cudaStream_t st = as_stream(stream);
  SIMOPT_REQUIRE(mode == SIMOPT_FUSED_LR_GRAD || mode == SIMOPT_FUSED_LR_HVP, SIMOPT_E_CONFIG,
                 "bit-packed fused pass: logistic modes only (got %d)", mode);
  SIMOPT_REQUIRE(rows >= 0 && cols >= 0, SIMOPT_E_DIMENSION, "negative extent");
  SIMOPT_REQUIRE(cols <= 64 * kNT, SIMOPT_E_CONFIG, "bit-packed fused pass supports d <= %d", 64 * kNT);
  if (cols == 0 || rows == 0)  // an empty row shard still joins the cross-rank sums
    return finish(st, nullptr, nullptr, 0, cols, col_scale, nullptr,
                  (accumulate && cols) ? col_out : nullptr, scalar_out, peer);
  SIMOPT_REQUIRE(rowaux != nullptr, SIMOPT_E_CONFIG, "row weights missing");
  const int64_t W = ceil_div(cols, 64);
  if (ceil_div(cols, 4) > kMaxNibG) {  // banded nibble-table sweeps (d > 1024)
    const int nb = (int)ceil_div(W, kBandW);
    const size_t smem_r = (size_t)(kBandW * 256) * sizeof(double) + (size_t)kNT * kBandWS * 8;
    const size_t smem_c = (size_t)(17 * kNT) * sizeof(double) + (size_t)kNT * kBandWS * 8;
    static int gx = 0;
    if (!gx) {
      SIMOPT_CUDA(cudaFuncSetAttribute(k_nibb_rowdot, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r));
      SIMOPT_CUDA(cudaFuncSetAttribute(k_nibb_colsum, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_c));
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_nibb_colsum, kNT, smem_c) != cudaSuccess ||
          per_sm < 1)
        per_sm = 1;
      gx = per_sm * SIMOPT_NUM_SMS;
    }
    const int gxb = (int)(gx / nb > 0 ? gx / nb : 1);   // x-blocks per band: one resident wave
    const int acc = (accumulate && col_out) ? 1 : 0;
    // scratch: band partials [nb][N] | row weights [N] | col_part [gxb][cols] | scal [gxb]
    double* part = static_cast<double*>(
        simopt_scratch(st, ((int64_t)nb * rows + rows + (int64_t)gxb * cols + gxb) * sizeof(double)));
    SIMOPT_REQUIRE(part != nullptr, SIMOPT_E_CUDA, "%s", simopt_last_error());
    double* wbuf = part + (int64_t)nb * rows;
    double* cpart = wbuf + rows;
    double* spart = cpart + (int64_t)gxb * cols;
    k_nibb_rowdot<<<dim3((unsigned)gxb, (unsigned)nb), kNT, smem_r, st>>>(bits, rows, cols, W, v, part);
    SIMOPT_CHECK_LAUNCH("k_nibb_rowdot");
    if (mode == SIMOPT_FUSED_LR_GRAD)
      k_nibb_rowfin<SIMOPT_FUSED_LR_GRAD><<<gxb, kNT, 0, st>>>(part, rows, nb, rowaux, wbuf, t_out, dw_out, spart);
    else
      k_nibb_rowfin<SIMOPT_FUSED_LR_HVP><<<gxb, kNT, 0, st>>>(part, rows, nb, rowaux, wbuf, t_out, nullptr, spart);
    SIMOPT_CHECK_LAUNCH("k_nibb_rowfin");
    if (acc) {
      k_nibb_colsum<<<dim3((unsigned)gxb, (unsigned)nb), kNT, smem_c, st>>>(bits, rows, cols, W, wbuf, cpart);
      SIMOPT_CHECK_LAUNCH("k_nibb_colsum");
    }
    return finish(st, cpart, spart, gxb, cols, raw ? 1.0 : col_scale, nullptr, acc ? col_out : nullptr,
                  scalar_out, peer);
  }
  BitsFn fn = mode == SIMOPT_FUSED_LR_GRAD ? k_fused_nib<SIMOPT_FUSED_LR_GRAD>
                                           : k_fused_nib<SIMOPT_FUSED_LR_HVP>;
  const int64_t G = ceil_div(cols, 4), Gp = (G + 31) & ~31LL;
  const size_t smem = (size_t)(16 * 16 * W + 16 * Gp + kNT + kNT * (W + 1)) * sizeof(double);
  static std::mutex mu;
  static std::vector<std::pair<std::pair<BitsFn, int64_t>, int>> grids;  // (fn, W) -> grid
  int grid = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    for (auto& e : grids)
      if (e.first.first == fn && e.first.second == W) grid = e.second;
    if (!grid) {
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kNT, smem) != cudaSuccess ||
          per_sm < 1)
        per_sm = 1;
      grid = per_sm * SIMOPT_NUM_SMS;
      grids.emplace_back(std::make_pair(fn, W), grid);
    }
  }
  double* part = static_cast<double*>(simopt_scratch(st, ((int64_t)grid * cols + grid) * sizeof(double)));
  SIMOPT_REQUIRE(part != nullptr, SIMOPT_E_CUDA, "%s", simopt_last_error());
  const int acc = (accumulate && col_out) ? 1 : 0;
  fn<<<grid, kNT, smem, st>>>(bits, rows, cols, W, 0, v, rowaux, t_out,
                              mode == SIMOPT_FUSED_LR_GRAD ? dw_out : nullptr, part,
                              part + (int64_t)grid * cols, acc);
  SIMOPT_CHECK_LAUNCH("k_fused_nib");
  return finish(st, part, part + (int64_t)grid * cols, grid, cols, raw ? 1.0 : col_scale, nullptr,
                acc ? col_out : nullptr, scalar_out, peer);
}

extern "C" int64_t simopt_peer_reduce_bytes(int64_t world, int64_t cols) {
  return (2 * world * (cols + 1)) * (int64_t)sizeof(double) + 2 * world * kFB * (int64_t)sizeof(uint64_t);
}

extern "C" int simopt_mv_fw_epoch(void* stream, const double* X, int64_t rows, int64_t cols,
                                  const double* mean, double inv, double* ring, int64_t M,
                                  const double* gamma, int* status, double* wmin, double* wsum,
                                  double* lin, double* quad, int64_t* stamps) {
  cudaStream_t st = as_stream(stream);
  SIMOPT_REQUIRE(rows >= 1 && cols >= 1 && M >= 1, SIMOPT_E_DIMENSION, "empty epoch");
  int K = (int)((cols + 2 * kNT - 1) / (2 * kNT));
  SIMOPT_REQUIRE(K <= 4, SIMOPT_E_CONFIG, "persistent epoch supports up to %d columns", 8 * kNT);
  if (K == 3) K = 4;
  const bool vec = (cols % 2 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  using Fn = void (*)(MvEpochArgs);
  Fn fn = K == 1 ? (vec ? k_mv_fw_epoch<1, true> : k_mv_fw_epoch<1, false>)
        : K == 2 ? (vec ? k_mv_fw_epoch<2, true> : k_mv_fw_epoch<2, false>)
                 : (vec ? k_mv_fw_epoch<4, true> : k_mv_fw_epoch<4, false>);
  size_t smem = (size_t)2 * 2 * K * kNT * sizeof(double);
  const char* wr_env = getenv("SIMOPT_MV_EPOCH_WR");
  if (cols <= 1024 && !(wr_env && atoi(wr_env) == 0)) {  // warp-per-row pass
    int kw = 1;
    while (64 * kw < cols) kw *= 2;
    fn = kw == 1 ? (vec ? k_mv_fw_epoch_wr<1, true> : k_mv_fw_epoch_wr<1, false>)
       : kw == 2 ? (vec ? k_mv_fw_epoch_wr<2, true> : k_mv_fw_epoch_wr<2, false>)
       : kw == 4 ? (vec ? k_mv_fw_epoch_wr<4, true> : k_mv_fw_epoch_wr<4, false>)
       : kw == 8 ? (vec ? k_mv_fw_epoch_wr<8, true> : k_mv_fw_epoch_wr<8, false>)
                 : (vec ? k_mv_fw_epoch_wr<16, true> : k_mv_fw_epoch_wr<16, false>);
    smem = (size_t)(2 + kNW) * 64 * kw * sizeof(double);
  }
  int per_sm = 0;
  SIMOPT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SIMOPT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kNT, smem));
  SIMOPT_REQUIRE(per_sm >= 1, SIMOPT_E_CONFIG, "persistent epoch kernel does not fit an SM");
  if (const char* ev = getenv("SIMOPT_MV_EPOCH_PER_SM")) per_sm = std::min(per_sm, std::max(1, atoi(ev)));
  const int64_t G = (int64_t)per_sm * SIMOPT_NUM_SMS;
  unsigned char* ws = static_cast<unsigned char*>(
      simopt_scratch(st, (G * cols + G + cols) * sizeof(double) + 64));
  SIMOPT_REQUIRE(ws != nullptr, SIMOPT_E_CUDA, "%s", simopt_last_error());
  MvEpochArgs a;
  a.X = X;
  a.N = rows;
  a.d = cols;
  a.mean = mean;
  a.inv = inv;
  a.ring = ring;
  a.M = M;
  a.gamma = gamma;
  a.status = status;
  a.wmin = wmin;
  a.wsum = wsum;
  a.lin = lin;
  a.quad = quad;
  a.stamps = stamps;
  a.col_part = reinterpret_cast<double*>(ws);
  a.scal_part = a.col_part + G * cols;
  a.g = a.scal_part + G;
  a.bar = reinterpret_cast<unsigned*>(a.g + cols);
  SIMOPT_CUDA(cudaMemsetAsync(a.bar, 0, sizeof(unsigned), st));
  void* params[] = {&a};
  const char* coop = getenv("SIMOPT_MV_EPOCH_COOP");
  if (coop && atoi(coop) == 0)  // A/B: ordinary launch (co-residency by grid size only)
    SIMOPT_CUDA(cudaLaunchKernel((const void*)fn, dim3((unsigned)G), dim3(kNT), params, smem, st));
  else
    SIMOPT_CUDA(cudaLaunchCooperativeKernel((const void*)fn, dim3((unsigned)G), dim3(kNT), params, smem, st));
  return SIMOPT_OK;
}
