// Multi-product newsvendor on sm_100a: fused demand resample + ECDF-count gradient,
// single-budget LMO and Frank-Wolfe update (reference: sobench/tasks.py:141-188,
// sampling.py:173-193, lmo.py:68-89, frank_wolfe.py:62-82, _kernels.py:210-259).
//
// Data layout (per resampling epoch, resident in HBM):
//   dem   [d][S] f64   row j = product j's S demand draws, split into segments of
//                      NV_SEG = 2048 draws; inside a segment the draws are grouped by
//                      bucket (counting-sorted), buckets in ascending order.
//   off   [d][nseg][NV_B] u16   start of each bucket inside its segment.
//   kappa [d] f64      bucket scale B / (12 sigma_j).
// Bucket map  f_j(D) = clamp(floor((D - mu_j) * kappa_j + B/2), 0, B-1) is monotone
// non-decreasing in D (every rounding step is), so for a query x_j:
//   #{D <= x} = #{f(D) < f(x)} + #{D in bucket f(x) : D <= x}
// exactly: elements of lower buckets are < x, elements of higher buckets are > x.
// The count equals the reference's upper-bound binary search on the fully sorted
// row (ecdf_count_block) for every x, while an epoch writes the demands once and
// each gradient reads one bucket per segment instead of the whole row.
#include "common.cuh"
#include "fw.cuh"
#include "glibc_math.cuh"
#include "glibc_tables.h"
#include "newsvendor.cuh"
#include "philox.cuh"
#include "reduce_device.cuh"
#include "rng_device.cuh"

namespace {

constexpr int kResampleThreads = 256;

__global__ void k_nv_kappa(const double* __restrict__ sigma, int64_t d, double* __restrict__ kappa) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < d;
       j += (int64_t)gridDim.x * blockDim.x)
    kappa[j] = (double)NV_B / (12.0 * sigma[j]);
}

// Persistent CTAs walk (product j, segment s) pairs.  Per segment: generate the
// segment's draws D = mu_j + sigma_j * z (sampling.py:190-191) in registers,
// histogram them by bucket in shared memory, scan, scatter into bucket order, and
// stream the segment and its bucket starts out.  The sin/cos table is staged once
// per CTA.
constexpr int kResampleMinBlocks = 4;

__global__ void __launch_bounds__(kResampleThreads, kResampleMinBlocks)
    k_nv_resample(uint64_t seed, uint64_t sid, uint64_t clo, uint64_t chi, int64_t d, int64_t S,
                  int nseg, const double* __restrict__ mu, const double* __restrict__ sigma,
                  const double* __restrict__ kappa, double* __restrict__ dem,
                  uint16_t* __restrict__ off) {
  extern __shared__ __align__(16) unsigned char nv_smem[];
  double* tab = reinterpret_cast<double*>(nv_smem);             // 440 doubles
  double* raw = tab + 448;                                        // NV_SEG
  double* sorted_ = raw + NV_SEG;                                 // NV_SEG
  int* hist = reinterpret_cast<int*>(sorted_ + NV_SEG);           // NV_B
  uint16_t* bid = reinterpret_cast<uint16_t*>(hist + NV_B);       // NV_SEG bucket ids
  __shared__ int wsum[kResampleThreads / 32];
  load_sincostab(tab);  // includes __syncthreads()
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nblk = d * nseg;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int64_t j = blk / nseg;
    const int s = (int)(blk - j * nseg);
    const int64_t e0 = (int64_t)s * NV_SEG;
    const int len = (int)((S - e0) < NV_SEG ? (S - e0) : NV_SEG);
    const double muj = mu[j], sj = sigma[j], kj = kappa[j];
    for (int i = threadIdx.x; i < NV_B; i += blockDim.x) hist[i] = 0;
    __syncthreads();

    // 1) generate normals i0 .. i0+len-1 of the epoch's standard_normal(d*S) draw
    const int64_t i0 = j * S + e0;
    const int64_t q0 = i0 >> 2, q1 = (i0 + len - 1) >> 2;
    for (int64_t q = q0 + threadIdx.x; q <= q1; q += blockDim.x) {
      double z[4];
      normals4(seed, sid, clo, chi, (uint64_t)q, tab, z);
      const int64_t l0 = (q << 2) - i0;
      if (l0 >= 0 && l0 + 4 <= len) {
        uint16_t bb[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double dv = muj + sj * z[k];
          raw[l0 + k] = dv;
          const int b = nv_bucket(dv, muj, kj);
          bb[k] = (uint16_t)b;
          atomicAdd(&hist[b], 1);
        }
        if ((l0 & 3) == 0) {
          reinterpret_cast<uint2*>(bid)[l0 >> 2] =
              make_uint2(bb[0] | ((uint32_t)bb[1] << 16), bb[2] | ((uint32_t)bb[3] << 16));
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) bid[l0 + k] = bb[k];
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int64_t l = l0 + k;
          if (l >= 0 && l < len) {
            const double dv = muj + sj * z[k];
            raw[l] = dv;
            const int b = nv_bucket(dv, muj, kj);
            bid[l] = (uint16_t)b;
            atomicAdd(&hist[b], 1);
          }
        }
      }
    }
    __syncthreads();
    // 2) exclusive scan of the histogram (NV_B entries, kPer per thread)
    {
      constexpr int kPer = NV_B / kResampleThreads;
      int v[kPer];
      int run = 0;
#pragma unroll
      for (int k = 0; k < kPer; ++k) { v[k] = hist[threadIdx.x * kPer + k]; run += v[k]; }
      int incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) wsum[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        int w = lane < kResampleThreads / 32 ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, w, o);
          if (lane >= o) w += t;
        }
        if (lane < kResampleThreads / 32) wsum[lane] = w;  // inclusive warp prefix
      }
      __syncthreads();
      int base = incl - run + (warp > 0 ? wsum[warp - 1] : 0);
      uint32_t packed = 0;
      uint16_t* o = off + ((j * nseg + s) * (int64_t)NV_B);
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int b = threadIdx.x * kPer + k;
        packed |= (uint32_t)(uint16_t)base << (16 * k);
        hist[b] = base;  // becomes the scatter cursor
        base += v[k];
      }
      static_assert(kPer == 2, "bucket starts are stored as one u32 per thread");
      reinterpret_cast<uint32_t*>(o)[threadIdx.x] = packed;
    }
    __syncthreads();
    // 3) scatter into bucket order (order inside a bucket is irrelevant to every count)
    for (int l = threadIdx.x; l < len; l += blockDim.x) {
      const int pos = atomicAdd(&hist[bid[l]], 1);
      sorted_[pos] = raw[l];
    }
    __syncthreads();
    double* dst = dem + j * S + e0;
    for (int l = threadIdx.x; l < len; l += blockDim.x) dst[l] = sorted_[l];
    __syncthreads();
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// ECDF count for one product, one warp: lanes take segments.
__device__ __forceinline__ int64_t nv_count_warp(const double* __restrict__ dem,
                                                 const uint16_t* __restrict__ off, int64_t j,
                                                 int64_t S, int nseg, double x, double muj,
                                                 double kj) {
  const int lane = threadIdx.x & 31;
  const int b = nv_bucket(x, muj, kj);
  int64_t cnt = 0;
  for (int s = lane; s < nseg; s += 32) {
    const int len = (int)((S - (int64_t)s * NV_SEG) < NV_SEG ? (S - (int64_t)s * NV_SEG) : NV_SEG);
    const uint16_t* o = off + (j * nseg + s) * (int64_t)NV_B;
    const int start = o[b];
    const int end = (b + 1 < NV_B) ? o[b + 1] : len;
    const double* seg = dem + j * S + (int64_t)s * NV_SEG;
    int c = start;
    for (int p = start; p < end; ++p) c += (seg[p] <= x) ? 1 : 0;
    cnt += c;
  }
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o2);
  return cnt;
}

// gradient (tasks.py:158-160): g = (k - v) + ((h + v) * (count / S))
__device__ __forceinline__ double nv_grad_value(int64_t cnt, int64_t S, double k, double h,
                                                double v) {
  const double frac = (double)cnt / (double)S;
  return (k - v) + ((h + v) * frac);
}

namespace {

constexpr int kIterWarps = 8;

// Fused FW step for the newsvendor:
//   (1) if do_update: x_j <- (gamma * ((-1 * x_j) + s_j)) + x_j with the vertex of the
//       previous LMO (frank_wolfe.py:69-82), record x_j < -FEAS_TOL, objective term;
//   (2) if do_grad: g_j at the (new) x_j, LMO values g_j * (C / c_j), argmin over all
//       products (last-block reduction), NaN flag.
__global__ void __launch_bounds__(kIterWarps * 32)
    k_nv_iter(NvIterArgs a) {
  __shared__ ArgMin warp_best[kIterWarps];
  __shared__ int nan_seen;
  __shared__ bool am_last;
  if (threadIdx.x == 0) nan_seen = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  ArgMin best{INFINITY, INT64_MAX};
  NvState* st = a.state;
  const int64_t jstar = st->jstar;
  const double sval = st->sval;
  for (int64_t j = (int64_t)blockIdx.x * kIterWarps + warp; j < a.d;
       j += (int64_t)gridDim.x * kIterWarps) {
    double x = a.x_in[j];
    if (a.do_update) {
      const double sj = (j == jstar) ? sval : 0.0;
      const double dir = (-1.0 * x) + sj;
      x = a.gamma * dir + x;
      if (lane == 0) {
        a.x[j] = x;
        if (x < -1e-10) atomicOr(&a.flags[a.step], NV_FLAG_NEGATIVE);
        a.terms[j] = nv_cost_term(x, a.mu[j], a.sigma[j], a.k[j], a.h[j], a.v[j]);
      }
    }
    if (a.do_grad) {
      const int64_t cnt = nv_count_warp(a.dem, a.off, j, a.S, a.nseg, x, a.mu[j], a.kappa[j]);
      const double g = nv_grad_value(cnt, a.S, a.k[j], a.h[j], a.v[j]);
      if (lane == 0) {
        a.g[j] = g;
        if (g != g) nan_seen = 1;
        const double val = g * (a.budget / a.c[j]);  // lmo.py:84
        best = amin(best, ArgMin{val, j});
      }
    }
  }
  if (!a.do_grad) return;
  if (lane == 0) warp_best[warp] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    ArgMin b = warp_best[0];
    for (int w = 1; w < kIterWarps; ++w) b = amin(b, warp_best[w]);
    a.part_v[blockIdx.x] = b.v;
    a.part_i[blockIdx.x] = b.i;
    if (nan_seen) atomicOr(&a.flags[a.grad_step], NV_FLAG_NAN_GRADIENT);
    __threadfence();
    const unsigned prev = atomicAdd(&st->blocks_done, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  // last block: reduce the per-block partials (deterministic: lexicographic min).
  ArgMin b{INFINITY, INT64_MAX};
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x)
    b = amin(b, ArgMin{((volatile double*)a.part_v)[i], ((volatile int64_t*)a.part_i)[i]});
  b = warp_amin(b);
  if (lane == 0) warp_best[warp] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    ArgMin r = warp_best[0];
    for (int w = 1; w < kIterWarps; ++w) r = amin(r, warp_best[w]);
    // lmo_single_budget (lmo.py:84-89): s_j* = C / c_j* iff g_j* < 0
    const double gj = a.g[r.i];
    st->jstar = r.i;
    st->sval = (gj < 0.0) ? a.budget / a.c[r.i] : 0.0;
    st->blocks_done = 0;
  }
}

}  // namespace

int simopt_nv_kappa_impl(cudaStream_t st, const double* sigma, int64_t d, double* kappa) {
  k_nv_kappa<<<(int)ceil_div(d, 256), 256, 0, st>>>(sigma, d, kappa);
  SIMOPT_CHECK_LAUNCH("k_nv_kappa");
  return SIMOPT_OK;
}

extern "C" int simopt_nv_geometry(int64_t* seg, int64_t* buckets) {
  if (seg) *seg = NV_SEG;
  if (buckets) *buckets = NV_B;
  return SIMOPT_OK;
}

extern "C" int simopt_nv_layout(int64_t d, int64_t S, int64_t* nseg, int64_t* dem_elems,
                                int64_t* off_elems) {
  SIMOPT_REQUIRE(d >= 1 && S >= 1, SIMOPT_E_EMPTY, "need d >= 1 products and S >= 1 samples");
  const int64_t ns = ceil_div(S, NV_SEG);
  if (nseg) *nseg = ns;
  if (dem_elems) *dem_elems = d * S;
  if (off_elems) *off_elems = d * ns * NV_B;
  return SIMOPT_OK;
}

extern "C" int simopt_nv_resample(void* stream, uint64_t seed, uint64_t sid, uint64_t clo,
                                  uint64_t chi, int64_t d, int64_t S, const double* mu,
                                  const double* sigma, double* kappa, double* dem, uint16_t* off) {
  SIMOPT_REQUIRE(d >= 1 && S >= 1, SIMOPT_E_EMPTY, "need at least one demand sample per product");
  cudaStream_t st = as_stream(stream);
  const int rc = simopt_nv_kappa_impl(st, sigma, d, kappa);
  if (rc) return rc;
  const int64_t nseg = ceil_div(S, NV_SEG);
  const int64_t nblk = d * nseg;
  SIMOPT_REQUIRE(nblk < (1LL << 31), SIMOPT_E_CONFIG, "too many segments");
  const size_t smem = (448 + 2 * NV_SEG) * sizeof(double) + NV_B * sizeof(int) +
                      NV_SEG * sizeof(uint16_t);
  static bool attr = false;
  if (!attr) {
    SIMOPT_CUDA(cudaFuncSetAttribute(k_nv_resample, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    attr = true;
  }
  const int64_t grid = nblk < (int64_t)SIMOPT_NUM_SMS * kResampleMinBlocks * 8
                           ? nblk : (int64_t)SIMOPT_NUM_SMS * kResampleMinBlocks * 8;
  k_nv_resample<<<(unsigned)grid, kResampleThreads, smem, st>>>(seed, sid, clo, chi, d, S,
                                                                (int)nseg, mu, sigma, kappa, dem,
                                                                off);
  SIMOPT_CHECK_LAUNCH("k_nv_resample");
  return SIMOPT_OK;
}

extern "C" int simopt_nv_iter(void* stream, const NvIterArgs* args) {
  NvIterArgs a = *args;
  const int grid = (int)(ceil_div(a.d, kIterWarps) < 16 * SIMOPT_NUM_SMS ? ceil_div(a.d, kIterWarps)
                                                                          : 16 * SIMOPT_NUM_SMS);
  SIMOPT_REQUIRE(grid <= a.part_capacity, SIMOPT_E_CONFIG, "partials buffer too small");
  k_nv_iter<<<grid, kIterWarps * 32, 0, as_stream(stream)>>>(a);
  SIMOPT_CHECK_LAUNCH("k_nv_iter");
  return SIMOPT_OK;
}

namespace {
__global__ void k_nv_counts(const double* __restrict__ dem, const uint16_t* __restrict__ off,
                            const double* __restrict__ kappa, const double* __restrict__ mu,
                            int64_t d, int64_t S, int nseg, const double* __restrict__ x,
                            int64_t* __restrict__ counts) {
  const int warp = threadIdx.x >> 5;
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; j < d;
       j += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const int64_t c = nv_count_warp(dem, off, j, S, nseg, x[j], mu[j], kappa[j]);
    if ((threadIdx.x & 31) == 0) counts[j] = c;
  }
}
}  // namespace

extern "C" int simopt_nv_counts(void* stream, const double* dem, const uint16_t* off,
                                const double* kappa, const double* mu, int64_t d, int64_t S,
                                const double* x, int64_t* counts) {
  const int64_t nseg = ceil_div(S, NV_SEG);
  const int grid = (int)(ceil_div(d, 8) < 8 * SIMOPT_NUM_SMS ? ceil_div(d, 8) : 8 * SIMOPT_NUM_SMS);
  k_nv_counts<<<grid, 256, 0, as_stream(stream)>>>(dem, off, kappa, mu, d, S, (int)nseg, x, counts);
  SIMOPT_CHECK_LAUNCH("k_nv_counts");
  return SIMOPT_OK;
}

namespace {
__global__ void k_nv_cost(const double* __restrict__ x, const double* __restrict__ mu,
                          const double* __restrict__ sigma, const double* __restrict__ unit,
                          const double* __restrict__ hold, const double* __restrict__ sell,
                          int64_t d, double* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < d;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = nv_cost_term(x[j], mu[j], sigma[j], unit[j], hold[j], sell[j]);
}
}  // namespace

extern "C" int simopt_nv_cost_terms(void* stream, const double* x, const double* mu,
                                    const double* sigma, const double* unit, const double* hold,
                                    const double* sell, int64_t d, double* out) {
  if (d == 0) return SIMOPT_OK;
  k_nv_cost<<<(int)(ceil_div(d, 256) < 2048 ? ceil_div(d, 256) : 2048), 256, 0,
              as_stream(stream)>>>(x, mu, sigma, unit, hold, sell, d, out);
  SIMOPT_CHECK_LAUNCH("k_nv_cost");
  return SIMOPT_OK;
}

namespace {
// ecdf_count_block (_kernels.py:245-259): upper-bound binary search on sorted rows.
__global__ void k_ecdf_sorted(const double* __restrict__ samples, int64_t rows, int64_t s,
                              const double* __restrict__ x, int64_t* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < rows;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double xj = x[j];
    const double* row = samples + j * s;
    int64_t lo = 0, hi = s;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (row[mid] <= xj) lo = mid + 1; else hi = mid;
    }
    out[j] = lo;
  }
}

__global__ void k_nv_grad_counts(const int64_t* __restrict__ cnt, int64_t S,
                                 const double* __restrict__ k, const double* __restrict__ h,
                                 const double* __restrict__ v, int64_t d, double* __restrict__ g) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < d;
       j += (int64_t)gridDim.x * blockDim.x)
    g[j] = nv_grad_value(cnt[j], S, k[j], h[j], v[j]);
}
}  // namespace

extern "C" int simopt_ecdf_count_sorted(void* stream, const double* samples, int64_t rows,
                                        int64_t s, const double* x, int64_t* counts) {
  if (rows == 0) return SIMOPT_OK;
  k_ecdf_sorted<<<(int)(ceil_div(rows, 128) < 4096 ? ceil_div(rows, 128) : 4096), 128, 0,
                  as_stream(stream)>>>(samples, rows, s, x, counts);
  SIMOPT_CHECK_LAUNCH("k_ecdf_sorted");
  return SIMOPT_OK;
}

extern "C" int simopt_nv_grad_from_counts(void* stream, const int64_t* counts, int64_t S,
                                          const double* k, const double* h, const double* v,
                                          int64_t d, double* g) {
  if (d == 0) return SIMOPT_OK;
  k_nv_grad_counts<<<(int)(ceil_div(d, 256) < 4096 ? ceil_div(d, 256) : 4096), 256, 0,
                     as_stream(stream)>>>(counts, S, k, h, v, d, g);
  SIMOPT_CHECK_LAUNCH("k_nv_grad_counts");
  return SIMOPT_OK;
}
