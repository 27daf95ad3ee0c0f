// Exact fixed-tree reductions (reference: sobench/_kernels.py:1-156, backend.py:80-141).
//
// The tree is a function of (length, chunk) only: each chunk of `chunk`
// consecutive elements is summed strictly left to right, and the chunk partials
// are folded pairwise in index order (odd tail carried).  Every chunk chain is
// a dependent DADD sequence, so these kernels are latency-bound per chain and
// get their throughput from running many chains at once: one thread per
// (row|column, chunk).  -fmad=false keeps x*y and s+p unfused, as in numba.
#include "common.cuh"
#include "reduce_device.cuh"

namespace {

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

constexpr int kFoldSmem = 4096;  // partials folded in one CTA's shared memory

// --- chunk partials of dot / sum ------------------------------------------------
// One warp per chunk.  The warp stages 256-element tiles through shared memory
// (coalesced loads, products formed by all lanes, next tile already in flight)
// and lane 0 adds the tile in index order: a single dependent DADD chain per
// chunk, fed from shared memory so the chain runs at DADD latency.
constexpr int kTile = 256;
constexpr int kPartialWarps = 4;

struct TreeJob {
  const double* x;
  const double* y;  // NULL: plain sum
  int64_t n;
  double* out;      // root (device scalar)
};
struct TreeJobs {
  TreeJob job[4];
  int njobs;
  int64_t chunk;
  int64_t first_chunk[5];  // prefix of chunk counts
};

// Raw tile loads (no consumer until the next iteration, so they stay in flight
// while lane 0 walks the previous tile).
__device__ __forceinline__ void tile_load(const double* __restrict__ x, const double* __restrict__ y,
                                          int64_t base, int64_t hi, int lane,
                                          double (&xr)[kTile / 32], double (&yr)[kTile / 32]) {
#pragma unroll
  for (int t = 0; t < kTile / 32; ++t) {
    const int64_t i = base + lane + 32 * t;
    xr[t] = (i < hi) ? x[i] : 0.0;
    yr[t] = (y != nullptr && i < hi) ? y[i] : 1.0;
  }
}

__device__ __forceinline__ double warp_chunk_sum(const double* __restrict__ x,
                                                 const double* __restrict__ y, int64_t lo,
                                                 int64_t hi, double* buf) {
  const int lane = threadIdx.x & 31;
  const bool has_y = y != nullptr;
  double xr[kTile / 32], yr[kTile / 32];
  double s = 0.0;
  tile_load(x, y, lo, hi, lane, xr, yr);
  int parity = 0;
  for (int64_t base = lo; base < hi; base += kTile) {
    double* b = buf + parity * kTile;
#pragma unroll
    for (int t = 0; t < kTile / 32; ++t) b[lane + 32 * t] = has_y ? xr[t] * yr[t] : xr[t];
    __syncwarp();
    if (base + kTile < hi) tile_load(x, y, base + kTile, hi, lane, xr, yr);
    if (lane == 0) {
      const int cnt = (int)(hi - base < kTile ? hi - base : kTile);
      if (cnt == kTile) {
        // 16-element register batches, next batch loaded before the current is added
        double v[16], w[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = b[k];
#pragma unroll
        for (int i = 0; i < kTile; i += 32) {
#pragma unroll
          for (int k = 0; k < 16; ++k) w[k] = b[i + 16 + k];
#pragma unroll
          for (int k = 0; k < 16; ++k) s = s + v[k];
          if (i + 32 < kTile) {
#pragma unroll
            for (int k = 0; k < 16; ++k) v[k] = b[i + 32 + k];
          }
#pragma unroll
          for (int k = 0; k < 16; ++k) s = s + w[k];
        }
      } else {
        for (int i = 0; i < cnt; ++i) s = s + b[i];
      }
    }
    parity ^= 1;
  }
  __syncwarp();
  return s;
}

__global__ void __launch_bounds__(kPartialWarps * 32)
    k_tree_jobs(TreeJobs jobs, double* __restrict__ partials, unsigned* __restrict__ counters) {
  __shared__ double buf[kPartialWarps][2 * kTile];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t total = jobs.first_chunk[jobs.njobs];
  for (int64_t g = (int64_t)blockIdx.x * kPartialWarps + warp; g < total;
       g += (int64_t)gridDim.x * kPartialWarps) {
    int jb = 0;
    while (g >= jobs.first_chunk[jb + 1]) ++jb;
    const TreeJob J = jobs.job[jb];
    const int64_t c = g - jobs.first_chunk[jb];
    const int64_t nch = jobs.first_chunk[jb + 1] - jobs.first_chunk[jb];
    const int64_t lo = c * jobs.chunk;
    const int64_t hi = lo + jobs.chunk < J.n ? lo + jobs.chunk : J.n;
    const double s = warp_chunk_sum(J.x, J.y, lo, hi, buf[warp]);
    double* p = partials + jobs.first_chunk[jb];
    if (lane == 0) {
      p[c] = s;
      if (nch <= 64) {  // the warp finishing a small job folds it (otherwise host folds)
        __threadfence();
        const unsigned prev = atomicAdd(&counters[jb], 1u);
        if (prev == nch - 1) {
          __threadfence();
          volatile double* vp = p;
          double q[64];
          for (int i = 0; i < nch; ++i) q[i] = vp[i];
          int m = (int)nch;
          while (m > 1) {
            const int h = m >> 1;
            for (int i = 0; i < h; ++i) q[i] = q[2 * i] + q[2 * i + 1];
            if (m & 1) { q[h] = q[m - 1]; m = h + 1; } else { m = h; }
          }
          *J.out = q[0];
          counters[jb] = 0;
        }
      }
    }
  }
}

// One fold level in global memory: dst[i] = src[2i] + src[2i+1]; odd tail carried.
__global__ void k_fold_level(const double* __restrict__ src, double* __restrict__ dst, int64_t m) {
  const int64_t h = m >> 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < h;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[2 * i] + src[2 * i + 1];
  if ((m & 1) && blockIdx.x == 0 && threadIdx.x == 0) dst[h] = src[m - 1];
}

__global__ void __launch_bounds__(512) k_fold_final(const double* __restrict__ src, int m,
                                                    double* __restrict__ out) {
  extern __shared__ double sm[];
  double* a = sm;
  double* b = sm + kFoldSmem;
  for (int i = threadIdx.x; i < m; i += blockDim.x) a[i] = src[i];
  const double r = block_fold_pairwise(a, b, m);
  if (threadIdx.x == 0) *out = r;
}

// --- matvec: out[r] = tree-dot(row(r) - center, x) -------------------------------
// One warp per (32-row strip, column chunk); lane r owns row r's chain.  Row
// segments (32 columns, 256 B, coalesced) stream through a kTStages-deep cp.async
// ring; the tile row stride is padded to 33 doubles so the lane-per-row reads are
// conflict-free.
constexpr int kRStages = 5;

template <bool kCenter, bool kIdx, bool kV16>
__global__ void __launch_bounds__(32) k_matvec_rows(const double* __restrict__ a, int64_t cols,
                                                    const int64_t* __restrict__ idx, int64_t rows,
                                                    const double* __restrict__ center,
                                                    const double* __restrict__ x, int64_t chunk,
                                                    int64_t nch, double* __restrict__ out) {
  __shared__ __align__(16) double tile[kRStages][32][34];  // 272-B rows: 16-B aligned, 2-way banks
  __shared__ __align__(16) double xs[kRStages][32];
  __shared__ __align__(16) double cs[kRStages][32];
  const int lane = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int64_t c = blockIdx.y;
  const int64_t clo = c * chunk;
  const int64_t chi = clo + chunk < cols ? clo + chunk : cols;
  const int64_t nst = (chi - clo + 31) / 32;
  const int h = lane >> 4, m2 = 2 * (lane & 15);
  int64_t rowA = 0, rowB = 0;  // v16: rows 2rr+h handled by this lane are fetched per stage
  (void)rowA; (void)rowB;
  auto issue = [&](int64_t st) {
    const int buf = (int)(st % kRStages);
    const int64_t j0 = clo + st * 32;
    const int64_t jj = j0 + lane;
    const bool jv = jj < chi;
    if (kV16) {
      const bool pv = (j0 + m2 < chi);  // chi even (cols even, chunk even)
#pragma unroll 4
      for (int rr = 0; rr < 16; ++rr) {
        const int r = 2 * rr + h;
        const int64_t grow = r0 + r;
        const bool v = grow < rows && pv;
        const int64_t row = (grow < rows) ? (kIdx ? idx[grow] : grow) : 0;
        cp_async16(&tile[buf][r][m2], a + row * cols + (pv ? j0 + m2 : 0), v);
      }
    } else {
#pragma unroll 8
      for (int rr = 0; rr < 32; ++rr) {
        const int64_t grow = r0 + rr;
        const bool v = grow < rows && jv;
        const int64_t row = (grow < rows) ? (kIdx ? idx[grow] : grow) : 0;
        cp_async8(&tile[buf][rr][lane], a + row * cols + (jv ? jj : 0), v);
      }
    }
    cp_async8(&xs[buf][lane], x + (jv ? jj : 0), jv);
    if (kCenter) cp_async8(&cs[buf][lane], center + (jv ? jj : 0), jv);
    cp_async_commit();
  };
  for (int64_t st = 0; st < kRStages - 1; ++st) {
    if (st < nst) issue(st); else cp_async_commit();
  }
  double s = 0.0;
  for (int64_t st = 0; st < nst; ++st) {
    if (st + kRStages - 1 < nst) issue(st + kRStages - 1); else cp_async_commit();
    cp_async_wait<kRStages - 1>();
    __syncwarp();
    const int buf = (int)(st % kRStages);
    const int cnt = (int)((chi - clo) - st * 32 < 32 ? (chi - clo) - st * 32 : 32);
    if (cnt == 32) {
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        const double v = tile[buf][lane][jj];
        s = s + (kCenter ? v - cs[buf][jj] : v) * xs[buf][jj];
      }
    } else {
      for (int jj = 0; jj < cnt; ++jj) {
        const double v = tile[buf][lane][jj];
        s = s + (kCenter ? v - cs[buf][jj] : v) * xs[buf][jj];
      }
    }
    __syncwarp();
  }
  const int64_t r = r0 + lane;
  if (r < rows) {
    if (nch == 1) out[r] = s;
    else out[r * nch + c] = s;  // partials, folded by k_fold_strided
  }
}

// Per-row (or per-column) serial fold of `nch` partials laid out with stride.
__global__ void k_fold_strided(double* __restrict__ p, int64_t count, int64_t nch, int64_t s_item,
                               int64_t s_chunk, double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    double* q = p + t * s_item;
    int64_t m = nch;
    while (m > 1) {
      const int64_t h = m >> 1;
      for (int64_t i = 0; i < h; ++i) q[i * s_chunk] = q[2 * i * s_chunk] + q[(2 * i + 1) * s_chunk];
      if (m & 1) { q[h * s_chunk] = q[(m - 1) * s_chunk]; m = h + 1; } else { m = h; }
    }
    out[t] = q[0];
  }
}

// --- matvec_t: out[j] = tree over row chunks of sum x[r]*(a[row(r),j]-center[j]) ---
// One warp per (32-column strip, row chunk); lane j owns column j's chain.  Rows
// stream through a kStages-deep cp.async ring (32 rows x 32 columns per stage),
// so each chain runs at DADD latency instead of waiting on memory per row.
constexpr int kTStages = 5;
constexpr int kTRows = 32;

template <bool kCenter, bool kIdx, bool kV16>
__global__ void __launch_bounds__(32) k_matvec_t_cols(const double* __restrict__ a, int64_t cols,
                                                      const int64_t* __restrict__ idx, int64_t rows,
                                                      const double* __restrict__ center,
                                                      const double* __restrict__ x, int64_t chunk,
                                                      int64_t nch, double* __restrict__ out) {
  __shared__ __align__(16) double tile[kTStages][kTRows][32];
  __shared__ __align__(16) double xs[kTStages][kTRows];
  const int lane = threadIdx.x;
  const int64_t j0 = (int64_t)blockIdx.x * 32;
  const int64_t j = j0 + lane;
  const int64_t c = blockIdx.y;
  const int64_t lo = c * chunk;
  const int64_t hi = lo + chunk < rows ? lo + chunk : rows;
  const bool jv = j < cols;
  const double cj = (kCenter && jv) ? center[j] : 0.0;
  const int64_t nst = (hi - lo + kTRows - 1) / kTRows;
  // 16-byte copies: lane = (half h, pair m) moves columns j0+2m, j0+2m+1 of rows r0+2rr+h
  const int h = lane >> 4, m2 = 2 * (lane & 15);
  const bool pv = (j0 + m2 < cols);  // cols even => both columns valid together
  auto issue = [&](int64_t st) {
    const int buf = (int)(st % kTStages);
    const int64_t r0 = lo + st * kTRows;
    if (kV16) {
#pragma unroll 4
      for (int rr = 0; rr < kTRows / 2; ++rr) {
        const int r = 2 * rr + h;
        const int64_t grow = r0 + r;
        const bool v = grow < hi;
        const int64_t row = v ? (kIdx ? idx[grow] : grow) : 0;
        cp_async16(&tile[buf][r][m2], a + row * cols + (pv ? j0 + m2 : 0), v && pv);
      }
    } else {
#pragma unroll 8
      for (int r = 0; r < kTRows; ++r) {
        const int64_t grow = r0 + r;
        const bool v = grow < hi;
        const int64_t row = v ? (kIdx ? idx[grow] : grow) : 0;
        cp_async8(&tile[buf][r][lane], a + row * cols + (jv ? j : 0), v && jv);
      }
    }
    const int64_t rr = r0 + lane;
    cp_async8(&xs[buf][lane], x + (rr < hi ? rr : 0), rr < hi);
    cp_async_commit();
  };
  for (int64_t st = 0; st < kTStages - 1; ++st) {
    if (st < nst) issue(st); else cp_async_commit();
  }
  double s = 0.0;
  for (int64_t st = 0; st < nst; ++st) {
    if (st + kTStages - 1 < nst) issue(st + kTStages - 1); else cp_async_commit();
    cp_async_wait<kTStages - 1>();
    __syncwarp();
    const int buf = (int)(st % kTStages);
    const int cnt = (int)((hi - lo) - st * kTRows < kTRows ? (hi - lo) - st * kTRows : kTRows);
    if (cnt == kTRows) {
#pragma unroll
      for (int r = 0; r < kTRows; ++r) {
        const double v = tile[buf][r][lane];
        s = s + xs[buf][r] * (kCenter ? v - cj : v);
      }
    } else {
      for (int r = 0; r < cnt; ++r) {
        const double v = tile[buf][r][lane];
        s = s + xs[buf][r] * (kCenter ? v - cj : v);
      }
    }
    __syncwarp();
  }
  if (!jv) return;
  if (nch == 1) out[j] = s;
  else out[c * cols + j] = s;  // partials, folded by k_fold_strided
}

bool vec16_ok(const void* a, int64_t cols) {
  return ((reinterpret_cast<uintptr_t>(a) & 15u) == 0) && (cols % 2 == 0);
}

__global__ void k_axpy_ptr(const double* __restrict__ alpha, const double* __restrict__ x,
                           const double* __restrict__ y, int64_t n, double* __restrict__ out) {
  const double a = *alpha;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a * x[i] + y[i];
}

__global__ void k_axpy(double alpha, const double* __restrict__ x, const double* __restrict__ y,
                       int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = alpha * x[i] + y[i];
}

__global__ void k_map(int kernel, const double* __restrict__ x, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double t = x[i];
    if (kernel == SIMOPT_MAP_NEGATE) out[i] = -t;
    else if (kernel == SIMOPT_MAP_EXP) out[i] = dev_exp(t);
    else out[i] = dev_sigmoid(t);
  }
}

int elementwise_grid(int64_t n) {
  const int64_t g = ceil_div(n, 256);
  const int64_t cap = (int64_t)SIMOPT_NUM_SMS * 16;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

// Fold p[0..m) (device, destroyed) into *out.  Enqueued on `st`.
int simopt_fold_partials(cudaStream_t st, double* p, double* tmp, int64_t m, double* out) {
  if (m == 0) {
    SIMOPT_CUDA(cudaMemsetAsync(out, 0, sizeof(double), st));
    return SIMOPT_OK;
  }
  double* src = p;
  double* dst = tmp;
  while (m > kFoldSmem) {
    const int64_t h = m >> 1;
    k_fold_level<<<elementwise_grid(h), 256, 0, st>>>(src, dst, m);
    SIMOPT_CHECK_LAUNCH("k_fold_level");
    m = (m & 1) ? h + 1 : h;
    double* t = src; src = dst; dst = t;
  }
  static bool attr_set = false;
  if (!attr_set) {
    SIMOPT_CUDA(cudaFuncSetAttribute(k_fold_final, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     2 * kFoldSmem * (int)sizeof(double)));
    attr_set = true;
  }
  k_fold_final<<<1, 512, 2 * kFoldSmem * sizeof(double), st>>>(src, (int)m, out);
  SIMOPT_CHECK_LAUNCH("k_fold_final");
  return SIMOPT_OK;
}

// Enqueue up to 4 independent fixed-tree reductions in one launch.
static int tree_jobs(cudaStream_t st, TreeJob* js, int nj, int64_t chunk) {
  SIMOPT_REQUIRE(chunk >= 1, SIMOPT_E_CONFIG, "chunk_size must be >= 1, got %lld", (long long)chunk);
  TreeJobs J{};
  J.chunk = chunk;
  int k = 0;
  for (int i = 0; i < nj; ++i) {
    if (js[i].n == 0) {
      SIMOPT_CUDA(cudaMemsetAsync(js[i].out, 0, sizeof(double), st));
      continue;
    }
    J.job[k++] = js[i];
  }
  if (k == 0) return SIMOPT_OK;
  J.njobs = k;
  J.first_chunk[0] = 0;
  for (int i = 0; i < k; ++i) J.first_chunk[i + 1] = J.first_chunk[i] + ceil_div(J.job[i].n, chunk);
  const int64_t total = J.first_chunk[k];
  unsigned char* ws = static_cast<unsigned char*>(simopt_scratch(st, 2 * total * sizeof(double) + 64));
  SIMOPT_REQUIRE(ws != nullptr, SIMOPT_E_CUDA, "%s", simopt_last_error());
  double* partials = reinterpret_cast<double*>(ws);
  unsigned* counters = reinterpret_cast<unsigned*>(ws + 2 * total * sizeof(double));
  SIMOPT_CUDA(cudaMemsetAsync(counters, 0, 4 * sizeof(unsigned), st));
  const int64_t g = ceil_div(total, kPartialWarps);
  const int grid = (int)(g < 16 * SIMOPT_NUM_SMS ? g : 16 * SIMOPT_NUM_SMS);
  k_tree_jobs<<<grid, kPartialWarps * 32, 0, st>>>(J, partials, counters);
  SIMOPT_CHECK_LAUNCH("k_tree_jobs");
  for (int i = 0; i < k; ++i) {
    const int64_t nch = J.first_chunk[i + 1] - J.first_chunk[i];
    if (nch > 64) {
      const int rc = simopt_fold_partials(st, partials + J.first_chunk[i], partials + total + J.first_chunk[i],
                                          nch, J.job[i].out);
      if (rc) return rc;
    }
  }
  return SIMOPT_OK;
}

static int tree_reduce(cudaStream_t st, const double* x, const double* y, int64_t n, int64_t chunk,
                       double* out) {
  TreeJob j{x, y, n, out};
  return tree_jobs(st, &j, 1, chunk);
}

extern "C" int simopt_tree_sums2(void* stream, const double* x0, const double* y0, int64_t n0,
                                 double* out0, const double* x1, const double* y1, int64_t n1,
                                 double* out1, int64_t chunk) {
  TreeJob j[2] = {{x0, y0, n0, out0}, {x1, y1, n1, out1}};
  return tree_jobs(as_stream(stream), j, 2, chunk);
}

extern "C" int simopt_dot(void* stream, const double* x, const double* y, int64_t n, int64_t chunk,
                          double* out) {
  return tree_reduce(as_stream(stream), x, y, n, chunk, out);
}

namespace {
// One CTA, fixed order: thread t sums x[i] * y[i] for i = t, t + 1024, ... (no FMA), then a
// fixed xor tree per warp and the 32 warp sums in warp order.  Deterministic, not the
// reference's tree: for the fused solvers' short d-vectors, where the tree's 4096-long
// sequential chain (~10 us per dot) is the cost.
constexpr int kDotFastThreads = 1024;
__global__ void __launch_bounds__(kDotFastThreads) k_dot_fast(const double* __restrict__ x,
                                                              const double* __restrict__ y,
                                                              int64_t n, double* __restrict__ out) {
  __shared__ double ws[kDotFastThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  double s = 0.0;
  for (int64_t i = tid; i < n; i += kDotFastThreads) s += x[i] * y[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) ws[w] = s;
  __syncthreads();
  if (w == 0) {
    double t = ws[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) *out = t;
  }
}
}  // namespace

extern "C" int simopt_dot_fast(void* stream, const double* x, const double* y, int64_t n, double* out) {
  SIMOPT_REQUIRE(n >= 0, SIMOPT_E_DIMENSION, "negative length");
  k_dot_fast<<<1, kDotFastThreads, 0, as_stream(stream)>>>(x, y, n, out);
  SIMOPT_CHECK_LAUNCH("k_dot_fast");
  return SIMOPT_OK;
}

namespace {
// Column sums of a row-major rows x cols matrix in a fixed order: row group g (rows
// [g R, (g + 1) R)) summed sequentially per column by one lane (a warp covers 32 adjacent
// columns: 256-byte rows), then the groups' partials folded in group order.  Deterministic,
// not the reference's 4096-chunk tree: chains of R instead of 4096 sequential additions.
constexpr int kColGroups = 256;
__global__ void k_col_sums_part(const double* __restrict__ x, int64_t rows, int64_t cols, int64_t R,
                                double* __restrict__ part) {
  const int64_t c = (int64_t)blockIdx.x * 32 + (threadIdx.x & 31);
  const int64_t g = (int64_t)blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= cols || g >= kColGroups) return;
  const int64_t r0 = g * R, r1 = r0 + R < rows ? r0 + R : rows;
  double s = 0.0;
  for (int64_t r = r0; r < r1; ++r) s += x[r * cols + c];
  part[g * cols + c] = s;
}
__global__ void k_col_sums_fold(const double* __restrict__ part, int64_t cols, double* __restrict__ out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  double s = 0.0;
  for (int g = 0; g < kColGroups; ++g) s += part[g * cols + c];
  out[c] = s;
}
}  // namespace

extern "C" int simopt_col_sums_fast(void* stream, const double* x, int64_t rows, int64_t cols,
                                    double* out) {
  SIMOPT_REQUIRE(rows >= 0 && cols >= 0, SIMOPT_E_DIMENSION, "negative extent");
  if (cols == 0) return SIMOPT_OK;
  cudaStream_t st = as_stream(stream);
  double* part = static_cast<double*>(simopt_scratch(st, (size_t)kColGroups * cols * sizeof(double)));
  SIMOPT_REQUIRE(part != nullptr, SIMOPT_E_CUDA, "%s", simopt_last_error());
  const int64_t R = (rows + kColGroups - 1) / kColGroups;
  k_col_sums_part<<<dim3((unsigned)ceil_div(cols, 32), kColGroups / 4), 128, 0, st>>>(x, rows, cols, R, part);
  SIMOPT_CHECK_LAUNCH("k_col_sums_part");
  k_col_sums_fold<<<(unsigned)ceil_div(cols, 256), 256, 0, st>>>(part, cols, out);
  SIMOPT_CHECK_LAUNCH("k_col_sums_fold");
  return SIMOPT_OK;
}

extern "C" int simopt_vec_sum(void* stream, const double* x, int64_t n, int64_t chunk, double* out) {
  return tree_reduce(as_stream(stream), x, nullptr, n, chunk, out);
}

extern "C" int simopt_matvec(void* stream, const double* a, int64_t lda_rows, int64_t cols,
                             const int64_t* idx, int64_t rows, const double* center,
                             const double* x, int64_t chunk, double* out) {
  (void)lda_rows;
  SIMOPT_REQUIRE(chunk >= 1, SIMOPT_E_CONFIG, "chunk_size must be >= 1");
  cudaStream_t st = as_stream(stream);
  if (rows == 0) return SIMOPT_OK;
  if (cols == 0) {
    SIMOPT_CUDA(cudaMemsetAsync(out, 0, rows * sizeof(double), st));
    return SIMOPT_OK;
  }
  const int64_t nch = ceil_div(cols, chunk);
  SIMOPT_REQUIRE(nch < 65536, SIMOPT_E_CONFIG, "too many column chunks (%lld)", (long long)nch);
  SIMOPT_REQUIRE(ceil_div(rows, 32) < (1LL << 31), SIMOPT_E_CONFIG, "too many rows");
  double* p = out;
  if (nch > 1) {
    p = static_cast<double*>(simopt_scratch(st, rows * nch * sizeof(double)));
    SIMOPT_REQUIRE(p != nullptr, SIMOPT_E_CUDA, "%s", simopt_last_error());
  }
  const dim3 grid((unsigned)ceil_div(rows, 32), (unsigned)nch);
  const int sel = (center ? 1 : 0) | (idx ? 2 : 0);
  const bool v16 = vec16_ok(a, cols) && (chunk % 2 == 0);
  switch (sel) {
    case 0: if (v16) k_matvec_rows<false, false, true><<<grid, 32, 0, st>>>(a, cols, idx, rows, center, x, chunk, nch, p); else k_matvec_rows<false, false, false><<<grid, 32, 0, st>>>(a, cols, idx, rows, center, x, chunk, nch, p); break;
    case 1: if (v16) k_matvec_rows<true, false, true><<<grid, 32, 0, st>>>(a, cols, idx, rows, center, x, chunk, nch, p); else k_matvec_rows<true, false, false><<<grid, 32, 0, st>>>(a, cols, idx, rows, center, x, chunk, nch, p); break;
    case 2: if (v16) k_matvec_rows<false, true, true><<<grid, 32, 0, st>>>(a, cols, idx, rows, center, x, chunk, nch, p); else k_matvec_rows<false, true, false><<<grid, 32, 0, st>>>(a, cols, idx, rows, center, x, chunk, nch, p); break;
    default: if (v16) k_matvec_rows<true, true, true><<<grid, 32, 0, st>>>(a, cols, idx, rows, center, x, chunk, nch, p); else k_matvec_rows<true, true, false><<<grid, 32, 0, st>>>(a, cols, idx, rows, center, x, chunk, nch, p); break;
  }
  SIMOPT_CHECK_LAUNCH("k_matvec_rows");
  if (nch > 1) {
    k_fold_strided<<<elementwise_grid(rows), 256, 0, st>>>(p, rows, nch, nch, 1, out);
    SIMOPT_CHECK_LAUNCH("k_fold_strided");
  }
  return SIMOPT_OK;
}

extern "C" int simopt_matvec_t(void* stream, const double* a, int64_t lda_rows, int64_t cols,
                               const int64_t* idx, int64_t rows, const double* center,
                               const double* x, int64_t chunk, double* out) {
  (void)lda_rows;
  SIMOPT_REQUIRE(chunk >= 1, SIMOPT_E_CONFIG, "chunk_size must be >= 1");
  cudaStream_t st = as_stream(stream);
  if (cols == 0) return SIMOPT_OK;
  if (rows == 0) {
    SIMOPT_CUDA(cudaMemsetAsync(out, 0, cols * sizeof(double), st));
    return SIMOPT_OK;
  }
  const int64_t nch = ceil_div(rows, chunk);
  SIMOPT_REQUIRE(nch < 65536, SIMOPT_E_CONFIG, "too many row chunks (%lld)", (long long)nch);
  double* p = out;
  if (nch > 1) {
    p = static_cast<double*>(simopt_scratch(st, cols * nch * sizeof(double)));
    SIMOPT_REQUIRE(p != nullptr, SIMOPT_E_CUDA, "%s", simopt_last_error());
  }
  const dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)nch);
  const int sel = (center ? 1 : 0) | (idx ? 2 : 0);
  const bool v16 = vec16_ok(a, cols);
  switch (sel) {
    case 0: if (v16) k_matvec_t_cols<false, false, true><<<grid, 32, 0, st>>>(a, cols, idx, rows, center, x, chunk, nch, p); else k_matvec_t_cols<false, false, false><<<grid, 32, 0, st>>>(a, cols, idx, rows, center, x, chunk, nch, p); break;
    case 1: if (v16) k_matvec_t_cols<true, false, true><<<grid, 32, 0, st>>>(a, cols, idx, rows, center, x, chunk, nch, p); else k_matvec_t_cols<true, false, false><<<grid, 32, 0, st>>>(a, cols, idx, rows, center, x, chunk, nch, p); break;
    case 2: if (v16) k_matvec_t_cols<false, true, true><<<grid, 32, 0, st>>>(a, cols, idx, rows, center, x, chunk, nch, p); else k_matvec_t_cols<false, true, false><<<grid, 32, 0, st>>>(a, cols, idx, rows, center, x, chunk, nch, p); break;
    default: if (v16) k_matvec_t_cols<true, true, true><<<grid, 32, 0, st>>>(a, cols, idx, rows, center, x, chunk, nch, p); else k_matvec_t_cols<true, true, false><<<grid, 32, 0, st>>>(a, cols, idx, rows, center, x, chunk, nch, p); break;
  }
  SIMOPT_CHECK_LAUNCH("k_matvec_t_cols");
  if (nch > 1) {
    k_fold_strided<<<elementwise_grid(cols), 256, 0, st>>>(p, cols, nch, 1, cols, out);
    SIMOPT_CHECK_LAUNCH("k_fold_strided");
  }
  return SIMOPT_OK;
}

// Chunk partials of matvec_t without the fold: out[c * cols + j] = chain of row chunk c
// (_kernels.py:124-156 before fold_pairwise).  Row-sharded ranks whose shards start on
// chunk boundaries produce exactly the reference's partials for their chunks; gathered
// in rank order and folded (simopt_fold_partials) they give the single-process result
// bit for bit (SURVEY 8e deterministic mode).
extern "C" int simopt_matvec_t_partials(void* stream, const double* a, int64_t rows, int64_t cols,
                                        const double* center, const double* x, int64_t chunk,
                                        double* out) {
  SIMOPT_REQUIRE(chunk >= 1, SIMOPT_E_CONFIG, "chunk_size must be >= 1");
  cudaStream_t st = as_stream(stream);
  if (cols == 0 || rows == 0) return SIMOPT_OK;
  const int64_t nch = ceil_div(rows, chunk);
  SIMOPT_REQUIRE(nch < 65536, SIMOPT_E_CONFIG, "too many row chunks (%lld)", (long long)nch);
  const dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)nch);
  const bool v16 = vec16_ok(a, cols);
  if (center) {
    if (v16) k_matvec_t_cols<true, false, true><<<grid, 32, 0, st>>>(a, cols, nullptr, rows, center, x, chunk, nch, out);
    else k_matvec_t_cols<true, false, false><<<grid, 32, 0, st>>>(a, cols, nullptr, rows, center, x, chunk, nch, out);
  } else {
    if (v16) k_matvec_t_cols<false, false, true><<<grid, 32, 0, st>>>(a, cols, nullptr, rows, center, x, chunk, nch, out);
    else k_matvec_t_cols<false, false, false><<<grid, 32, 0, st>>>(a, cols, nullptr, rows, center, x, chunk, nch, out);
  }
  SIMOPT_CHECK_LAUNCH("k_matvec_t_cols<partials>");
  return SIMOPT_OK;
}

// out[j] = fold_pairwise(p[0*count + j], ..., p[(nch-1)*count + j]); p is overwritten.
extern "C" int simopt_fold_partials(void* stream, double* p, int64_t nch, int64_t count, double* out) {
  if (count == 0) return SIMOPT_OK;
  cudaStream_t st = as_stream(stream);
  if (nch == 0) {
    SIMOPT_CUDA(cudaMemsetAsync(out, 0, count * sizeof(double), st));
    return SIMOPT_OK;
  }
  k_fold_strided<<<elementwise_grid(count), 256, 0, st>>>(p, count, nch, 1, count, out);
  SIMOPT_CHECK_LAUNCH("k_fold_strided");
  return SIMOPT_OK;
}

extern "C" int simopt_axpy(void* stream, double alpha, const double* x, const double* y, int64_t n,
                           double* out) {
  if (n == 0) return SIMOPT_OK;
  k_axpy<<<elementwise_grid(n), 256, 0, as_stream(stream)>>>(alpha, x, y, n, out);
  SIMOPT_CHECK_LAUNCH("k_axpy");
  return SIMOPT_OK;
}

extern "C" int simopt_map_kernel(void* stream, int kernel, const double* x, int64_t n, double* out) {
  SIMOPT_REQUIRE(kernel >= 0 && kernel <= 2, SIMOPT_E_CONFIG, "unknown map kernel id %d", kernel);
  if (n == 0) return SIMOPT_OK;
  k_map<<<elementwise_grid(n), 256, 0, as_stream(stream)>>>(kernel, x, n, out);
  SIMOPT_CHECK_LAUNCH("k_map");
  return SIMOPT_OK;
}

namespace {
// out = x * alpha - y (y may be NULL): the epilogues `col_sums * (1.0 / n)`
// (tasks.py:62) and `gq * (1.0 / (N - 1)) - mean` (tasks.py:85), unfused.
__global__ void k_scale_sub(const double* __restrict__ x, double alpha, const double* __restrict__ y,
                            int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double t = x[i] * alpha;
    out[i] = y ? t - y[i] : t;
  }
}
}  // namespace

extern "C" int simopt_scale_sub(void* stream, const double* x, double alpha, const double* y,
                                int64_t n, double* out) {
  if (n == 0) return SIMOPT_OK;
  k_scale_sub<<<elementwise_grid(n), 256, 0, as_stream(stream)>>>(x, alpha, y, n, out);
  SIMOPT_CHECK_LAUNCH("k_scale_sub");
  return SIMOPT_OK;
}

extern "C" int simopt_axpy_ptr(void* stream, const double* alpha, const double* x, const double* y,
                               int64_t n, double* out) {
  if (n == 0) return SIMOPT_OK;
  k_axpy_ptr<<<elementwise_grid(n), 256, 0, as_stream(stream)>>>(alpha, x, y, n, out);
  SIMOPT_CHECK_LAUNCH("k_axpy_ptr");
  return SIMOPT_OK;
}
