// Bit-packed binary features for the classification task.
//
// synth_classification's features are exactly 0/1: X[i,j] = [u >= 0.5], the MSB of a
// Philox4x64-10 word (sobench/sampling.py:246-255).  Stored as fp64 (the reference's
// layout) config 5 (N = 10^7, d = 8192) needs 655 GB; as bits it needs 10 GB, so it
// fits one B200 per shard at any of 1/2/4/8 GPUs, and every streaming pass reads 1/64
// of the bytes.  Layout: row-major, W = ceil(d/64) u64 words per row, feature j of row
// i is bit (j & 63) of word (i, j >> 6); padding bits are 0.
//
// Arithmetic on bits is the fp64 arithmetic on 0.0/1.0: x*v is v or +-0, and adding
// +-0 never changes a running sum that starts at +0 (round-to-nearest), so a chain
// that adds v_j over the set bits in column order is bit-identical to the reference's
// fixed-tree chain over all columns (_kernels.py:71-121).
#include "common.cuh"
#include "philox.cuh"
#include "rng_device.cuh"

extern "C" int simopt_fold_partials(void* stream, double* p, int64_t nch, int64_t count, double* out);

namespace {

// words (r, w) of rows [row_lo, row_lo + nrows): bit b = MSB of element (row_lo+r)*d + 64w + b
__global__ void __launch_bounds__(256) k_bernoulli_bits(uint64_t seed, uint64_t sid, uint64_t clo,
                                                        uint64_t chi, int64_t row_lo, int64_t nrows,
                                                        int64_t d, int64_t W,
                                                        uint64_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nrows * W;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / W, w = t - r * W;
    const int64_t c0 = 64 * w;
    const int nb = (int)(d - c0 < 64 ? d - c0 : 64);
    const int64_t e0 = (row_lo + r) * d + c0;
    uint64_t bits = 0;
    int64_t q = -1;
    phx4 blk;
    for (int b = 0; b < nb; ++b) {
      const int64_t e = e0 + b;
      if ((e >> 2) != q) {
        q = e >> 2;
        blk = philox4x64_10(stream_block_counter(clo, chi, (uint64_t)q), seed, sid);
      }
      bits |= (blk.v[e & 3] >> 63) << b;
    }
    out[t] = bits;
  }
}

constexpr int kMbRows = 128;
constexpr int kMbSlab = 16;
// s + x*t with x = bit ? 1.0 : 0.0 as one DFMA: the product is exact (t or +-0), so the
// fused result is the reference's s + (x*t) bit for bit -- including x = 0 with t = +-inf
// or NaN, where the reference's 0.0*t is NaN as well.  Adding +-0 leaves every sum that
// starts at +0.0 unchanged (it never becomes -0.0).
__device__ __forceinline__ void add_if_set(double& s, double t, uint32_t bit) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 hi;\n\t.reg .f64 x;\n\t"
      "setp.ne.u32 p, %2, 0;\n\tselp.b32 hi, 0x3FF00000, 0, p;\n\t"
      "mov.b64 x, {0, hi};\n\tfma.rn.f64 %0, x, %1, %0;\n\t}"
      : "+d"(s) : "d"(t), "r"(bit));
}
// Exact-tree row dots over bits, any chunk size (the slab kernel below needs chunk % 64 == 0):
// partial of (row r, column chunk c) = the chain over the chunk's columns in increasing
// order (p[c * rows + r]), folded afterwards.
__global__ void __launch_bounds__(128) k_matvec_bits(const uint64_t* __restrict__ bits, int64_t rows,
                                                     int64_t d, int64_t W,
                                                     const double* __restrict__ v, int64_t chunk,
                                                     int64_t nch, double* __restrict__ p) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * nch;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / rows, r = t - c * rows;
    const int64_t lo = c * chunk, hi = lo + chunk < d ? lo + chunk : d;
    const uint64_t* row = bits + r * W;
    double s = 0.0;
    for (int64_t j = lo; j < hi; ++j)
      add_if_set(s, v[j], (uint32_t)(row[j >> 6] >> (j & 63)) & 1u);
    p[c * rows + r] = s;
  }
}

// Exact-tree row dots, slab-staged (chunk % 64 == 0): one row per thread, 128 rows per block.
// A slab of 16 words x 128 rows is staged in shared memory with coalesced loads (row
// stride 17 words: conflict-free per-thread reads), its 1024 v entries beside it; each
// thread then walks its row's bits in column order with one DFMA per column (add_if_set)
// and v broadcast from shared memory -- no per-lane gather, no divergence.  The chain per
// row is the reference's: s = s + v_j over the set bits j, restarted at every chunk
// boundary (partial p[c * rows + r]).  rows_idx (nullable) gathers batch rows.
__global__ void __launch_bounds__(kMbRows) k_matvec_bits_slab(const uint64_t* __restrict__ bits,
                                                              int64_t W, int64_t d,
                                                              const int64_t* __restrict__ idx,
                                                              int64_t rows,
                                                              const double* __restrict__ v,
                                                              int64_t cw, int64_t nch,
                                                              double* __restrict__ p) {
  __shared__ uint64_t sb[kMbRows * (kMbSlab + 1)];
  __shared__ __align__(16) double sv[kMbSlab * 64];
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * kMbRows, r = r0 + tid;
  double s = 0.0;
  int64_t next_cut = cw, c = 0;
  for (int64_t w0 = 0; w0 < W; w0 += kMbSlab) {
    const int nw = (int)(W - w0 < kMbSlab ? W - w0 : kMbSlab);
    __syncthreads();
    for (int e = tid; e < kMbRows * nw; e += kMbRows) {
      const int rr = e / nw, ww = e - rr * nw;
      const int64_t row = r0 + rr;
      uint64_t x = 0;
      if (row < rows) x = bits[(idx ? idx[row] : row) * W + w0 + ww];
      sb[rr * (kMbSlab + 1) + ww] = x;
    }
    for (int e = tid; e < nw * 64; e += kMbRows) {
      const int64_t j = w0 * 64 + e;
      sv[e] = j < d ? v[j] : 0.0;
    }
    __syncthreads();
    for (int ww = 0; ww < nw; ++ww) {
      if (w0 + ww == next_cut) {  // chunk boundary: the chain restarts
        if (r < rows) p[c * rows + r] = s;
        s = 0.0;
        ++c;
        next_cut += cw;
      }
      const uint64_t m = sb[tid * (kMbSlab + 1) + ww];
      const uint32_t halves[2] = {(uint32_t)m, (uint32_t)(m >> 32)};
      const double2* vv = reinterpret_cast<const double2*>(sv + ww * 64);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t q = halves[h];
#pragma unroll
        for (int b = 0; b < 16; ++b) {
          const double2 t = vv[h * 16 + b];
          add_if_set(s, t.x, q & (1u << (2 * b)));
          add_if_set(s, t.y, q & (1u << (2 * b + 1)));
        }
      }
    }
  }
  if (r < rows) p[c * rows + r] = s;
  (void)nch;
}

// Exact-tree column sums over bits: partial (column j, row chunk c) = the chain over the
// chunk's rows i (in order, through rows_idx when given) of x_ij * x_i.  One
// column per thread; the 64 threads of a word read the same u64 (broadcast).
__global__ void __launch_bounds__(128) k_matvec_t_bits(const uint64_t* __restrict__ bits, int64_t W,
                                                       int64_t d, const int64_t* __restrict__ idx,
                                                       int64_t rows, const double* __restrict__ x,
                                                       int64_t chunk, double* __restrict__ p) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, c = blockIdx.y;
  if (j >= d) return;
  const int64_t lo = c * chunk, hi = lo + chunk < rows ? lo + chunk : rows;
  const int64_t wj = j >> 6;
  const uint64_t bit = 1ULL << (j & 63);
  double s = 0.0;
  for (int64_t i = lo; i < hi; ++i) {
    const int64_t row = idx ? idx[i] : i;
    add_if_set(s, x[i], (uint32_t)((bits[row * W + wj] & bit) != 0));
  }
  p[c * d + j] = s;
}

__global__ void k_unpack_bits(const uint64_t* __restrict__ bits, int64_t rows, int64_t d, int64_t W,
                              double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * d;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / d, j = e - r * d;
    out[e] = ((bits[r * W + (j >> 6)] >> (j & 63)) & 1ULL) ? 1.0 : 0.0;
  }
}

int grid_for(int64_t n, int per) {
  const int64_t g = ceil_div(n, per), cap = (int64_t)SIMOPT_NUM_SMS * 16;
  return (int)(g < 1 ? 1 : (g < cap ? g : cap));
}

}  // namespace

extern "C" int simopt_bernoulli_bits(void* stream, uint64_t seed, uint64_t sid, uint64_t clo,
                                     uint64_t chi, int64_t row_lo, int64_t row_hi, int64_t d,
                                     uint64_t* out) {
  SIMOPT_REQUIRE(d >= 1 && 0 <= row_lo && row_lo <= row_hi, SIMOPT_E_CONFIG, "bad bit-matrix extent");
  const int64_t W = ceil_div(d, 64), n = (row_hi - row_lo) * W;
  if (n == 0) return SIMOPT_OK;
  k_bernoulli_bits<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(seed, sid, clo, chi, row_lo,
                                                                    row_hi - row_lo, d, W, out);
  SIMOPT_CHECK_LAUNCH("k_bernoulli_bits");
  return SIMOPT_OK;
}

extern "C" int simopt_matvec_bits_idx(void* stream, const uint64_t* bits, int64_t total_rows,
                                      int64_t d, const int64_t* idx, int64_t rows, const double* v,
                                      int64_t chunk, double* out) {
  (void)total_rows;
  SIMOPT_REQUIRE(chunk >= 1, SIMOPT_E_CONFIG, "chunk_size must be >= 1");
  cudaStream_t st = as_stream(stream);
  if (rows == 0) return SIMOPT_OK;
  if (d == 0) {
    SIMOPT_CUDA(cudaMemsetAsync(out, 0, rows * sizeof(double), st));
    return SIMOPT_OK;
  }
  const int64_t W = ceil_div(d, 64), nch = ceil_div(d, chunk);
  double* p = out;
  if (nch > 1) {
    p = static_cast<double*>(simopt_scratch(st, rows * nch * sizeof(double)));
    SIMOPT_REQUIRE(p != nullptr, SIMOPT_E_CUDA, "%s", simopt_last_error());
  }
  if (chunk % 64 == 0) {
    k_matvec_bits_slab<<<(unsigned)ceil_div(rows, kMbRows), kMbRows, 0, st>>>(bits, W, d, idx, rows,
                                                                                v, chunk / 64, nch, p);
    SIMOPT_CHECK_LAUNCH("k_matvec_bits_slab");
  } else {
    SIMOPT_REQUIRE(idx == nullptr, SIMOPT_E_CONFIG, "row gather over bits needs chunk %% 64 == 0");
    k_matvec_bits<<<grid_for(rows * nch, 128), 128, 0, st>>>(bits, rows, d, W, v, chunk, nch, p);
    SIMOPT_CHECK_LAUNCH("k_matvec_bits");
  }
  if (nch > 1) return simopt_fold_partials(stream, p, nch, rows, out);
  return SIMOPT_OK;
}

extern "C" int simopt_matvec_bits(void* stream, const uint64_t* bits, int64_t rows, int64_t d,
                                  const double* v, int64_t chunk, double* out) {
  return simopt_matvec_bits_idx(stream, bits, rows, d, nullptr, rows, v, chunk, out);
}

extern "C" int simopt_matvec_t_bits(void* stream, const uint64_t* bits, int64_t total_rows,
                                    int64_t d, const int64_t* idx, int64_t rows, const double* x,
                                    int64_t chunk, double* out) {
  (void)total_rows;
  SIMOPT_REQUIRE(chunk >= 1, SIMOPT_E_CONFIG, "chunk_size must be >= 1");
  cudaStream_t st = as_stream(stream);
  if (d == 0) return SIMOPT_OK;
  if (rows == 0) {
    SIMOPT_CUDA(cudaMemsetAsync(out, 0, d * sizeof(double), st));
    return SIMOPT_OK;
  }
  const int64_t nch = ceil_div(rows, chunk);
  SIMOPT_REQUIRE(nch < 65536, SIMOPT_E_CONFIG, "too many row chunks (%lld)", (long long)nch);
  double* p = out;
  if (nch > 1) {
    p = static_cast<double*>(simopt_scratch(st, d * nch * sizeof(double)));
    SIMOPT_REQUIRE(p != nullptr, SIMOPT_E_CUDA, "%s", simopt_last_error());
  }
  const dim3 grid((unsigned)ceil_div(d, 128), (unsigned)nch);
  k_matvec_t_bits<<<grid, 128, 0, st>>>(bits, ceil_div(d, 64), d, idx, rows, x, chunk, p);
  SIMOPT_CHECK_LAUNCH("k_matvec_t_bits");
  if (nch > 1) return simopt_fold_partials(stream, p, nch, d, out);
  return SIMOPT_OK;
}

extern "C" int simopt_unpack_bits(void* stream, const uint64_t* bits, int64_t rows, int64_t d,
                                  double* out) {
  if (rows == 0 || d == 0) return SIMOPT_OK;
  k_unpack_bits<<<grid_for(rows * d, 256), 256, 0, as_stream(stream)>>>(bits, rows, d,
                                                                       ceil_div(d, 64), out);
  SIMOPT_CHECK_LAUNCH("k_unpack_bits");
  return SIMOPT_OK;
}
