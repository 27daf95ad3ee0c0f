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

// Exact-tree row dots over bits: partial of (row r, column chunk c) = v_j summed over the
// set bits j of the chunk in increasing order (p[c * rows + r]), folded afterwards.
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
    for (int64_t w = lo >> 6; w <= (hi - 1) >> 6; ++w) {
      uint64_t m = row[w];
      const int64_t base = w << 6;
      if (base < lo) m &= ~0ULL << (lo - base);                  // chunk starts mid-word
      if (hi - base < 64) m &= (hi - base >= 64) ? ~0ULL : ((1ULL << (hi - base)) - 1ULL);
      while (m) {
        const int b = __ffsll((long long)m) - 1;
        s = s + v[base + b];
        m &= m - 1;
      }
    }
    p[c * rows + r] = s;
  }
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

extern "C" int simopt_matvec_bits(void* stream, const uint64_t* bits, int64_t rows, int64_t d,
                                  const double* v, int64_t chunk, double* out) {
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
  k_matvec_bits<<<grid_for(rows * nch, 128), 128, 0, st>>>(bits, rows, d, W, v, chunk, nch, p);
  SIMOPT_CHECK_LAUNCH("k_matvec_bits");
  if (nch > 1) return simopt_fold_partials(stream, p, nch, rows, out);
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
