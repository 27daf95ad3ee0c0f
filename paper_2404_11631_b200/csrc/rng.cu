// Counter-based sampling kernels: uniform01, standard_normal, diag-Gaussian returns.
//
// Reference: sobench/sampling.py:51-170 (RngStream, uniform01, standard_normal,
// sample_returns) and _kernels.py:178-190 (boxmuller_block).  One thread owns one
// Philox4x64-10 block, i.e. 4 consecutive uniforms = 2 Box-Muller pairs = 4
// consecutive normals; nothing is staged through HBM but the output.
#include "common.cuh"
#include "glibc_math.cuh"
#include "glibc_tables.h"
#include "philox.cuh"
#include "rng_device.cuh"

namespace {

__global__ void __launch_bounds__(256) k_uniform01(uint64_t seed, uint64_t sid, uint64_t clo,
                                                   uint64_t chi, int64_t n, double* __restrict__ out) {
  const int64_t nblk = (n + 3) >> 2;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nblk;
       b += (int64_t)gridDim.x * blockDim.x) {
    const phx4 w = philox4x64_10(stream_block_counter(clo, chi, b), seed, sid);
    const int64_t e = b << 2;
    if (e + 4 <= n) {
      double2* o = reinterpret_cast<double2*>(out + e);
      o[0] = make_double2(phx_u01(w.v[0]), phx_u01(w.v[1]));
      o[1] = make_double2(phx_u01(w.v[2]), phx_u01(w.v[3]));
    } else {
      for (int k = 0; e + k < n; ++k) out[e + k] = phx_u01(w.v[k]);
    }
  }
}

// Normals e0 .. e0+n-1 of the stream (optionally affine per column: mu[j] + sigma[j]*z,
// j = e % d), written to out[e - e0].  e0 > 0 addresses a row shard of a larger draw
// (sample sharding): the values are those of the full draw.
// kNoCarry (checked on the host: the launch's counters clo + b + 1 stay in word 0): the
// Philox round keys come from the constant bank, rounds 0-1 use the launch-constant word 1
// (phx_pre), and round 0's product is carried from one grid-stride block to the next by a
// 128-bit add -- the resample's 17-product core.  The affine column index j = e % d is
// formed once per thread and advanced by the stride's residue.
template <bool kAffine, bool kNoCarry>
__global__ void __launch_bounds__(256) k_normal(const phx_keys rk, const phx_pre pre, uint64_t seed,
                                                uint64_t sid, uint64_t clo, uint64_t chi,
                                                int64_t e0, int64_t n, int64_t d,
                                                const double* __restrict__ mu,
                                                const double* __restrict__ sigma,
                                                double* __restrict__ out) {
  __shared__ double tab[SIMOPT_SINCOSTAB_N];
  load_sincostab(tab);
  const int64_t b0 = e0 >> 2;
  const int64_t e1 = e0 + n;
  const int64_t nblk = ((e1 + 3) >> 2) - b0;
  const bool aligned = (e0 & 3) == 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t bi0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  uint64_t r0h = 0, r0l = 0, sh = 0, sl = 0;
  if (kNoCarry) {
    phx_mulhilo(PHILOX_M0, clo + (uint64_t)(b0 + bi0) + 1, &r0h, &r0l);
    phx_mulhilo(PHILOX_M0, (uint64_t)stride, &sh, &sl);
  }
  int64_t j = 0, jstep = 0;  // affine column of the block's first element, and its advance
  if (kAffine) {
    j = ((b0 + bi0) << 2) % d;
    jstep = (stride << 2) % d;
  }
  for (int64_t bi = bi0; bi < nblk; bi += stride) {
    const int64_t b = b0 + bi;
    double z[4];
    if (kNoCarry) {
      const phx4 w = philox4x64_10_rk_r0(r0h, r0l, rk, pre);
      asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(r0l), "+l"(r0h) : "l"(sl), "l"(sh));
      glibc_boxmuller_fast(phx_u01(w.v[0]), phx_u01(w.v[1]), tab, &z[0], &z[1]);
      glibc_boxmuller_fast(phx_u01(w.v[2]), phx_u01(w.v[3]), tab, &z[2], &z[3]);
    } else {
      normals4(seed, sid, clo, chi, b, tab, z);
    }
    const int64_t e = b << 2;
    if (kAffine) {
      int64_t jj = j;
      for (int k = 0; k < 4; ++k) {
        z[k] = mu[jj] + sigma[jj] * z[k];
        if (++jj == d) jj = 0;
      }
      j += jstep;
      if (j >= d) j -= d;
    }
    if (aligned && e + 4 <= e1) {  // evict-first: a double-buffered draw must not push the
      // X the running epoch re-reads out of L2 (C1: 80 MB, read by every FW iteration)
      double2* o = reinterpret_cast<double2*>(out + (e - e0));
      __stcs(o, make_double2(z[0], z[1]));
      __stcs(o + 1, make_double2(z[2], z[3]));
    } else {
      for (int k = 0; k < 4; ++k)
        if (e + k >= e0 && e + k < e1) out[e + k - e0] = z[k];
    }
  }
}

// Launch k_normal for blocks b0 .. b0+nb-1 (the no-carry path when it applies).
// (128-thread blocks, which fit beside the persistent mean-variance epoch kernel, measured
// 1% slower alone and no better in the pipeline: the co-running draw is starved of warps)
constexpr int kNormalThreads = 256;

template <bool kAffine>
void launch_normal(cudaStream_t st, int64_t nblk, uint64_t seed, uint64_t sid, uint64_t clo, uint64_t chi,
                   int64_t e0, int64_t n, int64_t d, const double* mu, const double* sigma, double* out) {
  const phx_keys rk = phx_round_keys(seed, sid);
  const phx_pre pre = phx_precompute(chi, rk);
  const uint64_t last = (uint64_t)((e0 + n + 3) >> 2);  // counters clo + 1 .. clo + last
  const int64_t want = ceil_div(nblk, kNormalThreads), cap = (int64_t)SIMOPT_NUM_SMS * 8;
  const int grid = (int)(want < cap ? (want > 0 ? want : 1) : cap);
  if (phx_no_carry(clo, last))
    k_normal<kAffine, true><<<grid, kNormalThreads, 0, st>>>(rk, pre, seed, sid, clo, chi, e0, n, d, mu,
                                                            sigma, out);
  else
    k_normal<kAffine, false><<<grid, kNormalThreads, 0, st>>>(rk, pre, seed, sid, clo, chi, e0, n, d, mu,
                                                             sigma, out);
}

int grid_for(int64_t nblk) {
  const int64_t want = ceil_div(nblk, 256);
  const int64_t cap = (int64_t)SIMOPT_NUM_SMS * 8;
  return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

}  // namespace

extern "C" int simopt_uniform01(void* stream, uint64_t seed, uint64_t sid, uint64_t clo,
                                uint64_t chi, int64_t n, double* out) {
  SIMOPT_REQUIRE(n > 0, SIMOPT_E_EMPTY, "requested %lld uniforms", (long long)n);
  k_uniform01<<<grid_for((n + 3) / 4), 256, 0, as_stream(stream)>>>(seed, sid, clo, chi, n, out);
  SIMOPT_CHECK_LAUNCH("k_uniform01");
  return SIMOPT_OK;
}

extern "C" int simopt_standard_normal(void* stream, uint64_t seed, uint64_t sid, uint64_t clo,
                                      uint64_t chi, int64_t n, double* out) {
  SIMOPT_REQUIRE(n > 0, SIMOPT_E_EMPTY, "requested %lld normals", (long long)n);
  launch_normal<false>(as_stream(stream), (n + 3) / 4, seed, sid, clo, chi, 0, n, 1, nullptr, nullptr, out);
  SIMOPT_CHECK_LAUNCH("k_normal");
  return SIMOPT_OK;
}

extern "C" int simopt_sample_returns_diag(void* stream, uint64_t seed, uint64_t sid, uint64_t clo,
                                          uint64_t chi, int64_t n_samples, int64_t d,
                                          const double* mu, const double* sigma, double* out) {
  SIMOPT_REQUIRE(n_samples >= 2, SIMOPT_E_INSUFFICIENT,
                 "need at least 2 samples for a sample covariance, got %lld", (long long)n_samples);
  SIMOPT_REQUIRE(d >= 1, SIMOPT_E_DIMENSION, "empty return dimension");
  const int64_t n = n_samples * d;
  launch_normal<true>(as_stream(stream), (n + 3) / 4, seed, sid, clo, chi, 0, n, d, mu, sigma, out);
  SIMOPT_CHECK_LAUNCH("k_normal<affine>");
  return SIMOPT_OK;
}

extern "C" int simopt_sample_returns_diag_rows(void* stream, uint64_t seed, uint64_t sid,
                                               uint64_t clo, uint64_t chi, int64_t row_lo,
                                               int64_t row_hi, int64_t d, const double* mu,
                                               const double* sigma, double* out) {
  SIMOPT_REQUIRE(d >= 1, SIMOPT_E_DIMENSION, "empty return dimension");
  SIMOPT_REQUIRE(0 <= row_lo && row_lo <= row_hi, SIMOPT_E_CONFIG, "bad row range");
  const int64_t n = (row_hi - row_lo) * d;
  if (n == 0) return SIMOPT_OK;
  launch_normal<true>(as_stream(stream), (n + 3) / 4 + 1, seed, sid, clo, chi, row_lo * d, n, d, mu, sigma,
                      out);
  SIMOPT_CHECK_LAUNCH("k_normal<affine,rows>");
  return SIMOPT_OK;
}

namespace {
// synth_classification features (sampling.py:246-255): x = (u >= 0.5), i.e. the MSB
// of the Philox word, written as 0.0 / 1.0.
__global__ void __launch_bounds__(256) k_bernoulli_half(uint64_t seed, uint64_t sid, uint64_t clo,
                                                        uint64_t chi, int64_t e0, int64_t n,
                                                        double* __restrict__ out) {
  const int64_t b0 = e0 >> 2, e1 = e0 + n;
  const int64_t nblk = ((e1 + 3) >> 2) - b0;
  for (int64_t bi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; bi < nblk;
       bi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = b0 + bi;
    const phx4 w = philox4x64_10(stream_block_counter(clo, chi, b), seed, sid);
    const int64_t e = b << 2;
    for (int k = 0; k < 4; ++k)
      if (e + k >= e0 && e + k < e1) out[e + k - e0] = (w.v[k] >> 63) ? 1.0 : 0.0;
  }
}

// labels = (scores > median).astype(float64) (sampling.py:261)
__global__ void k_threshold(const double* __restrict__ x, double thr, int64_t n,
                            double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (x[i] > thr) ? 1.0 : 0.0;
}
}  // namespace

extern "C" int simopt_bernoulli_half(void* stream, uint64_t seed, uint64_t sid, uint64_t clo,
                                     uint64_t chi, int64_t n, double* out) {
  SIMOPT_REQUIRE(n > 0, SIMOPT_E_EMPTY, "requested %lld draws", (long long)n);
  k_bernoulli_half<<<grid_for((n + 3) / 4), 256, 0, as_stream(stream)>>>(seed, sid, clo, chi, 0, n,
                                                                         out);
  SIMOPT_CHECK_LAUNCH("k_bernoulli_half");
  return SIMOPT_OK;
}

extern "C" int simopt_bernoulli_half_range(void* stream, uint64_t seed, uint64_t sid, uint64_t clo,
                                           uint64_t chi, int64_t e_lo, int64_t e_hi, double* out) {
  SIMOPT_REQUIRE(0 <= e_lo && e_lo <= e_hi, SIMOPT_E_CONFIG, "bad element range");
  const int64_t n = e_hi - e_lo;
  if (n == 0) return SIMOPT_OK;
  k_bernoulli_half<<<grid_for((n + 3) / 4 + 1), 256, 0, as_stream(stream)>>>(seed, sid, clo, chi,
                                                                             e_lo, n, out);
  SIMOPT_CHECK_LAUNCH("k_bernoulli_half<range>");
  return SIMOPT_OK;
}

extern "C" int simopt_threshold(void* stream, const double* x, double thr, int64_t n, double* out) {
  if (n == 0) return SIMOPT_OK;
  k_threshold<<<grid_for((n + 3) / 4), 256, 0, as_stream(stream)>>>(x, thr, n, out);
  SIMOPT_CHECK_LAUNCH("k_threshold");
  return SIMOPT_OK;
}

// --- measurement: the Philox-only floor of the newsvendor resample ---------------------
// Blocks clo+1 .. clo+n of key (seed, sid) through the resample's own Philox core (round 0
// carried by a 128-bit add, 17 products per block), words XOR-folded into out[thread] so
// nothing is stored per block: the heavy-FMA-pipe time a resample of n blocks cannot beat.
namespace {
constexpr int kFloorThreads = 256;
__global__ void __launch_bounds__(kFloorThreads) k_philox_floor(const phx_keys rk, const phx_pre pre,
                                                                 uint64_t clo, int64_t n,
                                                                 uint64_t* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * kFloorThreads;
  const int64_t t0 = (int64_t)blockIdx.x * kFloorThreads + threadIdx.x;
  uint64_t acc = 0, h0 = 0, l0 = 0;
  if (t0 < n) phx_mulhilo(PHILOX_M0, clo + 1 + (uint64_t)t0, &h0, &l0);
  const uint64_t sl = (uint64_t)stride * PHILOX_M0;  // M0 * stride mod 2^128, formed once
  const uint64_t sh = __umul64hi((uint64_t)stride, PHILOX_M0);
  for (int64_t t = t0; t < n; t += stride) {
    const phx4 w = philox4x64_10_rk_r0(h0, l0, rk, pre);
    acc ^= w.v[0] ^ w.v[1] ^ w.v[2] ^ w.v[3];
    asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(l0), "+l"(h0) : "l"(sl), "l"(sh));
  }
  out[t0] = acc;
}
}  // namespace

extern "C" int simopt_philox_floor(void* stream, uint64_t seed, uint64_t sid, uint64_t clo,
                                   int64_t nblocks, uint64_t* out, int64_t out_len) {
  SIMOPT_REQUIRE(nblocks > 0, SIMOPT_E_EMPTY, "requested %lld blocks", (long long)nblocks);
  SIMOPT_REQUIRE(phx_no_carry(clo, (uint64_t)nblocks), SIMOPT_E_CONFIG, "counter would carry");
  const int grid = 8 * SIMOPT_NUM_SMS;
  SIMOPT_REQUIRE(out_len >= (int64_t)grid * kFloorThreads, SIMOPT_E_CONFIG,
                 "out needs %lld words", (long long)grid * kFloorThreads);
  const phx_keys rk = phx_round_keys(seed, sid);
  k_philox_floor<<<grid, kFloorThreads, 0, as_stream(stream)>>>(rk, phx_precompute(0, rk), clo,
                                                               nblocks, out);
  SIMOPT_CHECK_LAUNCH("k_philox_floor");
  return SIMOPT_OK;
}
