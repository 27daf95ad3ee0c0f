// Explicit logistic Hessian H = (1/N) X^T diag(D) X on the FP64 tensor pipe (DMMA).
//
// Not in the reference package: its oracle is tests/test_tasks.py:292-304
// (`(x.T * (c*(1-c))) @ x / N`, numpy BLAS, any summation order), and the
// parity bar is rtol 1e-10.  BASELINE.json configs[4] (d = 8192, N = 10^7) is the
// only dense contraction on the path.  tcgen05 has no f64 kind, so the tensor
// path is the warp-level mma.sync.m8n8k4.f64 (SASS DMMA).
//
// Tiling: one CTA owns a 64x64 tile of H (symmetric: only tiles with bj <= bk
// are computed, the transpose is mirrored by the epilogue); 4 warps each own a
// 32x32 quadrant = 4x4 m8n8 accumulators.  The sample axis is the GEMM K axis:
// 16-row slabs of X (the j- and the k-columns) and of D are staged through shared
// memory, double-buffered with cp.async (zero-fill past the edges); D_i scales
// the B fragment as it is loaded (the oracle's summation order is BLAS's, so
// only the 1e-10 tolerance binds).
#include "common.cuh"

namespace {

constexpr int kTile = 64;   // H tile
constexpr int kSlab = 16;   // samples per smem stage
constexpr int kPad = 2;     // row padding (doubles) against bank conflicts

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

// kBits: x is the bit-packed binary design matrix (csrc/bits.cu layout, W words per
// row); a 64-column tile block is exactly one word, so a slab stages 16 words per
// operand and the DMMA fragments are expanded (0.0 / 1.0) in registers.
template <bool kBits>
__global__ void __launch_bounds__(128) k_xtdx(const double* __restrict__ x,
                                              const uint64_t* __restrict__ xb, int64_t W,
                                              const double* __restrict__ dw, int64_t n, int64_t d,
                                              double scale, double* __restrict__ h) {
  // map blockIdx.x -> (bj, bk) with bj <= bk
  const int nt = (int)((d + kTile - 1) / kTile);
  int t = blockIdx.x, bj = 0;
  while (t >= nt - bj) { t -= nt - bj; ++bj; }
  const int bk = bj + t;
  const int64_t j0 = (int64_t)bj * kTile, k0 = (int64_t)bk * kTile;

  __shared__ __align__(16) double As[2][kSlab][kTile + kPad];
  __shared__ __align__(16) double Bs[2][kSlab][kTile + kPad];
  __shared__ __align__(16) double Ds[2][kSlab];
  __shared__ __align__(16) uint64_t Aw[2][kSlab], Bw[2][kSlab];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;  // warp quadrant inside the tile
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  auto stage = [&](int buf, int64_t i0) {
    if (kBits) {
      if (threadIdx.x < 2 * kSlab) {
        const int r = threadIdx.x & (kSlab - 1);
        const int64_t i = i0 + r;
        const int64_t wcol = (threadIdx.x < kSlab ? j0 : k0) >> 6;
        cp_async8(threadIdx.x < kSlab ? (void*)&Aw[buf][r] : (void*)&Bw[buf][r],
                  xb + (i < n ? i : 0) * W + wcol, i < n);
      }
    }
    for (int e = threadIdx.x; !kBits && e < kSlab * kTile; e += blockDim.x) {
      const int r = e / kTile, c = e % kTile;
      const int64_t i = i0 + r;
      const bool vi = i < n;
      const int64_t ii = vi ? i : 0;
      cp_async8(&As[buf][r][c], x + ii * d + (j0 + c < d ? j0 + c : 0), vi && j0 + c < d);
      cp_async8(&Bs[buf][r][c], x + ii * d + (k0 + c < d ? k0 + c : 0), vi && k0 + c < d);
    }
    if (threadIdx.x < kSlab) {
      const int64_t i = i0 + threadIdx.x;
      cp_async8(&Ds[buf][threadIdx.x], dw + (i < n ? i : 0), i < n);
    }
    cp_async_commit();
  };

  const int64_t nslab = (n + kSlab - 1) / kSlab;
  stage(0, 0);
  for (int64_t s = 0; s < nslab; ++s) {
    const int buf = (int)(s & 1);
    if (s + 1 < nslab) {
      stage(buf ^ 1, (s + 1) * kSlab);
      cp_async_wait1();
    } else {
      cp_async_wait0();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kSlab; kk += 4) {
      // A frag (8x4 row-major = X^T):  a = X[kk + lane%4][wm + 8mi + lane/4]
      // B frag (4x8 col-major):        b = D[kk + lane%4] * X[kk + lane%4][wn + 8ni + lane/4]
      const int kr = kk + (lane & 3);
      const double di = Ds[buf][kr];
      double af[4], bf[4];
      if (kBits) {
        const uint64_t aw = Aw[buf][kr], bw = Bw[buf][kr];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) af[mi] = ((aw >> (wm + mi * 8 + (lane >> 2))) & 1ULL) ? 1.0 : 0.0;
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) bf[ni] = ((bw >> (wn + ni * 8 + (lane >> 2))) & 1ULL) ? di : 0.0;
      } else {
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) af[mi] = As[buf][kr][wm + mi * 8 + (lane >> 2)];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) bf[ni] = di * Bs[buf][kr][wn + ni * 8 + (lane >> 2)];
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
    __syncthreads();
  }
  // epilogue: C frag element (row = lane/4, col = 2*(lane%4) + e); write tile and its mirror
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t r = j0 + wm + mi * 8 + (lane >> 2);
        const int64_t c = k0 + wn + ni * 8 + 2 * (lane & 3) + e;
        if (r < d && c < d) {
          const double v = acc[mi][ni][e] * scale;
          h[r * d + c] = v;
          h[c * d + r] = v;
        }
      }
}

}  // namespace

extern "C" int simopt_logistic_xtdx(void* stream, const double* x, const double* dw, int64_t n,
                                    int64_t d, double* h) {
  SIMOPT_REQUIRE(n >= 1 && d >= 1, SIMOPT_E_DIMENSION, "empty design matrix");
  const int64_t nt = (d + kTile - 1) / kTile;
  const int64_t tiles = nt * (nt + 1) / 2;
  SIMOPT_REQUIRE(tiles < (1LL << 31), SIMOPT_E_CONFIG, "d too large");
  k_xtdx<false><<<(unsigned)tiles, 128, 0, as_stream(stream)>>>(x, nullptr, 0, dw, n, d,
                                                                1.0 / (double)n, h);
  SIMOPT_CHECK_LAUNCH("k_xtdx");
  return SIMOPT_OK;
}

// Same Hessian from bit-packed binary features (csrc/bits.cu): H = (1/n) X^T diag(dw) X.
extern "C" int simopt_logistic_xtdx_bits(void* stream, const uint64_t* xbits, const double* dw,
                                         int64_t n, int64_t d, double* h) {
  SIMOPT_REQUIRE(n >= 1 && d >= 1, SIMOPT_E_DIMENSION, "empty design matrix");
  const int64_t nt = (d + kTile - 1) / kTile;
  const int64_t tiles = nt * (nt + 1) / 2;
  SIMOPT_REQUIRE(tiles < (1LL << 31), SIMOPT_E_CONFIG, "d too large");
  k_xtdx<true><<<(unsigned)tiles, 128, 0, as_stream(stream)>>>(nullptr, xbits, (d + 63) / 64, dw, n,
                                                               d, 1.0 / (double)n, h);
  SIMOPT_CHECK_LAUNCH("k_xtdx<bits>");
  return SIMOPT_OK;
}
