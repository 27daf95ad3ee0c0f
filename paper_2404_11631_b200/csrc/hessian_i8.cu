// Explicit logistic Hessian H = (1/n) X^T diag(dw) X for BINARY X on the integer tensor
// cores: exact limb decomposition (an Ozaki-style split of dw, possible because X is 0/1).
//
// dw in [0, 1/4] is rounded once to the fixed point q = round(dw * 2^41) <= 2^39 and
// split into five 8-bit limbs L_k = (q >> 8k) & 255.  Then
//     H = (1/n) * sum_k 2^(8k-41) * G_k,     G_k[i][j] = sum_r x_ri * x_rj * L_rk,
// and every G_k is an integer GEMM with u8 operands (x in {0,1}, L_k in [0,255]) and
// exact int32 accumulation (a sample chunk holds <= 2^23 rows: 2^23 * 255 < 2^31).
// The only rounding is the quantisation of dw (<= 2^-42 absolute per term, ~1e-11
// relative on H) and the final fp64 scaling/summation -- inside the 1e-10 tolerance
// of the reference's explicit-Hessian oracle (tests/test_tasks.py:292-304).
//
// Data: X^T as u8 in sample blocks of CH samples, [np/CH][d][CH] (np = rows padded to a
// multiple of CH, CH = 4096 or np when smaller): within a block the 128 feature rows of
// a tile are CH bytes apart, so a k-slab touches a 512 KB window (a flat [d][np] layout
// put them 10 MB apart at C5's N = 10^7 and thrashed the TLB: 2.5x slower per sample).
// Built once per data set from the bit-packed features (csrc/bits.cu).  Kernel: legacy
// warp-level IMMA (mma.sync.m16n8k32.u8.u8.s32 -- measured 963 TOPS on this B200,
// tools/micro/imma.cu, 26x the FP64 DMMA pipe), 128x128 output tiles on the upper
// triangle, 8 warps of 64x32, 32-sample k-slabs in a 3-stage cp.async ring, fragments
// by ldmatrix (48-byte padded rows: conflict-free), the limb applied to the B fragment
// with two integer ops per 4 samples: (b * 255) & L.
#include "common.cuh"

namespace {

constexpr int kBM = 128, kBK = 32, kRS = 48, kStages = 3, kThreads = 256;
constexpr int kLimbs = 5, kLimbBits = 8, kFixBits = 41;
// Samples per launch (<= 2^23 keeps the int32 accumulation exact).
constexpr int64_t kChunk = 1LL << 20;
// Feature rows of a sample block are ch + kRowPad bytes apart: a power-of-two stride would
// map the 128 rows of a tile onto the same L2 sets.
constexpr int64_t kRowPad = 32;

__device__ __forceinline__ void cp16(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(valid ? 16 : 0));
}

__device__ __forceinline__ void ldsm_x4(unsigned (&r)[4], const void* smem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(s));
}

__device__ __forceinline__ void imma(int (&c)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__global__ void __launch_bounds__(kThreads, 2)
    k_xtdx_i8(const uint8_t* __restrict__ xt, int lg_ch, int64_t d, const uint8_t* __restrict__ limb,
              int64_t s0, int64_t s1, double scale, int beta, double* __restrict__ h) {
  const int nt = (int)((d + kBM - 1) / kBM);
  int t = blockIdx.x, bj = 0;
  while (t >= nt - bj) { t -= nt - bj; ++bj; }
  const int bk = bj + t;
  const int64_t i0 = (int64_t)bj * kBM, j0 = (int64_t)bk * kBM;

  __shared__ __align__(128) uint8_t As[kStages][kBM * kRS];
  __shared__ __align__(128) uint8_t Bs[kStages][kBM * kRS];
  __shared__ __align__(16) uint8_t Ls[kStages][kBK];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 2) * 64, wn = (warp & 3) * 32;
  int acc[4][4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0;

  const int64_t nslab = (s1 - s0) / kBK;
  // per-thread constants of the stage copies: this thread's A/B feature rows in a block
  const int64_t ch = 1LL << lg_ch, rs = ch + kRowPad;
  const int srow = tid >> 1, half = tid & 1;
  const bool va = i0 + srow < d, vb = j0 + srow < d;
  const int64_t offa = (va ? i0 + srow : 0) * rs + half * 16;
  const int64_t offb = (vb ? j0 + srow : 0) * rs + half * 16;
  uint8_t* sa = &As[0][srow * kRS + half * 16];
  uint8_t* sb = &Bs[0][srow * kRS + half * 16];
  auto stage = [&](int buf, int64_t s) {
    const uint8_t* blk = xt + (s >> lg_ch) * (d * rs) + (s & (ch - 1));  // sample block of s
    cp16(sa + buf * (kBM * kRS), blk + offa, va);
    cp16(sb + buf * (kBM * kRS), blk + offb, vb);
    if (tid < 2) cp16(&Ls[buf][tid * 16], limb + s + tid * 16, true);
    asm volatile("cp.async.commit_group;\n" ::);
  };
  for (int p = 0; p < kStages - 1; ++p) {
    if (p < nslab) stage(p, s0 + p * kBK);
    else asm volatile("cp.async.commit_group;\n" ::);
  }
  const int q = lane >> 3, rr = lane & 7, tq = lane & 3;
  for (int64_t sl = 0; sl < nslab; ++sl) {
    const int buf = (int)(sl % kStages);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(kStages - 2));
    __syncthreads();
    {  // refill the slot consumed in the previous iteration
      const int64_t nx = sl + kStages - 1;
      if (nx < nslab) stage((int)(nx % kStages), s0 + nx * kBK);
      else asm volatile("cp.async.commit_group;\n" ::);
    }
    const uint8_t* A = As[buf];
    const uint8_t* B = Bs[buf];
    const unsigned L0 = *reinterpret_cast<const unsigned*>(&Ls[buf][4 * tq]);
    const unsigned L1 = *reinterpret_cast<const unsigned*>(&Ls[buf][16 + 4 * tq]);
    unsigned af[4][4], bfr[2][4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
      ldsm_x4(af[mi], A + (wm + 16 * mi + (q & 1) * 8 + rr) * kRS + (q >> 1) * 16);
#pragma unroll
    for (int nj = 0; nj < 2; ++nj)
      ldsm_x4(bfr[nj], B + (wn + 8 * (2 * nj + (q >> 1)) + rr) * kRS + (q & 1) * 16);
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      // B fragment of n8 block ni: k = 4t..4t+3 and 16+4t..; scale x in {0,1} by the limb
      const unsigned b0 = (bfr[ni >> 1][2 * (ni & 1)] * 255u) & L0;
      const unsigned b1 = (bfr[ni >> 1][2 * (ni & 1) + 1] * 255u) & L1;
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) imma(acc[mi][ni], af[mi], b0, b1);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  // epilogue: C frag c0,c1 = (row g, cols 2t, 2t+1), c2,c3 = (row g+8, ...); upper entries
  // (i <= j) and their mirrors
  const int g = lane >> 2;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t i = i0 + wm + 16 * mi + g + (e >> 1) * 8;
        const int64_t j = j0 + wn + 8 * ni + 2 * tq + (e & 1);
        if (i < d && j < d && i <= j) {
          const double v = (double)acc[mi][ni][e] * scale;
          if (beta) {
            h[i * d + j] += v;
            if (i != j) h[j * d + i] += v;
          } else {
            h[i * d + j] = v;
            if (i != j) h[j * d + i] = v;
          }
        }
      }
}

// out[block r/ch][j][r%ch] = bit (r, j) of the packed rows, 0 for r >= rows (16 samples
// per thread)
__global__ void k_bits_to_u8t(const uint64_t* __restrict__ bits, int64_t rows, int64_t d, int64_t W,
                              int64_t np, int64_t ch, uint8_t* __restrict__ out) {
  const int64_t per = np / 16;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < d * per;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t % d, r0 = (t / d) * 16;  // consecutive threads: consecutive features
    uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int64_t r = r0 + k;
      const uint32_t b = r < rows ? (uint32_t)((bits[r * W + (j >> 6)] >> (j & 63)) & 1ULL) : 0u;
      w[k >> 2] |= b << (8 * (k & 3));
    }
    *reinterpret_cast<uint4*>(out + (r0 / ch) * (d * (ch + kRowPad)) + j * (ch + kRowPad) +
                              (r0 % ch)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// limbs[k][r] = byte k of round(dw[r] * 2^41), 0 for r >= n
__global__ void k_limbs(const double* __restrict__ dw, int64_t n, int64_t np, uint8_t* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < np;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint64_t q = 0;
    if (r < n) {
      double v = dw[r];
      v = v < 0.0 ? 0.0 : (v > 0.25 ? 0.25 : v);
      q = (uint64_t)rint(v * 2199023255552.0);  // 2^41: q <= 2^39 (dw = 1/4 at t = 0)
    }
#pragma unroll
    for (int k = 0; k < kLimbs; ++k) out[k * np + r] = (uint8_t)((q >> (kLimbBits * k)) & 255ULL);
  }
}

int egrid(int64_t n) {
  const int64_t g = ceil_div(n, 256), cap = (int64_t)SIMOPT_NUM_SMS * 16;
  return (int)(g < 1 ? 1 : (g < cap ? g : cap));
}

}  // namespace

// Sample-block width ch (a power of two, 32..4096) and padded row count np of the u8
// operand for n rows; the operand occupies (np / ch) * d * (ch + 32) bytes.
extern "C" int simopt_u8t_geometry(int64_t n, int64_t* ch, int64_t* np) {
  int64_t c = 32;
  while (c < 4096 && c < n) c <<= 1;
  *ch = c;
  *np = ceil_div(n < 1 ? 1 : n, c) * c;
  return SIMOPT_OK;
}

extern "C" int simopt_bits_to_u8t(void* stream, const uint64_t* bits, int64_t rows, int64_t d,
                                  int64_t np, uint8_t* out) {
  int64_t ch = 0, np_want = 0;
  simopt_u8t_geometry(rows, &ch, &np_want);
  SIMOPT_REQUIRE(np == np_want, SIMOPT_E_CONFIG, "np must come from simopt_u8t_geometry");
  if (d == 0 || np == 0) return SIMOPT_OK;
  k_bits_to_u8t<<<egrid(d * (np / 16)), 256, 0, as_stream(stream)>>>(bits, rows, d, (d + 63) / 64, np,
                                                                      ch, out);
  SIMOPT_CHECK_LAUNCH("k_bits_to_u8t");
  return SIMOPT_OK;
}

// H = (1/n) X^T diag(dw) X from the u8 feature-major X^T (np padded rows); limbs is scratch
// u8 [5][np] (rebuilt from dw here).
extern "C" int simopt_logistic_xtdx_i8(void* stream, const uint8_t* xt, int64_t np, int64_t n,
                                       int64_t d, const double* dw, uint8_t* limbs, double* h) {
  SIMOPT_REQUIRE(n >= 1 && d >= 1, SIMOPT_E_DIMENSION, "empty design matrix");
  int64_t ch = 0, np_want = 0;
  simopt_u8t_geometry(n, &ch, &np_want);
  SIMOPT_REQUIRE(np == np_want, SIMOPT_E_CONFIG, "np must come from simopt_u8t_geometry");
  cudaStream_t st = as_stream(stream);
  int lg = 0;
  while ((1LL << lg) < ch) ++lg;
  k_limbs<<<egrid(np), 256, 0, st>>>(dw, n, np, limbs);
  SIMOPT_CHECK_LAUNCH("k_limbs");
  const int64_t nt = (d + kBM - 1) / kBM;
  const int64_t tiles = nt * (nt + 1) / 2;
  SIMOPT_REQUIRE(tiles < (1LL << 31), SIMOPT_E_CONFIG, "d too large");
  int beta = 0;
  for (int64_t c0 = 0; c0 < np; c0 += kChunk) {
    const int64_t c1 = c0 + kChunk < np ? c0 + kChunk : np;
    for (int k = 0; k < kLimbs; ++k) {
      const double scale = ldexp(1.0, kLimbBits * k - kFixBits) / (double)n;
      k_xtdx_i8<<<(unsigned)tiles, kThreads, 0, st>>>(xt, lg, d, limbs + k * np, c0, c1, scale, beta, h);
      SIMOPT_CHECK_LAUNCH("k_xtdx_i8");
      beta = 1;
    }
  }
  return SIMOPT_OK;
}
