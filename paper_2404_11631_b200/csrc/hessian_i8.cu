// Explicit logistic Hessian H = (1/n) X^T diag(dw) X for BINARY X on the integer tensor
// cores: exact limb decomposition (an Ozaki-style split of dw, possible because X is 0/1).
//
// dw in [0, 1/4] is rounded once to the fixed point q = round(dw * 2^41) <= 2^39 and
// split into five 8-bit limbs L_k = (q >> 8k) & 255.  Then
//     H = (1/n) * sum_k 2^(8k-41) * G_k,     G_k[i][j] = sum_r x_ri * x_rj * L_rk,
// and every G_k is an integer GEMM with u8 operands (x in {0,1}, L_k in [0,255]) and
// exact int32 accumulation (a sample chunk holds <= 2^23 rows: 2^23 * 255 < 2^31).
// The only rounding is the quantisation of dw and the final fp64 scaling/summation.
// The fixed-point exponent follows max(dw) (2^41 when max(dw) = 1/4), and a guard
// (limb_hessian) adds exact-residual refinement passes whenever the worst-case
// quantisation bound 2^-40 max(dw)/mean(dw) exceeds 1e-11 -- so H stays inside the
// 1e-10 tolerance of the reference's explicit-Hessian oracle (tests/test_tasks.py:
// 292-304) for any spread of c(1-c), e.g. a confident model.
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
#include <stdlib.h>
#include <string.h>

#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>
#include <utility>
#include <vector>

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

// ---------------------------------------------------------------------------------------
// tcgen05 version (5th-gen tensor cores, TMEM accumulators).  One CTA (4 warps) owns a
// 128 (i) x 96 (j) tile of H and keeps all five limb accumulators D_k (s32, 128 lanes x
// 96 columns each = 480 of the SM's 512 TMEM columns) resident for the whole sample
// range.  Per 32-sample k-step: cp.async brings the A tile (X, 128 x 32 B) and the raw B
// tile (X, 96 x 32 B) straight into the SWIZZLE_NONE K-major canonical layout (8-row x
// 16-byte core matrices), all threads expand B into the five limb-scaled copies
// (b * 255) & L_k, and one elected thread issues five tcgen05.mma.kind::i8 (M=128, N=96,
// K=32) and commits them to the stage's mbarrier, which frees the stage four steps later.
// Epilogue: tcgen05.ld of the five accumulators, fp64 combination 2^(8k-41)/n, upper
// entries and their mirrors.  (tools/micro/tc_i8.cu is the single-MMA smoke test.)
constexpr int kTM = 128, kTN = 96;
constexpr int kTK = 64;              // samples per stage = two K=32 MMAs per limb
constexpr int kRing = 8, kTP = 6;    // cp.async ring depth (power of two: cheap slot and phase math), prefetch distance
constexpr int kTP_THREADS = 256;     // producer threads (warps 0-7; warps 0-3 also run the epilogue)
constexpr int kTT = kTP_THREADS + 32;  // + one MMA-issuer warp (warp 8)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t umma_desc(const void* p) {  // SWIZZLE_NONE, K-major
  return (uint64_t)((smem_u32(p) >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(256 >> 4) << 32) | ((uint64_t)1 << 46);
}
// canonical byte offset of (row r, k-byte kb < 64) in an R x 64-byte operand stage:
// sub-tile kb/32 (one MMA's K), then 8-row x 16-byte core matrices (LBO 128, SBO 256)
template <int R>
__device__ __forceinline__ int canon(int r, int kb) {
  return (kb >> 5) * (R * 32) + (r >> 3) * 256 + ((kb >> 4) & 1) * 128 + (r & 7) * 16 + (kb & 15);
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

struct TcSmem {
  uint8_t a[kRing][kTM * kTK];          // X rows i (MMA operand A, read in place)
  uint8_t braw[kRing][kTN * kTK];       // X rows j
  uint8_t limb[kRing][kLimbs][kTK];
  uint8_t b[2][kLimbs][kTN * kTK];      // limb-scaled B operands (double-buffered)
  uint64_t done[kRing];                 // MMAs of the step that used ring slot s completed
  uint64_t full[kRing];                 // producers: stage in slot s loaded and expanded
  uint32_t taddr;
};

__global__ void __launch_bounds__(kTT, 1)
    k_xtdx_tc(const uint8_t* __restrict__ xt, int lg_ch, int64_t d, const uint8_t* __restrict__ limbs,
              int64_t np, const int2* __restrict__ tiles, int64_t s0, int64_t s1, double inv_n, int beta,
              double* __restrict__ h) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  TcSmem& sm = *reinterpret_cast<TcSmem*>(smraw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int2 tile = tiles[blockIdx.x];
  const int64_t i0 = (int64_t)tile.x * kTM, j0 = (int64_t)tile.y * kTN;
  const int64_t ch = 1LL << lg_ch, rs = ch + kRowPad;
  if (tid == 0) {
    for (int q = 0; q < kRing; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sm.done[q])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&sm.full[q])),
                   "r"(kTP_THREADS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&sm.taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t taddr = sm.taddr;
  const uint32_t idesc = (2u << 4) | ((uint32_t)(kTN >> 3) << 17) | ((uint32_t)(kTM >> 4) << 24);
  // descriptor arithmetic below adds byte offsets >> 4 to the start-address field: the
  // whole shared window must stay below 2^18 bytes (14-bit field), which it does
  const int64_t T = (s1 - s0) / kTK;
  // this thread's cp.async chunks, fixed for every stage: (source offset in a sample
  // block, destination offset in a ring slot, bytes); 16-byte chunks of the A rows, the
  // B rows, then the limb rows
  constexpr int kA = kTM * 4, kB = kTN * 4, kL = kLimbs * 4;
  constexpr int kPer = (kA + kB + kL + kTP_THREADS - 1) / kTP_THREADS;
  int64_t csrc[kPer];
  int cdst[kPer], cbytes[kPer];
  constexpr int kSlot = (int)(sizeof(TcSmem::a[0]));
  const int a_base = (int)(sm.a[0] - smraw), b_base = (int)(sm.braw[0] - smraw);
  const int l_base = (int)(&sm.limb[0][0][0] - smraw);
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int c = tid + u * kTP_THREADS;
    csrc[u] = 0; cdst[u] = 0; cbytes[u] = -1;  // -1: no chunk
    if (c < kA + kB) {
      const bool isa = c < kA;
      const int cc = isa ? c : c - kA;
      const int r = cc >> 2, kb = (cc & 3) * 16;
      const int64_t feat = (isa ? i0 : j0) + r;
      cbytes[u] = feat < d ? 16 : 0;
      csrc[u] = (feat < d ? feat : 0) * rs + kb;
      cdst[u] = isa ? a_base + canon<kTM>(r, kb) : b_base + canon<kTN>(r, kb);
    } else if (c < kA + kB + kL) {
      const int cc = c - kA - kB, k = cc >> 2, kb = (cc & 3) * 16;
      cbytes[u] = 16;
      csrc[u] = -1 - (k * np + kb);  // negative: a limb row (offset from `limbs`)
      cdst[u] = l_base + k * kTK + kb;
    }
  }
  const uint32_t sbase = smem_u32(smraw);
  auto issue = [&](int64_t t) {  // cp.async of stage t into ring slot t % kRing
    const int q = (int)(t % kRing);
    const int64_t smp = s0 + t * kTK;
    const uint8_t* blk = xt + (smp >> lg_ch) * (d * rs) + (smp & (ch - 1));
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      if (cbytes[u] < 0) continue;
      const bool lim = csrc[u] < 0;
      const uint8_t* src = lim ? limbs + (-1 - csrc[u]) + smp : blk + csrc[u];
      const uint32_t dst = sbase + (uint32_t)cdst[u] +
                           (uint32_t)q * (lim ? (uint32_t)sizeof(TcSmem::limb[0]) : (uint32_t)(cdst[u] < b_base ? kSlot : (int)sizeof(TcSmem::braw[0])));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(cbytes[u]));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  if (warp < kTP_THREADS / 32) {
    // ===== producers: cp.async ring, limb expansion, arrive on full[slot] =====
    for (int64_t t = 0; t < kTP; ++t) {
      if (t < T) issue(t);
      else asm volatile("cp.async.commit_group;\n" ::);
    }
    for (int64_t t = 0; t < T; ++t) {
      const int q = (int)(t % kRing), bb = (int)(t & 1);
      // MMAs of stage t-2 read b[bb] and ring slot (t+kTP) % kRing: wait for them
      if (t >= 2) mbar_wait(&sm.done[(t - 2) % kRing], (uint32_t)(((t - 2) / kRing) & 1));
      {
        const int64_t tp = t + kTP;
        if (tp < T) issue(tp);
        else asm volatile("cp.async.commit_group;\n" ::);
      }
      asm volatile("cp.async.wait_group %0;\n" ::"n"(kTP));
      asm volatile("bar.sync 1, %0;" ::"n"(kTP_THREADS));  // every producer's copies landed
      // B_k = (x * 255) & L_k, four samples per word, same canonical offsets as the raw
      // tile.  Task = (16-sample column kb, 32-row group): a warp's lanes share kb, so the
      // five limb vectors are broadcast reads.
      for (int task = warp; task < 4 * (kTN / 32); task += kTP_THREADS / 32) {
        const int kb = (task & 3) * 16, r = (task >> 2) * 32 + lane;
        const int off = canon<kTN>(r, kb);
        const uint4 x = *reinterpret_cast<const uint4*>(&sm.braw[q][off]);
        const uint4 m = make_uint4(x.x * 255u, x.y * 255u, x.z * 255u, x.w * 255u);
#pragma unroll
        for (int k = 0; k < kLimbs; ++k) {
          const uint4 L = *reinterpret_cast<const uint4*>(&sm.limb[q][k][kb]);
          *reinterpret_cast<uint4*>(&sm.b[bb][k][off]) =
              make_uint4(m.x & L.x, m.y & L.y, m.z & L.z, m.w & L.w);
        }
      }
      // generic-proxy writes (cp.async'd A, expanded B) -> visible to the tensor core
      asm volatile("fence.proxy.async.shared::cta;");
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&sm.full[q])) : "memory");
    }
  } else if (lane == 0) {
    // ===== MMA issuer (warp 8, one lane): per stage one A copy into TMEM and five
    // limb MMAs per K-step, committed to done[slot] =====
    const uint64_t da0 = umma_desc(sm.a[0]), db0 = umma_desc(sm.b[0][0]);
    const uint64_t a_slot = (uint64_t)(sizeof(TcSmem::a[0]) >> 4);
    const uint64_t b_buf = (uint64_t)(sizeof(TcSmem::b[0]) >> 4), b_limb = (uint64_t)(sizeof(TcSmem::b[0][0]) >> 4);
    for (int64_t t = 0; t < T; ++t) {
      const int q = (int)(t % kRing), bb = (int)(t & 1);
      mbar_wait(&sm.full[q], (uint32_t)((t / kRing) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int ks = 0; ks < kTK / 32; ++ks) {
        // A (shared by the five limb MMAs) is copied into TMEM once per K-step and the MMAs
        // read it from there (TS mode): shared memory serves only the B operands.  cp and
        // mma issued by this thread execute in order; 4 rotating 8-column A slots.
        const uint32_t ta = taddr + (uint32_t)(kLimbs * kTN + 8 * (int)((2 * t + ks) & 3));
        const uint64_t da = da0 + (uint64_t)q * a_slot + (uint64_t)(ks * kTM * 32 >> 4);
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(ta), "l"(da));
#pragma unroll
        for (int k = 0; k < kLimbs; ++k) {
          const uint64_t db = db0 + (uint64_t)bb * b_buf + (uint64_t)k * b_limb + (uint64_t)(ks * kTN * 32 >> 4);
          const uint32_t acc = (t > 0 || ks > 0) ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(
                  taddr + (uint32_t)(k * kTN)),
              "r"(ta), "l"(db), "r"(idesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&sm.done[q])));
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  if (T > 0) mbar_wait(&sm.done[(T - 1) % kRing], (uint32_t)(((T - 1) / kRing) & 1));
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {  // epilogue: row i = i0 + 32*warp + lane, columns j0 .. j0+95
    const int64_t i = i0 + warp * 32 + lane;
    for (int c0 = 0; c0 < kTN; c0 += 32) {
      double hv[32];
#pragma unroll
      for (int qq = 0; qq < 32; ++qq) hv[qq] = 0.0;
#pragma unroll
      for (int k = 0; k < kLimbs; ++k) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
              "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
              "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
              "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr + ((uint32_t)(warp * 32) << 16) + (uint32_t)(k * kTN + c0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        const double sc = ldexp(1.0, kLimbBits * k - kFixBits) * inv_n;
#pragma unroll
        for (int qq = 0; qq < 32; ++qq) hv[qq] += (double)(int)v[qq] * sc;
      }
      if (i < d) {
#pragma unroll
        for (int qq = 0; qq < 32; ++qq) {
          const int64_t j = j0 + c0 + qq;
          if (j < d && i <= j) {
            if (beta) {
              h[i * d + j] += hv[qq];
              if (i != j) h[j * d + i] += hv[qq];
            } else {
              h[i * d + j] = hv[qq];
              if (i != j) h[j * d + i] = hv[qq];
            }
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr));
}

// ---------------------------------------------------------------------------------------
// TMA-fed tcgen05 version (the default for binary X).  Same 128 x 96 tile and the same
// limb algebra as k_xtdx_tc, re-balanced for the three limits measured on this B200:
//  * operands by TMA: per 64-sample stage one thread issues one box of the 128 A rows, one
//    of the 96 B rows (3-D tensor maps over the sample-blocked X^T [block][feature][sample],
//    64-byte rows with the 64-byte swizzle: whole sectors, one request per row) and one of
//    the five limb rows, completing on the slot's tma_full mbarrier (expect_tx bytes);
//  * wide MMAs (kWide): a tcgen05.mma.kind::i8 costs ~55 ns per SM for any N <= 128 and
//    ~69 ns at N = 256 (tools/micro/tc_i8_rate.cu), so the five limb copies of each
//    48-column half of B are stacked along N: a K step is 2 MMAs of N = 240 (two
//    accumulators of 5 x 48 columns = 480 TMEM columns) instead of 5 of N = 96;
//  * the limb expansion ((x * 255) & L_k into kBB rotating buffers) is the shared-memory
//    bandwidth bound that remains: 12 warps, one 16-sample chunk each, mapped so that a
//    warp's 32 rows share one logical chunk -- its reads and writes are conflict-free under
//    the swizzle and its limb reads are broadcasts.
// A is copied into TMEM once per K step (tcgen05.cp) and read from there by the MMAs.
// kSW = 16 keeps the first version (16-byte boxes per K half, SWIZZLE_NONE) for comparison.
constexpr int kMR = 8;                 // TMA ring depth (stages in flight)
constexpr int kQThreads = 384;         // expansion threads, one 16-sample chunk of B each (warps 0-11; 0-3 also the epilogue)
constexpr int kQT = kQThreads + 64;    // + TMA warp (12) + MMA warp (13)
constexpr uint32_t kStageTx = 2 * 2 * (kTM + kTN) * 16 + kLimbs * kTK;  // bytes per stage
constexpr int kBB = 3;                 // expanded-B buffers: expansion runs kBB-1 stages ahead of the MMAs

struct TmaSmem {
  // operand stages, 64 samples of 128 (A) / 96 (B) feature rows each; layout kSW:
  //   16: [K step][K half][row][16 B] (SWIZZLE_NONE core matrices, one box per K half)
  //   64: [row][64 B] with the 64-byte swizzle (one box per stage)
  uint8_t a[kMR][kTM * 64];
  uint8_t braw[kMR][kTN * 64];
  uint8_t limb[kMR][384];                   // [5][64] (+ pad: 128-byte aligned slots)
  uint8_t b[kBB][kLimbs][kTN * 64];         // limb-scaled B (kBB-buffered), layout of braw
  uint64_t tma_full[kMR], full[kMR], done[kMR];
  uint32_t taddr;
};

// K-major SWIZZLE_NONE descriptor: LBO = K-half stride, SBO = 8-row-group stride (bytes)
__device__ __forceinline__ uint64_t umma_desc_kn(const void* p, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((smem_u32(p) >> 4) & 0x3FFF) | ((uint64_t)(lbo >> 4) << 16) |
         ((uint64_t)(sbo >> 4) << 32) | ((uint64_t)1 << 46);
}

__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                       uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
        "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// K-major SWIZZLE_64B descriptor (layout type 4): 8-row x 64-byte swizzle atoms, SBO = 512 B
__device__ __forceinline__ uint64_t umma_desc_sw64(const void* p) {
  return (uint64_t)((smem_u32(p) >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}

// kWide (with kSW = 64): the tile's two 48-column halves each get ONE accumulator of
// N = 5 x 48 = 240 columns -- the five limb copies of a half's B rows are stacked along N --
// so a K step takes 2 MMAs of N = 240 instead of 5 of N = 96.  A tcgen05.mma.kind::i8
// costs ~55 ns per SM up to N = 128 and ~69 ns at N = 256 (tools/micro/tc_i8_rate.cu):
// the narrow MMAs, not the operands, set the narrow kernel's pace.
template <int kSW, bool kWide>
__global__ void __launch_bounds__(kQT, 1)
    k_xtdx_tma(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               const __grid_constant__ CUtensorMap map_l, int lg_ch, int64_t d,
               const int2* __restrict__ tiles, int64_t s0, int64_t s1, double inv_n, int beta,
               double* __restrict__ h) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  TmaSmem& sm = *reinterpret_cast<TmaSmem*>(smraw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int2 tile = tiles[blockIdx.x];
  const int64_t i0 = (int64_t)tile.x * kTM, j0 = (int64_t)tile.y * kTN;
  const int64_t ch = 1LL << lg_ch;
  if (tid == 0) {
    for (int q = 0; q < kMR; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sm.tma_full[q])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&sm.full[q])),
                   "r"(kQThreads / 32));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sm.done[q])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&sm.taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t taddr = sm.taddr;
  constexpr int kHN = kTN / 2, kWN = kLimbs * kHN;  // wide: half width 48, MMA N = 240
  const uint32_t idesc = (2u << 4) | ((uint32_t)((kWide ? kWN : kTN) >> 3) << 17) |
                         ((uint32_t)(kTM >> 4) << 24);
  const int64_t T = (s1 - s0) / kTK;
  if (warp < kQThreads / 32) {
    // ===== limb expansion: B_k = (x * 255) & L_k per 16-sample chunk =====
    int bb = 0;
    for (int64_t t = 0; t < T; ++t, bb = (bb + 1 == kBB ? 0 : bb + 1)) {
      const int q = (int)(t % kMR);
      if (t >= kBB) mbar_wait(&sm.done[(t - kBB) % kMR], (uint32_t)(((t - kBB) / kMR) & 1));
      mbar_wait(&sm.tma_full[q], (uint32_t)((t / kMR) & 1));
      for (int c = tid; c < 4 * kTN; c += kQThreads) {
        int off, lc;  // byte offset of this 16-sample chunk, its logical chunk (samples lc*16..)
        if (kSW == 16) {
          const int kh = c / kTN, r = c - kh * kTN;  // kh = 2 * K step + K half
          off = kh * (kTN * 16) + r * 16;
          lc = kh;
        } else {
          // a warp takes one logical chunk of 32 rows: its x reads and limb-scaled writes
          // are conflict-free under the swizzle, its limb reads are broadcasts
          // (Swizzle<2,4,3>: physical chunk = logical ^ ((row >> 1) & 3))
          const int wv = c >> 5, r = (wv >> 2) * 32 + (c & 31);
          lc = wv & 3;
          off = r * 64 + ((lc ^ ((r >> 1) & 3)) * 16);
        }
        const uint4 x = *reinterpret_cast<const uint4*>(&sm.braw[q][off]);
        const uint4 m = make_uint4(x.x * 255u, x.y * 255u, x.z * 255u, x.w * 255u);
#pragma unroll
        for (int k = 0; k < kLimbs; ++k) {
          const uint4 L = *reinterpret_cast<const uint4*>(&sm.limb[q][k * kTK + lc * 16]);
          const uint4 v = make_uint4(m.x & L.x, m.y & L.y, m.z & L.z, m.w & L.w);
          if (kWide) {  // row r of half hh -> row hh*240 + k*48 + (r - 48 hh): same swizzle phase
            const int r = off >> 6, hh = r >= kHN ? 1 : 0;
            *reinterpret_cast<uint4*>(&sm.b[bb][0][(hh * kWN + k * kHN + r - hh * kHN) * 64 + (off & 63)]) = v;
          } else {
            *reinterpret_cast<uint4*>(&sm.b[bb][k][off]) = v;
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;");
      __syncwarp();  // one arrival per warp (count kQThreads / 32)
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&sm.full[q])) : "memory");
    }
  } else if (warp == kQThreads / 32) {
    if (lane == 0) {  // ===== TMA issue =====
      for (int64_t t = 0; t < T; ++t) {
        const int q = (int)(t % kMR);
        if (t >= kMR) mbar_wait(&sm.done[(t - kMR) % kMR], (uint32_t)(((t - kMR) / kMR) & 1));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&sm.tma_full[q])),
                     "r"(kStageTx) : "memory");
        const int64_t smp = s0 + t * kTK;
        const int blk = (int)(smp >> lg_ch), so = (int)(smp & (ch - 1));
        if (kSW == 16) {
#pragma unroll
          for (int kh = 0; kh < 4; ++kh) {
            tma_3d(&sm.a[q][kh * kTM * 16], &map_a, so + 16 * kh, (int)i0, blk, &sm.tma_full[q]);
            tma_3d(&sm.braw[q][kh * kTN * 16], &map_b, so + 16 * kh, (int)j0, blk, &sm.tma_full[q]);
          }
        } else {
          tma_3d(sm.a[q], &map_a, so, (int)i0, blk, &sm.tma_full[q]);
          tma_3d(sm.braw[q], &map_b, so, (int)j0, blk, &sm.tma_full[q]);
        }
        tma_2d(sm.limb[q], &map_l, (int)smp, 0, &sm.tma_full[q]);
      }
    }
  } else if (lane == 0) {
    // ===== MMA issuer: per K step one A copy into TMEM and five limb MMAs =====
    int bb = 0;
    for (int64_t t = 0; t < T; ++t, bb = (bb + 1 == kBB ? 0 : bb + 1)) {
      const int q = (int)(t % kMR);
      mbar_wait(&sm.tma_full[q], (uint32_t)((t / kMR) & 1));
      mbar_wait(&sm.full[q], (uint32_t)((t / kMR) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const uint32_t ta = taddr + (uint32_t)(kLimbs * kTN + 8 * (int)((2 * t + ks) & 3));
        const uint64_t da = kSW == 16 ? umma_desc_kn(&sm.a[q][ks * kTM * 32], kTM * 16, 128)
                                      : umma_desc_sw64(&sm.a[q][ks * 32]);
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(ta), "l"(da));
        constexpr int kNM = kWide ? 2 : kLimbs;  // MMAs per K step
#pragma unroll
        for (int k = 0; k < kNM; ++k) {
          const uint64_t db = kWide ? umma_desc_sw64(&sm.b[bb][0][k * kWN * 64 + ks * 32])
                              : kSW == 16 ? umma_desc_kn(&sm.b[bb][k][ks * kTN * 32], kTN * 16, 128)
                                          : umma_desc_sw64(&sm.b[bb][k][ks * 32]);
          const uint32_t acc = (t > 0 || ks > 0) ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(
                  taddr + (uint32_t)(k * (kWide ? kWN : kTN))),
              "r"(ta), "l"(db), "r"(idesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&sm.done[q])));
    }
  }
  if (T > 0) mbar_wait(&sm.done[(T - 1) % kMR], (uint32_t)(((T - 1) / kMR) & 1));
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (kWide && warp < 4) {  // epilogue (wide): column jj = 48 h + c sums D_h[k*48 + c] over k
    const int64_t i = i0 + warp * 32 + lane;
    for (int hc = 0; hc < 6; ++hc) {
      const int hh = hc / 3, c0 = (hc % 3) * 16;
      double hv[16];
#pragma unroll
      for (int qq = 0; qq < 16; ++qq) hv[qq] = 0.0;
#pragma unroll
      for (int k = 0; k < kLimbs; ++k) {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
              "=r"(v[14]), "=r"(v[15])
            : "r"(taddr + ((uint32_t)(warp * 32) << 16) + (uint32_t)(hh * kWN + k * kHN + c0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        const double sc = ldexp(1.0, kLimbBits * k - kFixBits) * inv_n;
#pragma unroll
        for (int qq = 0; qq < 16; ++qq) hv[qq] += (double)(int)v[qq] * sc;
      }
      if (i < d) {
#pragma unroll
        for (int qq = 0; qq < 16; ++qq) {
          const int64_t j = j0 + hh * kHN + c0 + qq;
          if (j < d && i <= j) {
            if (beta) {
              h[i * d + j] += hv[qq];
              if (i != j) h[j * d + i] += hv[qq];
            } else {
              h[i * d + j] = hv[qq];
              if (i != j) h[j * d + i] = hv[qq];
            }
          }
        }
      }
    }
  }
  if (!kWide && warp < 4) {  // epilogue: row i = i0 + 32*warp + lane, columns j0 .. j0+95
    const int64_t i = i0 + warp * 32 + lane;
    for (int c0 = 0; c0 < kTN; c0 += 32) {
      double hv[32];
#pragma unroll
      for (int qq = 0; qq < 32; ++qq) hv[qq] = 0.0;
#pragma unroll
      for (int k = 0; k < kLimbs; ++k) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
              "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
              "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
              "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr + ((uint32_t)(warp * 32) << 16) + (uint32_t)(k * kTN + c0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        const double sc = ldexp(1.0, kLimbBits * k - kFixBits) * inv_n;
#pragma unroll
        for (int qq = 0; qq < 32; ++qq) hv[qq] += (double)(int)v[qq] * sc;
      }
      if (i < d) {
#pragma unroll
        for (int qq = 0; qq < 32; ++qq) {
          const int64_t j = j0 + c0 + qq;
          if (j < d && i <= j) {
            if (beta) {
              h[i * d + j] += hv[qq];
              if (i != j) h[j * d + i] += hv[qq];
            } else {
              h[i * d + j] = hv[qq];
              if (i != j) h[j * d + i] = hv[qq];
            }
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr));
}

// ---------------------------------------------------------------------------------------
// CTA-pair version (cta_group::2): a cluster of two CTAs on one TPC owns a 256 x 96 tile.
// Each CTA TMA-loads its own 128 A rows, the 96 raw B rows and the limb rows; the
// limb-scaled B' of each 48-column half (240 rows: 5 limbs x 48) is SPLIT between the two
// CTAs -- rows 0..119 in CTA 0, 120..239 in CTA 1, at the same shared-memory offset -- so
// each CTA expands and each SM's tensor core reads half of what the single-CTA kernel
// does, which was its shared-memory bound.  The leader's single thread issues the M = 256
// MMAs (A and B' from both CTAs' shared memory); their commits are multicast to both
// CTAs' `done` barriers; both CTAs' expansion warps arrive on the leader's `full`
// barrier.  Each CTA's TMEM holds its 128 accumulator rows (2 x 240 columns).
// Measured on the C5 slice: 19.6 ms against 17.7 ms for k_xtdx_tma<64, wide> -- the pair
// MMAs themselves run at the full 4.5 POPS (tools/micro/tc_i8_pair_rate.cu), but each
// stage's expansion waits on the multicast completion of the MMAs kPBB stages back, and the
// shared memory left after the TMA ring allows only 7 buffers.  Opt-in: SIMOPT_XTDX_PAIR=1.
constexpr int kPR = 8;                   // TMA ring depth (slot/phase kept as counters)
constexpr int kPBB = 7;                   // expanded-B' buffers
constexpr int kPH = 120;                  // B' rows per CTA per half
// `done` barriers are indexed by TMA slot: an expansion buffer may not outlive its slot
static_assert(kPBB <= kPR, "expanded-B' reuse waits on the done barrier of a live TMA slot");
struct PairSmem {
  uint8_t a[kPR][kTM * 64];
  uint8_t braw[kPR][kTN * 64];
  uint8_t limb[kPR][384];
  uint8_t b[kPBB][2][kPH * 64];
  uint64_t tma_full[kPR], full[kPR], done[kPR], fwd[kPR];
  uint32_t taddr;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kQT, 1)
    k_xtdx_pair(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                const __grid_constant__ CUtensorMap map_l, int lg_ch, int64_t d,
                const int2* __restrict__ tiles, int64_t s0, int64_t s1, double inv_n, int beta,
                double* __restrict__ h) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  PairSmem& sm = *reinterpret_cast<PairSmem*>(smraw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const int2 tile = tiles[blockIdx.x >> 1];
  const int64_t i0 = (int64_t)tile.x * (2 * kTM), j0 = (int64_t)tile.y * kTN;
  const int64_t ia = i0 + (int64_t)rank * kTM;  // this CTA's A rows
  const int64_t ch = 1LL << lg_ch;
  constexpr int kHN = kTN / 2, kWN = kLimbs * kHN;  // 48, 240
  if (tid == 0) {
    for (int q = 0; q < kPR; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sm.tma_full[q])));
      // leader: its own 12 expansion warps + one forwarded arrival from the follower
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&sm.full[q])),
                   "r"(kQThreads / 32 + 1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sm.done[q])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&sm.fwd[q])),
                   "r"(kQThreads / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&sm.taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t taddr = sm.taddr;
  const uint32_t idesc = (2u << 4) | ((uint32_t)(kWN >> 3) << 17) | ((uint32_t)((2 * kTM) >> 4) << 24);
  const int64_t T = (s1 - s0) / kTK;
  if (warp < kQThreads / 32) {
    // ===== expansion: raw row f (0..95), logical chunk lc -> this CTA's limb rows =====
    // leader's full barrier, in the cluster window
    uint32_t full0;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(full0) : "r"(smem_u32(&sm.full[0])));
    const int wv = tid >> 5, f = (wv >> 2) * 32 + lane, lc = wv & 3;
    const int hh = f >= kHN ? 1 : 0, c = f - hh * kHN;
    const int off = f * 64 + ((lc ^ ((f >> 1) & 3)) * 16);
    const int pc = off & 63;  // physical chunk offset (same swizzle phase in B')
    int bb = 0, q = 0, dq = 0;
    uint32_t ph = 0, dph = 0;  // (slot, phase) of stage t and of stage t - kPBB
    for (int64_t t = 0; t < T; ++t, bb = (bb + 1 == kPBB ? 0 : bb + 1)) {
      if (t >= kPBB) {
        mbar_wait(&sm.done[dq], dph);
        if (++dq == kPR) { dq = 0; dph ^= 1u; }
      }
      mbar_wait(&sm.tma_full[q], ph);
      const uint4 x = *reinterpret_cast<const uint4*>(&sm.braw[q][off]);      const uint4 m = make_uint4(x.x * 255u, x.y * 255u, x.z * 255u, x.w * 255u);
#pragma unroll
      for (int k = 0; k < kLimbs; ++k) {
        const int R = k * kHN + c - (int)rank * kPH;  // B'_h row in this CTA
        if (R >= 0 && R < kPH) {
          const uint4 L = *reinterpret_cast<const uint4*>(&sm.limb[q][k * kTK + lc * 16]);
          *reinterpret_cast<uint4*>(&sm.b[bb][hh][R * 64 + pc]) =
              make_uint4(m.x & L.x, m.y & L.y, m.z & L.z, m.w & L.w);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;");
      __syncwarp();
      // CTA-scope arrivals (cheap): the leader's warps on its full barrier, the
      // follower's on a local barrier that one thread forwards across the pair
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
                         smem_u32(rank == 0 ? &sm.full[q] : &sm.fwd[q])) : "memory");
      if (++q == kPR) { q = 0; ph ^= 1u; }
    }
    (void)full0;
  } else if (warp == kQThreads / 32) {
    if (lane == 0) {  // ===== TMA issue (own rows, own smem, own barrier) =====
      int q = 0;
      uint32_t ph = 0;
      for (int64_t t = 0; t < T; ++t) {
        if (t >= kPR) mbar_wait(&sm.done[q], ph ^ 1u);  // stage t - kPR used this slot
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&sm.tma_full[q])),
                     "r"(kStageTx) : "memory");
        const int64_t smp = s0 + t * kTK;
        const int blk = (int)(smp >> lg_ch), so = (int)(smp & (ch - 1));
        tma_3d(sm.a[q], &map_a, so, (int)ia, blk, &sm.tma_full[q]);
        tma_3d(sm.braw[q], &map_b, so, (int)j0, blk, &sm.tma_full[q]);
        tma_2d(sm.limb[q], &map_l, (int)smp, 0, &sm.tma_full[q]);
        if (++q == kPR) { q = 0; ph ^= 1u; }
      }
    }
  } else if (rank == 1) {
    // ===== follower: forward each stage's local arrivals to the leader's full barrier,
    // one lane per ring slot so the cluster-scope releases overlap =====
    if (lane < kPR) {
      uint32_t full0;
      asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(full0) : "r"(smem_u32(&sm.full[0])));
      uint32_t ph = 0;
      for (int64_t t = lane; t < T; t += kPR, ph ^= 1u) {
        mbar_wait(&sm.fwd[lane], ph);
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                         full0 + (uint32_t)(lane * 8)) : "memory");
      }
    }
  } else if (lane == 0) {
    // ===== MMA issuer (leader): per K step 2 MMAs of M = 256, N = 240 =====
    int bb = 0, q = 0;
    uint32_t ph = 0;
    for (int64_t t = 0; t < T; ++t, bb = (bb + 1 == kPBB ? 0 : bb + 1)) {
      mbar_wait_cluster(&sm.full[q], ph);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const uint64_t da = umma_desc_sw64(&sm.a[q][ks * 32]);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const uint64_t db = umma_desc_sw64(&sm.b[bb][hh][ks * 32]);
          const uint32_t acc = (t > 0 || ks > 0) ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(
                  taddr + (uint32_t)(hh * kWN)),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&sm.done[q])), "h"((uint16_t)3));
      if (++q == kPR) { q = 0; ph ^= 1u; }
    }
  }
  if (T > 0) mbar_wait(&sm.done[(T - 1) % kPR], (uint32_t)(((T - 1) / kPR) & 1));
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {  // epilogue: this CTA's row i = ia + 32*warp + lane
    const int64_t i = ia + warp * 32 + lane;
    for (int hc = 0; hc < 6; ++hc) {
      const int hh = hc / 3, c0 = (hc % 3) * 16;
      double hv[16];
#pragma unroll
      for (int qq = 0; qq < 16; ++qq) hv[qq] = 0.0;
#pragma unroll
      for (int k = 0; k < kLimbs; ++k) {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
              "=r"(v[14]), "=r"(v[15])
            : "r"(taddr + ((uint32_t)(warp * 32) << 16) + (uint32_t)(hh * kWN + k * kHN + c0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        const double sc = ldexp(1.0, kLimbBits * k - kFixBits) * inv_n;
#pragma unroll
        for (int qq = 0; qq < 16; ++qq) hv[qq] += (double)(int)v[qq] * sc;
      }
      if (i < d) {
#pragma unroll
        for (int qq = 0; qq < 16; ++qq) {
          const int64_t j = j0 + hh * kHN + c0 + qq;
          if (j < d && i <= j) {
            if (beta) {
              h[i * d + j] += hv[qq];
              if (i != j) h[j * d + i] += hv[qq];
            } else {
              h[i * d + j] = hv[qq];
              if (i != j) h[j * d + i] = hv[qq];
            }
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(taddr));
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

// limbs[k][r] = byte k of q = round(dw[r] * 2^e), 0 for r >= n (qscale = 2^e with
// max(dw) * 2^e < 2^40, so q fits the five limbs).  With r_pos/r_neg, the rounding
// residual dw - q 2^-e (exact: the bits of dw below 2^-e) is split into its positive
// and negative parts for the refinement passes.
__global__ void k_limbs(const double* __restrict__ dw, int64_t n, int64_t np, double qscale,
                        uint8_t* __restrict__ out, double* __restrict__ r_pos, double* __restrict__ r_neg) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < np;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint64_t q = 0;
    if (r < n) {
      double v = dw[r];
      v = v < 0.0 ? 0.0 : (v > 0.25 ? 0.25 : v);
      const double qd = rint(v * qscale);
      q = (uint64_t)qd;
      if (r_pos) {
        const double res = v - qd / qscale;
        r_pos[r] = res > 0.0 ? res : 0.0;
        r_neg[r] = res < 0.0 ? -res : 0.0;
      }
    }
#pragma unroll
    for (int k = 0; k < kLimbs; ++k) out[k * np + r] = (uint8_t)((q >> (kLimbBits * k)) & 255ULL);
  }
}

// max (as IEEE bits: the clamped weights are >= 0, so bit order is value order) and sum
// of the clamped weights -- the limb exponent and the precision guard
__global__ void k_dw_stats(const double* __restrict__ dw, int64_t n, unsigned long long* __restrict__ mx,
                           double* __restrict__ sum) {
  double m = 0.0, s = 0.0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    double v = dw[r];
    v = v < 0.0 ? 0.0 : (v > 0.25 ? 0.25 : v);
    m = fmax(m, v);
    s += v;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(mx, (unsigned long long)__double_as_longlong(m));
    atomicAdd(sum, s);
  }
}

int egrid(int64_t n) {
  const int64_t g = ceil_div(n, 256), cap = (int64_t)SIMOPT_NUM_SMS * 16;
  return (int)(g < 1 ? 1 : (g < cap ? g : cap));
}

// Limb exponent: the largest e <= 1000 with max * 2^e < 2^40 (e = 41 for max = 1/4).
int limb_exponent(double mx) {
  if (!(mx > 0.0)) return 41;
  const int e = 39 - ilogb(mx);
  return e > 1000 ? 1000 : e;
}

thread_local int g_passes = 0;

// Guarded limb Hessian.  One limb pass quantises dw to round(dw 2^e) (|error| <= 2^-(e+1)
// per sample), so entry (i,j) of H is off by at most 2^-(e+1) / mean(dw over its rows)
// relative; with e from max(dw) that is <= 2^-40 max(dw)/mean(dw).  When that bound
// exceeds kGuard (confident models: many tiny c(1-c)), two refinement passes add the
// exact rounding residual's positive and negative parts, each quantised with its own
// exponent (total error ~2^-80 relative).  `pass(inv_scale, beta)` enqueues the limb
// GEMMs of the limbs currently in `limbs`, scaled by inv_scale = 2^(41-e)/n (negative:
// subtract), accumulating into h when beta = 1.
constexpr double kGuard = 1e-11;

template <class Pass>
int limb_hessian(cudaStream_t st, int64_t n, int64_t np, const double* dw, uint8_t* limbs, Pass pass) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  SIMOPT_REQUIRE(cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone,
                 SIMOPT_E_CONFIG, "the limb Hessian reads max(dw) on the host: not capturable");
  char* sc = static_cast<char*>(simopt_scratch(st, 64 + 2 * (size_t)n * sizeof(double)));
  SIMOPT_REQUIRE(sc != nullptr, SIMOPT_E_CUDA, "%s", simopt_last_error());
  unsigned long long* mx = reinterpret_cast<unsigned long long*>(sc);
  double* sum = reinterpret_cast<double*>(sc + 8);
  double* rpos = reinterpret_cast<double*>(sc + 64);
  double* rneg = rpos + n;
  auto stats = [&](const double* w, double* host) -> int {
    SIMOPT_CUDA(cudaMemsetAsync(sc, 0, 16, st));
    k_dw_stats<<<egrid(n), 256, 0, st>>>(w, n, mx, sum);
    SIMOPT_CHECK_LAUNCH("k_dw_stats");
    SIMOPT_CUDA(cudaMemcpyAsync(host, sc, 16, cudaMemcpyDeviceToHost, st));
    SIMOPT_CUDA(cudaStreamSynchronize(st));
    return SIMOPT_OK;
  };
  double hs[2];
  if (int rc = stats(dw, hs)) return rc;
  double m;
  memcpy(&m, &hs[0], sizeof m);  // max arrived as IEEE bits
  const double mean = hs[1] / (double)n;
  const int e = limb_exponent(m);
  const bool refine = m > 0.0 && ldexp(1.0, -(e + 1)) > kGuard * mean;
  k_limbs<<<egrid(np), 256, 0, st>>>(dw, n, np, ldexp(1.0, e), limbs, refine ? rpos : nullptr,
                                     refine ? rneg : nullptr);
  SIMOPT_CHECK_LAUNCH("k_limbs");
  if (int rc = pass(ldexp(1.0, kFixBits - e) / (double)n, 0)) return rc;
  g_passes = 1;
  if (!refine) return SIMOPT_OK;
  for (int sgn = 0; sgn < 2; ++sgn) {
    const double* r = sgn ? rneg : rpos;
    if (int rc = stats(r, hs)) return rc;
    double mr;
    memcpy(&mr, &hs[0], sizeof mr);
    if (!(mr > 0.0)) continue;
    const int er = limb_exponent(mr);
    k_limbs<<<egrid(np), 256, 0, st>>>(r, n, np, ldexp(1.0, er), limbs, nullptr, nullptr);
    SIMOPT_CHECK_LAUNCH("k_limbs");
    const double inv = ldexp(1.0, kFixBits - er) / (double)n;
    if (int rc = pass(sgn ? -inv : inv, 1)) return rc;
    ++g_passes;
  }
  return SIMOPT_OK;
}

}  // namespace

extern "C" int simopt_xtdx_last_passes(void) { return g_passes; }

// Sample-block width ch (a power of two, 64..4096) and padded row count np of the u8
// operand for n rows; the operand occupies (np / ch) * d * (ch + 32) bytes.
extern "C" int simopt_u8t_geometry(int64_t n, int64_t* ch, int64_t* np) {
  int64_t c = 64;  // >= the tcgen05 kernel's 64-sample stage
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
  const int64_t nt = (d + kBM - 1) / kBM;
  const int64_t tiles = nt * (nt + 1) / 2;
  SIMOPT_REQUIRE(tiles < (1LL << 31), SIMOPT_E_CONFIG, "d too large");
  return limb_hessian(st, n, np, dw, limbs, [&](double inv, int beta) -> int {
    for (int64_t c0 = 0; c0 < np; c0 += kChunk) {
      const int64_t c1 = c0 + kChunk < np ? c0 + kChunk : np;
      for (int k = 0; k < kLimbs; ++k) {
        const double scale = ldexp(1.0, kLimbBits * k - kFixBits) * inv;
        k_xtdx_i8<<<(unsigned)tiles, kThreads, 0, st>>>(xt, lg, d, limbs + k * np, c0, c1, scale, beta, h);
        SIMOPT_CHECK_LAUNCH("k_xtdx_i8");
        beta = 1;
      }
    }
    return SIMOPT_OK;
  });
}

// upper-triangle list of 128 x 96 tiles (tile (bi, bj) holds some j >= i), cached per d
static int upper_tiles(int64_t d, int2** out, int* count, int tn = kTN, int tm = kTM) {
  static std::mutex mu;
  static std::vector<std::pair<int64_t, std::pair<int2*, int>>> cache;
  std::lock_guard<std::mutex> lock(mu);
  const int64_t key = (d * 1024 + tn) * 1024 + tm;
  for (auto& e : cache)
    if (e.first == key) {
      *out = e.second.first;
      *count = e.second.second;
      return SIMOPT_OK;
    }
  std::vector<int2> v;
  for (int64_t bi = 0; bi * tm < d; ++bi)
    for (int64_t bj = 0; bj * tn < d; ++bj)
      if (bj * tn + tn - 1 >= bi * tm) v.push_back(make_int2((int)bi, (int)bj));
  int2* tiles = nullptr;
  SIMOPT_CUDA(cudaMalloc(&tiles, v.size() * sizeof(int2)));
  SIMOPT_CUDA(cudaMemcpy(tiles, v.data(), v.size() * sizeof(int2), cudaMemcpyHostToDevice));
  cache.push_back({key, {tiles, (int)v.size()}});
  *out = tiles;
  *count = (int)v.size();
  return SIMOPT_OK;
}

// tcgen05 version of simopt_logistic_xtdx_i8 (same operands and result).
extern "C" int simopt_logistic_xtdx_tc(void* stream, const uint8_t* xt, int64_t np, int64_t n,
                                       int64_t d, const double* dw, uint8_t* limbs, double* h) {
  SIMOPT_REQUIRE(n >= 1 && d >= 1, SIMOPT_E_DIMENSION, "empty design matrix");
  int64_t ch = 0, np_want = 0;
  simopt_u8t_geometry(n, &ch, &np_want);
  SIMOPT_REQUIRE(np == np_want, SIMOPT_E_CONFIG, "np must come from simopt_u8t_geometry");
  cudaStream_t st = as_stream(stream);
  int lg = 0;
  while ((1LL << lg) < ch) ++lg;
  int2* tiles = nullptr;
  int ntiles = 0;
  SIMOPT_REQUIRE(upper_tiles(d, &tiles, &ntiles) == SIMOPT_OK, SIMOPT_E_CUDA, "%s", simopt_last_error());
  // > half the SM's shared memory: one CTA per SM, which then owns all 512 TMEM columns
  const size_t smem = sizeof(TcSmem) + 1024 > 120 * 1024 ? sizeof(TcSmem) + 1024 : 120 * 1024;
  static bool attr = false;
  if (!attr) {
    SIMOPT_CUDA(cudaFuncSetAttribute(k_xtdx_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  return limb_hessian(st, n, np, dw, limbs, [&](double inv, int beta) -> int {
    for (int64_t c0 = 0; c0 < np; c0 += kChunk) {
      const int64_t c1 = c0 + kChunk < np ? c0 + kChunk : np;
      k_xtdx_tc<<<ntiles, kTT, smem, st>>>(xt, lg, d, limbs, np, tiles, c0, c1, inv, beta, h);
      SIMOPT_CHECK_LAUNCH("k_xtdx_tc");
      beta = 1;
    }
    return SIMOPT_OK;
  });
}

// TMA-fed tcgen05 version (k_xtdx_tma): same operands and result as simopt_logistic_xtdx_tc.
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

static int xtdx_tma(void* stream, const uint8_t* xt, int64_t np, int64_t n, int64_t d,
                    const double* dw, uint8_t* limbs, double* h, bool force_pair) {
  SIMOPT_REQUIRE(n >= 1 && d >= 1, SIMOPT_E_DIMENSION, "empty design matrix");
  SIMOPT_REQUIRE(d < (1LL << 31), SIMOPT_E_CONFIG, "d too large for a tensor map");
  int64_t ch = 0, np_want = 0;
  simopt_u8t_geometry(n, &ch, &np_want);
  SIMOPT_REQUIRE(np == np_want, SIMOPT_E_CONFIG, "np must come from simopt_u8t_geometry");
  PFN_cuTensorMapEncodeTiled_v12000 encode = encode_fn();
  SIMOPT_REQUIRE(encode != nullptr, SIMOPT_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cudaStream_t st = as_stream(stream);
  int lg = 0;
  while ((1LL << lg) < ch) ++lg;
  int2* tiles = nullptr;
  int ntiles = 0;
  SIMOPT_REQUIRE(upper_tiles(d, &tiles, &ntiles) == SIMOPT_OK, SIMOPT_E_CUDA, "%s", simopt_last_error());
  // X^T blocks [np/ch][d][ch + kRowPad] u8; boxes of 16 samples x {128 | 96} feature rows
  const int64_t rs = ch + kRowPad;
  CUtensorMap ma, mb, ml;
  const cuuint64_t gdim[3] = {(cuuint64_t)rs, (cuuint64_t)d, (cuuint64_t)(np / ch)};
  const cuuint64_t gstr[2] = {(cuuint64_t)rs, (cuuint64_t)(d * rs)};
  const cuuint32_t estr[3] = {1, 1, 1};
  // SIMOPT_XTDX_TMA_BOX=16: 16-byte boxes per K half (no swizzle); default 64: one
  // 64-byte swizzled box per operand and stage (whole 32-byte sectors, 4x fewer requests)
  static const int sw = [] {
    const char* e = getenv("SIMOPT_XTDX_TMA_BOX");
    return e && atoi(e) == 16 ? 16 : 64;
  }();
  const cuuint32_t bw = (cuuint32_t)sw;
  const cuuint32_t box_a[3] = {bw, (cuuint32_t)kTM, 1}, box_b[3] = {bw, (cuuint32_t)kTN, 1};
  const CUtensorMapSwizzle swz = sw == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r1 = encode(&ma, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(xt), gdim, gstr, box_a,
                       estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = encode(&mb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(xt), gdim, gstr, box_b,
                       estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const cuuint64_t ldim[2] = {(cuuint64_t)np, (cuuint64_t)kLimbs};
  const cuuint64_t lstr[1] = {(cuuint64_t)np};
  const cuuint32_t box_l[2] = {(cuuint32_t)kTK, (cuuint32_t)kLimbs}, lestr[2] = {1, 1};
  CUresult r3 = encode(&ml, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, limbs, ldim, lstr, box_l, lestr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SIMOPT_REQUIRE(r1 == CUDA_SUCCESS && r2 == CUDA_SUCCESS && r3 == CUDA_SUCCESS, SIMOPT_E_CUDA,
                 "tensor map encoding failed (%d, %d, %d)", (int)r1, (int)r2, (int)r3);
  static const bool pair_env = [] {
    const char* e = getenv("SIMOPT_XTDX_PAIR");
    return e && atoi(e) == 1;
  }();
  if ((pair_env || force_pair) && sw == 64) {  // CTA pairs (k_xtdx_pair): 256 x 96 tiles
    int2* tp = nullptr;
    int ntp = 0;
    SIMOPT_REQUIRE(upper_tiles(d, &tp, &ntp, kTN, 2 * kTM) == SIMOPT_OK, SIMOPT_E_CUDA, "%s",
                   simopt_last_error());
    const size_t smem_p = sizeof(PairSmem) + 1024;
    static bool attr_p = false;
    if (!attr_p) {
      SIMOPT_CUDA(cudaFuncSetAttribute(k_xtdx_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p));
      attr_p = true;
    }
    return limb_hessian(st, n, np, dw, limbs, [&](double inv, int beta) -> int {
      for (int64_t c0 = 0; c0 < np; c0 += kChunk) {
        const int64_t c1 = c0 + kChunk < np ? c0 + kChunk : np;
        k_xtdx_pair<<<2 * ntp, kQT, smem_p, st>>>(ma, mb, ml, lg, d, tp, c0, c1, inv, beta, h);
        SIMOPT_CHECK_LAUNCH("k_xtdx_pair");
        beta = 1;
      }
      return SIMOPT_OK;
    });
  }
  const size_t smem = sizeof(TmaSmem) + 1024;
  // SIMOPT_XTDX_TMA_WIDE=0: five N = 96 MMAs per K step instead of two N = 240 (comparison)
  static const bool wide = [] {
    const char* e = getenv("SIMOPT_XTDX_TMA_WIDE");
    return !(e && atoi(e) == 0);
  }();
  auto kern = sw == 64 ? (wide ? k_xtdx_tma<64, true> : k_xtdx_tma<64, false>) : k_xtdx_tma<16, false>;
  static bool attr = false;
  if (!attr) {
    SIMOPT_CUDA(cudaFuncSetAttribute(k_xtdx_tma<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SIMOPT_CUDA(cudaFuncSetAttribute(k_xtdx_tma<64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SIMOPT_CUDA(cudaFuncSetAttribute(k_xtdx_tma<64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  return limb_hessian(st, n, np, dw, limbs, [&](double inv, int beta) -> int {
    for (int64_t c0 = 0; c0 < np; c0 += kChunk) {
      const int64_t c1 = c0 + kChunk < np ? c0 + kChunk : np;
      kern<<<ntiles, kQT, smem, st>>>(ma, mb, ml, lg, d, tiles, c0, c1, inv, beta, h);
      SIMOPT_CHECK_LAUNCH("k_xtdx_tma");
      beta = 1;
    }
    return SIMOPT_OK;
  });
}

extern "C" int simopt_logistic_xtdx_tma(void* stream, const uint8_t* xt, int64_t np, int64_t n,
                                        int64_t d, const double* dw, uint8_t* limbs, double* h) {
  return xtdx_tma(stream, xt, np, n, d, dw, limbs, h, false);
}

extern "C" int simopt_logistic_xtdx_pair(void* stream, const uint8_t* xt, int64_t np, int64_t n,
                                         int64_t d, const double* dw, uint8_t* limbs, double* h) {
  return xtdx_tma(stream, xt, np, n, d, dw, limbs, h, true);
}
