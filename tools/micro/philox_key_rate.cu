// Microbenchmark: the producer half of k_nv_resample_ws alone (Philox4x64-10 + the fp32
// Box-Muller key + shared-memory bucket count), for product formulations that move work
// between the heavy FMA pipe (IMAD.WIDE) and the ALU, and for round 0 carried
// incrementally (M0 * (c0 + 256) = M0 * c0 + (M0 << 8): a 128-bit add instead of a product).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2404_11631_b200/csrc \
//        -o philox_key_rate tools/micro/philox_key_rate.cu && ./philox_key_rate
// Every variant must produce the same XOR of keys (checked against variant 0).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "newsvendor.cuh"

// product formulations: 0 = a*m + __umul64hi (ptxas's mix), 1 = four mul.wide + ALU column sums
template <int F, uint64_t M>
__device__ __forceinline__ void mul128(uint64_t a, uint64_t& hi, uint64_t& lo) {
  if (F == 0) {
    lo = a * M;
    hi = __umul64hi(a, M);
  } else {
    uint32_t w0, w1, w2, w3;
    asm("{\n\t.reg .u64 t, q, r, s;\n\t.reg .u32 t1, q0, q1, r0, r1, s0, s1;\n\t"
        "mul.wide.u32 t, %4, %6;\n\t"
        "mul.wide.u32 q, %4, %7;\n\t"
        "mul.wide.u32 r, %5, %6;\n\t"
        "mul.wide.u32 s, %5, %7;\n\t"
        "mov.b64 {%0, t1}, t;\n\t"
        "mov.b64 {q0, q1}, q;\n\t"
        "mov.b64 {r0, r1}, r;\n\t"
        "mov.b64 {s0, s1}, s;\n\t"
        "add.cc.u32 %1, t1, q0;\n\t"
        "addc.cc.u32 %2, q1, s0;\n\t"
        "addc.u32 %3, s1, 0;\n\t"
        "add.cc.u32 %1, %1, r0;\n\t"
        "addc.cc.u32 %2, %2, r1;\n\t"
        "addc.u32 %3, %3, 0;\n\t"
        "}"
        : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
        : "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "n"((uint32_t)M), "n"((uint32_t)(M >> 32)));
    lo = (uint64_t)w1 << 32 | w0;
    hi = (uint64_t)w3 << 32 | w2;
  }
}

// Philox4x64-10 of counter (c0, hi, 0, 0) given round 0's product (h0, l0) = M0 * c0.
// F0/F1: formulation of the M0 / M1 products; mask selects per round (bit r: use F=1).
template <unsigned MaskM0, unsigned MaskM1>
__device__ __forceinline__ phx4 philox_from_r0(uint64_t hi0, uint64_t lo0, const phx_keys& rk,
                                               const phx_pre& pre) {
  uint64_t hi1, lo1;
  if (MaskM1 & 2u) mul128<1, PHILOX_M1>(hi0 ^ rk.k[1], hi1, lo1);
  else mul128<0, PHILOX_M1>(hi0 ^ rk.k[1], hi1, lo1);
  phx4 c;
  c.v[0] = hi1 ^ rk.k[2];
  c.v[1] = lo1;
  c.v[2] = pre.h1 ^ lo0 ^ rk.k[3];
  c.v[3] = pre.l1;
#pragma unroll
  for (int r = 2; r < 10; ++r) {
    if (MaskM0 & (1u << r)) mul128<1, PHILOX_M0>(c.v[0], hi0, lo0);
    else mul128<0, PHILOX_M0>(c.v[0], hi0, lo0);
    if (MaskM1 & (1u << r)) mul128<1, PHILOX_M1>(c.v[2], hi1, lo1);
    else mul128<0, PHILOX_M1>(c.v[2], hi1, lo1);
    phx4 o;
    o.v[0] = hi1 ^ c.v[1] ^ rk.k[2 * r];
    o.v[1] = lo1;
    o.v[2] = hi0 ^ c.v[3] ^ rk.k[2 * r + 1];
    o.v[3] = lo0;
    c = o;
  }
  return c;
}

constexpr int kThreads = 256;

template <bool kInc, unsigned MaskM0, unsigned MaskM1>
__global__ void __launch_bounds__(kThreads, 3)
    k_prod(const phx_keys rk, const phx_pre pre, uint64_t clo, int64_t nseg_total, uint32_t* out) {
  __shared__ __align__(16) uint32_t raw[NV_SEG];
  __shared__ int hist[NV_B];
  for (int i = threadIdx.x; i < NV_B; i += kThreads) hist[i] = 0;
  __syncthreads();
  uint32_t acc = 0;
  for (int64_t seg = blockIdx.x; seg < nseg_total; seg += gridDim.x) {
    const uint64_t c0 = clo + (uint64_t)seg * (NV_SEG / 4) + 1 + threadIdx.x;
    uint64_t h0, l0;
    if (kInc) mul128<0, PHILOX_M0>(c0, h0, l0);
#pragma unroll 1
    for (int t = threadIdx.x; t < NV_SEG / 4; t += kThreads) {
      if (!kInc) mul128<0, PHILOX_M0>(c0 + (uint64_t)(t - threadIdx.x), h0, l0);
      const phx4 w = philox_from_r0<MaskM0, MaskM1>(h0, l0, rk, pre);
      if (kInc) {  // M0 * (c + 256) = M0 * c + (M0 << 8)
        constexpr uint64_t kLo = PHILOX_M0 << 8, kHi = PHILOX_M0 >> 56;
        asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(l0), "+l"(h0) : "n"(kLo), "n"(kHi));
      }
      float z[4];
      nv_approx_pair(w.v[0], w.v[1], &z[0], &z[1]);
      nv_approx_pair(w.v[2], w.v[3], &z[2], &z[3]);
      uint32_t kk[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        kk[u] = nv_key(z[u], (uint32_t)(4 * t + u));
        atomicAdd(&hist[kk[u] >> (12 + NV_QBITS - 10)], 1);
      }
      reinterpret_cast<uint4*>(raw)[t] = make_uint4(kk[0], kk[1], kk[2], kk[3]);
    }
    __syncthreads();
    acc ^= raw[(threadIdx.x * 17) & (NV_SEG - 1)] ^ (uint32_t)hist[threadIdx.x];
    __syncthreads();
  }
  out[blockIdx.x * kThreads + threadIdx.x] = acc;
}

template <bool kInc, unsigned A, unsigned B>
float run(const phx_keys& rk, const phx_pre& pre, int grid, int64_t nseg, uint32_t* d, uint32_t* h,
          uint32_t* x) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_prod<kInc, A, B><<<grid, kThreads>>>(rk, pre, 1000, nseg, d);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    k_prod<kInc, A, B><<<grid, kThreads>>>(rk, pre, 1000, nseg, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaMemcpy(h, d, (size_t)grid * kThreads * 4, cudaMemcpyDeviceToHost);
  uint32_t v = 0;
  for (int i = 0; i < grid * kThreads; ++i) v ^= h[i];
  *x = v;
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t nseg = 10000LL * 25;  // C2: d = 10^4 products x 25 segments (2.5e8 Philox blocks)
  const phx_keys rk = phx_round_keys(42, 3);
  const phx_pre pre = phx_precompute(0, rk);
  uint32_t *d, *h;
  const int grid = sms * 3;
  cudaMalloc(&d, (size_t)grid * kThreads * 4);
  h = (uint32_t*)malloc((size_t)grid * kThreads * 4);
  uint32_t ref = 0, x = 0;
  float ms;
#define GO(INC, A, B, NAME)                                                                  \
  ms = run<INC, A, B>(rk, pre, grid, nseg, d, h, &x);                                        \
  if (ref == 0) ref = x;                                                                     \
  printf("%-44s %.3f ms  %s\n", NAME, ms, x == ref ? "same" : "DIFFERS");
  GO(false, 0u, 0u, "baseline (ptxas mix)")
  GO(true, 0u, 0u, "round 0 incremental")
  GO(true, 0u, 0x3FEu, "inc + M1 products as column sums")
  GO(true, 0x3FCu, 0u, "inc + M0 products as column sums")
  GO(true, 0x3FCu, 0x3FEu, "inc + all products as column sums")
  GO(true, 0x154u, 0x2AAu, "inc + alternate rounds (M0 even, M1 odd)")
  GO(true, 0x0F0u, 0x0F0u, "inc + rounds 4-7 column sums")
  GO(true, 0x30Cu, 0x0F2u, "inc + mixed 6 of 17")
  return 0;
}
