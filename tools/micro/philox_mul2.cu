// Microbenchmark: Philox4x64-10 with the 64x64->128 products formed so that the heavy FMA
// pipe only issues the four IMAD.WIDE.U32 partial products (no IMAD.MOV / IMAD.X glue).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o philox_mul2 philox_mul2.cu && ./philox_mul2
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define M0 0xD2E7470EE14C6C93ULL
#define M1 0xCA5A826395121157ULL
#define W0 0x9E3779B97F4A7C15ULL
#define W1 0xBB67AE8584CAA73BULL

__device__ __forceinline__ void mul_v0(uint64_t a, uint64_t m, uint64_t& hi, uint64_t& lo) {
  lo = a * m;
  hi = __umul64hi(a, m);
}

// V5: four products with zero addend, then the column sums by 32-bit add-with-carry
// (t1 + q0 + r0 into word 1, q1 + r1 + s0 + carries into word 2, s1 + carries into word 3)
template <uint32_t m0, uint32_t m1>
__device__ __forceinline__ void mul_v5(uint32_t a0, uint32_t a1, uint32_t& w0, uint32_t& w1,
                                       uint32_t& w2, uint32_t& w3) {
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
      : "r"(a0), "r"(a1), "n"(m0), "n"(m1));
}

// V6: the middle column as one 64-bit add (q + r, carry into word 3), then t.hi and s
template <uint32_t m0, uint32_t m1>
__device__ __forceinline__ void mul_v6(uint32_t a0, uint32_t a1, uint32_t& w0, uint32_t& w1,
                                       uint32_t& w2, uint32_t& w3) {
  asm("{\n\t.reg .u64 t, q, r, s;\n\t.reg .u32 t1, q0, q1, r0, r1, s0, s1, c;\n\t"
      "mul.wide.u32 t, %4, %6;\n\t"
      "mul.wide.u32 q, %4, %7;\n\t"
      "mul.wide.u32 r, %5, %6;\n\t"
      "mul.wide.u32 s, %5, %7;\n\t"
      "mov.b64 {%0, t1}, t;\n\t"
      "mov.b64 {q0, q1}, q;\n\t"
      "mov.b64 {r0, r1}, r;\n\t"
      "mov.b64 {s0, s1}, s;\n\t"
      "add.cc.u32 q0, q0, r0;\n\t"
      "addc.cc.u32 q1, q1, r1;\n\t"
      "addc.u32 c, 0, 0;\n\t"
      "add.cc.u32 %1, t1, q0;\n\t"
      "addc.cc.u32 %2, s0, q1;\n\t"
      "addc.u32 %3, s1, c;\n\t"
      "}"
      : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
      : "r"(a0), "r"(a1), "n"(m0), "n"(m1));
}

struct S4 { uint32_t c[8]; };  // four 64-bit words as (lo, hi) pairs

template <int V>
__device__ __forceinline__ void round32(S4& x, uint64_t k0, uint64_t k1) {
  uint32_t a[4], b[4];
  if (V == 5) {
    mul_v5<(uint32_t)M0, (uint32_t)(M0 >> 32)>(x.c[0], x.c[1], a[0], a[1], a[2], a[3]);
    mul_v5<(uint32_t)M1, (uint32_t)(M1 >> 32)>(x.c[4], x.c[5], b[0], b[1], b[2], b[3]);
  } else {
    mul_v6<(uint32_t)M0, (uint32_t)(M0 >> 32)>(x.c[0], x.c[1], a[0], a[1], a[2], a[3]);
    mul_v6<(uint32_t)M1, (uint32_t)(M1 >> 32)>(x.c[4], x.c[5], b[0], b[1], b[2], b[3]);
  }
  // o0 = hi1 ^ c1 ^ k0; o1 = lo1; o2 = hi0 ^ c3 ^ k1; o3 = lo0
  S4 o;
  o.c[0] = b[2] ^ x.c[2] ^ (uint32_t)k0;
  o.c[1] = b[3] ^ x.c[3] ^ (uint32_t)(k0 >> 32);
  o.c[2] = b[0];
  o.c[3] = b[1];
  o.c[4] = a[2] ^ x.c[6] ^ (uint32_t)k1;
  o.c[5] = a[3] ^ x.c[7] ^ (uint32_t)(k1 >> 32);
  o.c[6] = a[0];
  o.c[7] = a[1];
  x = o;
}

template <int V>
__global__ void k_philox(uint64_t k0i, uint64_t k1i, int64_t nblocks, uint64_t* out) {
  uint64_t acc = 0;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nblocks;
       b += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k0 = k0i, k1 = k1i;
    if (V == 0) {
      uint64_t c0 = (uint64_t)b + 1, c1 = 7, c2 = 0, c3 = 0;
#pragma unroll
      for (int r = 0; r < 10; ++r) {
        uint64_t hi0, lo0, hi1, lo1;
        mul_v0(c0, M0, hi0, lo0);
        mul_v0(c2, M1, hi1, lo1);
        const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += W0; k1 += W1;
      }
      acc ^= c0 ^ c1 ^ c2 ^ c3;
    } else {
      const uint64_t c0 = (uint64_t)b + 1;
      S4 x = {{(uint32_t)c0, (uint32_t)(c0 >> 32), 7, 0, 0, 0, 0, 0}};
#pragma unroll
      for (int r = 0; r < 10; ++r) {
        round32<V>(x, k0, k1);
        k0 += W0; k1 += W1;
      }
      acc ^= ((uint64_t)x.c[1] << 32 | x.c[0]) ^ ((uint64_t)x.c[3] << 32 | x.c[2]) ^
             ((uint64_t)x.c[5] << 32 | x.c[4]) ^ ((uint64_t)x.c[7] << 32 | x.c[6]);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  uint64_t* d;
  cudaMalloc(&d, 148 * 64 * 1024 * 8);
  uint64_t* h = (uint64_t*)malloc(148 * 8 * 256 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t nb = 1LL << 28;
  uint64_t ref = 0;
  for (int v : {0, 5, 6}) {
    for (int bpsm : {4, 8}) {
      auto go = [&]() {
        if (v == 0) k_philox<0><<<sms * bpsm, 256>>>(42, 7, nb, d);
        else if (v == 5) k_philox<5><<<sms * bpsm, 256>>>(42, 7, nb, d);
        else k_philox<6><<<sms * bpsm, 256>>>(42, 7, nb, d);
      };
      go();
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      go();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(h, d, (size_t)sms * bpsm * 256 * 8, cudaMemcpyDeviceToHost);
      uint64_t x = 0;
      for (int64_t i = 0; i < (int64_t)sms * bpsm * 256; ++i) x ^= h[i];
      if (v == 0 && bpsm == 4) ref = x;
      printf("philox V%d (%d CTAs/SM): %.3f ms per 2^28 blocks -> %.3f ms per 2.5e8; %s\n", v, bpsm, ms,
             ms * 2.5e8 / nb, x == ref ? "same output" : "OUTPUT DIFFERS");
    }
  }
  return 0;
}
