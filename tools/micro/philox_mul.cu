// Microbenchmark: Philox4x64-10 block rate on sm_100a for different 64x64->128 product
// formulations, and raw IMAD / IMAD.WIDE / IADD3 throughput (which pipe bounds k_nv_resample).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o philox_mul philox_mul.cu && ./philox_mul
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define M0 0xD2E7470EE14C6C93ULL
#define M1 0xCA5A826395121157ULL
#define W0 0x9E3779B97F4A7C15ULL
#define W1 0xBB67AE8584CAA73BULL

// V0: what the product code does (a*b + __umul64hi; ptxas picks the instruction mix)
__device__ __forceinline__ void mul_v0(uint64_t a, uint64_t m, uint64_t& hi, uint64_t& lo) {
  lo = a * m;
  hi = __umul64hi(a, m);
}

// V1: four mul.wide.u32 partial products, combined by 32-bit add-with-carry (ALU)
__device__ __forceinline__ void mul_v1(uint64_t a, uint64_t m, uint64_t& hi, uint64_t& lo) {
  const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32);
  const uint32_t m0 = (uint32_t)m, m1 = (uint32_t)(m >> 32);
  uint32_t l0, l1, h0, h1;
  asm("{\n\t.reg .u64 p00, p01, p10, p11;\n\t.reg .u32 q0, q1, r0, r1, s0, s1, t0, t1, x;\n\t"
      "mul.wide.u32 p00, %4, %6;\n\t"
      "mul.wide.u32 p01, %4, %7;\n\t"
      "mul.wide.u32 p10, %5, %6;\n\t"
      "mul.wide.u32 p11, %5, %7;\n\t"
      "mov.b64 {q0, q1}, p00;\n\t"
      "mov.b64 {r0, r1}, p01;\n\t"
      "mov.b64 {s0, s1}, p10;\n\t"
      "mov.b64 {t0, t1}, p11;\n\t"
      "mov.b32 %0, q0;\n\t"
      "add.cc.u32 x, q1, r0;\n\t"
      "addc.cc.u32 %2, t0, r1;\n\t"
      "addc.u32 %3, t1, 0;\n\t"
      "add.cc.u32 %1, x, s0;\n\t"
      "addc.cc.u32 %2, %2, s1;\n\t"
      "addc.u32 %3, %3, 0;\n\t"
      "}"
      : "=r"(l0), "=r"(l1), "=r"(h0), "=r"(h1)
      : "r"(a0), "r"(a1), "r"(m0), "r"(m1));
  lo = ((uint64_t)l1 << 32) | l0;
  hi = ((uint64_t)h1 << 32) | h0;
}

// V2: eight 32-bit multiply-adds with carry flags (mul.lo/hi, mad.lo.cc, madc.hi): no
// 64-bit register pairs, so no moves into aligned accumulators
__device__ __forceinline__ void mul_v2(uint64_t a, uint64_t m, uint64_t& hi, uint64_t& lo) {
  const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32);
  const uint32_t m0 = (uint32_t)m, m1 = (uint32_t)(m >> 32);
  uint32_t r0, r1, r2, r3;
  asm("{\n\t.reg .u32 t1, t2, t3;\n\t"
      "mul.lo.u32 %0, %4, %6;\n\t"
      "mul.hi.u32 t1, %4, %6;\n\t"
      "mad.lo.cc.u32 t1, %4, %7, t1;\n\t"
      "madc.hi.u32 t2, %4, %7, 0;\n\t"
      "mad.lo.cc.u32 %1, %5, %6, t1;\n\t"
      "madc.hi.cc.u32 t2, %5, %6, t2;\n\t"
      "addc.u32 t3, 0, 0;\n\t"
      "mad.lo.cc.u32 %2, %5, %7, t2;\n\t"
      "madc.hi.u32 %3, %5, %7, t3;\n\t"
      "}"
      : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
      : "r"(a0), "r"(a1), "r"(m0), "r"(m1));
  lo = ((uint64_t)r1 << 32) | r0;
  hi = ((uint64_t)r3 << 32) | r2;
}

// V3: cross products summed as one 64-bit add with carry, the high product's 64-bit
// addend (X.hi + carries) formed by ALU add-with-carry straight into an aligned pair
__device__ __forceinline__ void mul_v3(uint64_t a, uint64_t m, uint64_t& hi, uint64_t& lo) {
  const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32);
  const uint32_t m0 = (uint32_t)m, m1 = (uint32_t)(m >> 32);
  uint64_t h;
  uint32_t l0, l1;
  asm("{\n\t.reg .u64 X, T, Y, Z;\n\t.reg .u32 c, x0, x1, y0, y1, z0, z1;\n\t"
      "mul.wide.u32 X, %3, %6;\n\t"
      "mul.wide.u32 T, %4, %5;\n\t"
      "add.cc.u64 X, X, T;\n\t"
      "addc.u32 c, 0, 0;\n\t"
      "mul.wide.u32 Y, %3, %5;\n\t"
      "mov.b64 {y0, y1}, Y;\n\t"
      "mov.b64 {x0, x1}, X;\n\t"
      "mov.b32 %1, y0;\n\t"
      "add.cc.u32 %2, y1, x0;\n\t"
      "addc.cc.u32 z0, x1, 0;\n\t"
      "addc.u32 z1, c, 0;\n\t"
      "mov.b64 Z, {z0, z1};\n\t"
      "mad.wide.u32 %0, %4, %6, Z;\n\t"
      "}"
      : "=l"(h), "=r"(l0), "=r"(l1)
      : "r"(a0), "r"(a1), "r"(m0), "r"(m1));
  lo = ((uint64_t)l1 << 32) | l0;
  hi = h;
}

template <int V>
__device__ __forceinline__ void mul(uint64_t a, uint64_t m, uint64_t& hi, uint64_t& lo) {
  if (V == 0) mul_v0(a, m, hi, lo);
  else if (V == 1) mul_v1(a, m, hi, lo);
  else if (V == 2) mul_v2(a, m, hi, lo);
  else mul_v3(a, m, hi, lo);
}

template <int V>
__global__ void k_philox(uint64_t k0i, uint64_t k1i, int64_t nblocks, uint64_t* out) {
  uint64_t acc = 0;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nblocks;
       b += (int64_t)gridDim.x * blockDim.x) {
    uint64_t c0 = (uint64_t)b + 1, c1 = 7, c2 = 0, c3 = 0, k0 = k0i, k1 = k1i;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      uint64_t hi0, lo0, hi1, lo1;
      mul<V>(c0, M0, hi0, lo0);
      mul<V>(c2, M1, hi1, lo1);
      const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
      c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
      k0 += W0; k1 += W1;
    }
    acc ^= c0 ^ c1 ^ c2 ^ c3;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_check(uint64_t* out) {
  uint64_t x = 0x123456789abcdefULL, bad1 = 0, bad2 = 0;
  for (int i = 0; i < 100000; ++i) {
    x = x * 6364136223846793005ULL + 1442695040888963407ULL;
    const uint64_t m = (i & 1) ? M0 : M1 ^ x;
    uint64_t h0, l0, h1, l1, h2, l2;
    mul_v0(x, m, h0, l0);
    mul_v1(x, m, h1, l1);
    mul_v2(x, m, h2, l2);
    bad1 += (h0 != h1) | (l0 != l1);
    bad2 += (h0 != h2) | (l0 != l2);
    mul_v3(x, m, h2, l2);
    bad2 += (h0 != h2) | (l0 != l2);
  }
  out[0] = bad1;
  out[1] = bad2;
}

__global__ void k_imad_wide(uint64_t* out, uint32_t m, int n) {
  uint64_t s[8];
  for (int k = 0; k < 8; ++k) s[k] = threadIdx.x + k;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint64_t r;
      asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"((uint32_t)s[k]), "r"(m), "l"(s[k]));
      s[k] = r;
    }
  uint64_t t = 0;
  for (int k = 0; k < 8; ++k) t ^= s[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void k_imad(uint32_t* out, uint32_t m, int n) {
  uint32_t s[8];
  for (int k = 0; k < 8; ++k) s[k] = threadIdx.x + k;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(s[k]) : "r"(m));
  uint32_t t = 0;
  for (int k = 0; k < 8; ++k) t ^= s[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void k_iadd(uint32_t* out, uint32_t m, int n) {
  uint32_t s[8];
  for (int k = 0; k < 8; ++k) s[k] = threadIdx.x + k;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("xor.b32 %0, %0, %1;\n\tadd.u32 %0, %0, %1;" : "+r"(s[k]) : "r"(m));
  uint32_t t = 0;
  for (int k = 0; k < 8; ++k) t ^= s[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
  uint64_t* d;
  cudaMalloc(&d, 148 * 64 * 1024 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double ghz = 1.965;
  float ms;
  const int n = 1 << 14;
  auto rate = [&](const char* name, double ops_per_thread_iter, auto launch) {
    launch(16);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    launch(n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = ops_per_thread_iter * n * (double)sms * 8 * 256;
    printf("%-14s %.1f ops/clk/SM\n", name, ops / (ms * 1e-3) / (sms * ghz * 1e9));
  };
  rate("IMAD.WIDE", 8, [&](int it) { k_imad_wide<<<sms * 8, 256>>>(d, 0x9E3779B9u, it); });
  rate("IMAD", 8, [&](int it) { k_imad<<<sms * 8, 256>>>((uint32_t*)d, 0x9E3779B9u, it); });
  rate("LOP3+IADD3", 16, [&](int it) { k_iadd<<<sms * 8, 256>>>((uint32_t*)d, 0x9E3779B9u, it); });
  const int64_t nb = 1LL << 28;
  // correctness: the three product forms agree on random operands
  {
    uint64_t* h;
    cudaMallocManaged(&h, 3 * 8);
    k_check<<<1, 1>>>(h);
    cudaDeviceSynchronize();
    printf("product forms agree: %s\n", (h[0] == 0 && h[1] == 0) ? "yes" : "NO");
  }
  for (int v = 0; v < 4; ++v) {
    for (int bpsm : {4, 8}) {
      auto go = [&]() {
        if (v == 0) k_philox<0><<<sms * bpsm, 256>>>(42, 7, nb, d);
        else if (v == 1) k_philox<1><<<sms * bpsm, 256>>>(42, 7, nb, d);
        else if (v == 2) k_philox<2><<<sms * bpsm, 256>>>(42, 7, nb, d);
        else k_philox<3><<<sms * bpsm, 256>>>(42, 7, nb, d);
      };
      go();
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      go();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("philox V%d (%d CTAs/SM): %.3f ms for 2^28 blocks = %.1f G blocks/s -> %.3f ms per 2.5e8 blocks\n",
             v, bpsm, ms, nb / (ms * 1e-3) / 1e9, ms * 2.5e8 / nb);
    }
  }
  return 0;
}
