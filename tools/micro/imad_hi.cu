// Throughput of IMAD.HI.U32 (mul.hi.u32) vs IMAD (mul.lo / mad.lo) vs IMAD.WIDE on sm_100a:
// 8 independent chains per thread, 64 warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o imad_hi imad_hi.cu && ./imad_hi
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__global__ void k(uint32_t* out, uint32_t m, int n) {
  uint32_t s[8];
  for (int k = 0; k < 8; ++k) s[k] = threadIdx.x * 7 + k;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (V == 0) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(s[k]) : "r"(m));
      else if (V == 1) asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(s[k]) : "r"(m));
      else asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(s[k]) : "r"(m));
    }
  uint32_t t = 0;
  for (int k = 0; k < 8; ++k) t ^= s[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* d;
  cudaMalloc(&d, (size_t)sms * 8 * 256 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int n = 1 << 14;
  const double ghz = 1.965;
  const char* names[3] = {"IMAD.HI (mul.hi.u32)", "IMAD.HI (mad.hi.u32)", "IMAD (mad.lo.u32)"};
  for (int v = 0; v < 3; ++v) {
    auto go = [&](int nn) {
      if (v == 0) k<0><<<sms * 8, 256>>>(d, 0x9E3779B9u, nn);
      else if (v == 1) k<1><<<sms * 8, 256>>>(d, 0x9E3779B9u, nn);
      else k<2><<<sms * 8, 256>>>(d, 0x9E3779B9u, nn);
    };
    go(16);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    go(n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 8.0 * n * (double)sms * 8 * 256;
    printf("%-24s %.1f ops/clk/SM\n", names[v], ops / (ms * 1e-3) / (sms * ghz * 1e9));
  }
  return 0;
}
