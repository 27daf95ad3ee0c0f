// Microbenchmark: legacy warp-level integer MMA (mma.sync.m16n8k32.u8.u8.s32, SASS IMMA)
// throughput on sm_100a -- the candidate for an exact limb-decomposed X^T D X.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void imma(int (&c)[4], unsigned a0, unsigned a1, unsigned a2, unsigned a3,
                                     unsigned b0, unsigned b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__global__ void tput(int* out, unsigned a, unsigned b, int n) {
  int c[8][4];
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = c[k][2] = c[k][3] = threadIdx.x;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) imma(c[k], a, a + 1, a + 2, a + 3, b, b + k);
  int t = 0;
  for (int k = 0; k < 8; ++k) t += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
  int* out;
  cudaMalloc(&out, 148 * 16 * 1024 * sizeof(int));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int n = 4096;
  for (int warps : {4, 8, 16}) {
    const int grid = 148 * 4, block = 32 * warps;
    tput<<<grid, block>>>(out, 3, 5, n);
    cudaEventRecord(e0);
    tput<<<grid, block>>>(out, 3, 5, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 2.0 * 16 * 8 * 32 * 8 * n * (double)grid * warps;
    printf("IMMA m16n8k32 u8: %d warps/CTA: %.1f TOPS\n", warps, ops / ms / 1e9);
  }
  return 0;
}
