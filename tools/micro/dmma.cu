// Microbenchmark: FP64 tensor-pipe (DMMA, mma.sync.m8n8k4.f64) peak on sm_100a, next to
// DFMA.  Each warp keeps 8 independent accumulator pairs in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma dmma.cu && ./dmma
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void tput_dmma(double* out, double a, double b, int n) {
  double c[8][2];
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = threadIdx.x + k;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(c[k][0], c[k][1], a, b);
  double t = 0;
  for (int k = 0; k < 8; ++k) t += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void tput_fma(double* out, double a, int n) {
  double s[8];
  for (int k = 0; k < 8; ++k) s[k] = threadIdx.x + k;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) s[k] = fma(s[k], a, a);
  double t = 0;
  for (int k = 0; k < 8; ++k) t += s[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 16 * 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int n = 4096;
  for (int warps : {4, 8, 16}) {
    const int grid = 148 * 4, block = 32 * warps;
    tput_dmma<<<grid, block>>>(out, 1.0, 1e-300, n);
    cudaEventRecord(e0);
    tput_dmma<<<grid, block>>>(out, 1.0, 1e-300, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // one m8n8k4 = 8*8*4 FMA = 512 flops per warp-instruction
    const double flops = 512.0 * 8 * n * (double)grid * warps;
    printf("DMMA m8n8k4: %d warps/CTA x %d CTAs: %.2f TFLOP/s\n", warps, grid, flops / ms / 1e9);
    tput_fma<<<grid, block>>>(out, 1.0000001, n);
    cudaEventRecord(e0);
    tput_fma<<<grid, block>>>(out, 1.0000001, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA        : %d warps/CTA x %d CTAs: %.2f TFLOP/s\n", warps, grid,
           2.0 * 8 * n * (double)grid * block / ms / 1e9);
  }
  return 0;
}
