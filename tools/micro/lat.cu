// Microbenchmark: dependent-chain latency of DADD / DFMA / DMUL and FP64 throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain_add(double* out, double a, int n) {
  double s = out[threadIdx.x];
  for (int i = 0; i < n; ++i) { s = __dadd_rn(s, a); s = __dadd_rn(s, a); s = __dadd_rn(s, a); s = __dadd_rn(s, a); }
  out[threadIdx.x] = s;
}
__global__ void chain_fma(double* out, double a, int n) {
  double s = out[threadIdx.x];
  for (int i = 0; i < n; ++i) { s = fma(s, a, a); s = fma(s, a, a); s = fma(s, a, a); s = fma(s, a, a); }
  out[threadIdx.x] = s;
}
__global__ void tput_fma(double* out, double a, int n) {
  double s[8];
  for (int k = 0; k < 8; ++k) s[k] = out[blockIdx.x * blockDim.x + threadIdx.x] + k;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) s[k] = fma(s[k], a, a);
  double t = 0; for (int k = 0; k < 8; ++k) t += s[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void tput_add(double* out, double a, int n) {
  double s[8];
  for (int k = 0; k < 8; ++k) s[k] = out[blockIdx.x * blockDim.x + threadIdx.x] + k;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) s[k] = __dadd_rn(s[k], a);
  double t = 0; for (int k = 0; k < 8; ++k) t += s[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
  double* d; cudaMalloc(&d, 148 * 1024 * 8 * 8); cudaMemset(d, 0, 148 * 1024 * 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int n = 1 << 20;
  float ms;
  chain_add<<<1, 1>>>(d, 1e-9, 1000); cudaDeviceSynchronize();
  cudaEventRecord(e0); chain_add<<<1, 1>>>(d, 1e-9, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1); printf("DADD chain: %.2f ns/op = %.1f cycles @%d MHz\n", ms * 1e6 / (4.0 * n), ms * 1e6 / (4.0 * n) * clk / 1e6, clk / 1000);
  cudaEventRecord(e0); chain_fma<<<1, 1>>>(d, 0.999, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1); printf("DFMA chain: %.2f ns/op = %.1f cycles\n", ms * 1e6 / (4.0 * n), ms * 1e6 / (4.0 * n) * clk / 1e6);
  const int m = 1 << 14;
  for (int bs : {256, 512, 1024}) {
    tput_fma<<<148 * 4, bs>>>(d, 0.999, 100); cudaDeviceSynchronize();
    cudaEventRecord(e0); tput_fma<<<148 * 4, bs>>>(d, 0.999, m); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * m * 148.0 * 4 * bs;
    printf("DFMA throughput (bs=%d): %.2f TFLOP/s\n", bs, flops / (ms * 1e-3) / 1e12);
    cudaEventRecord(e0); tput_add<<<148 * 4, bs>>>(d, 1e-9, m); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DADD throughput (bs=%d): %.2f Gop/s\n", bs, 8.0 * m * 148.0 * 4 * bs / (ms * 1e-3) / 1e9);
  }
  return 0;
}
