// Maximum relative error of sqrt.approx.ftz.f32 (MUFU.SQRT) over every fp32 input in
// [2^-60, 80] -- the operand range of the newsvendor key's Box-Muller radius
// (csrc/newsvendor.cuh, nv_approx_pair: y = -2 log1p(-u1) in [2^-52, 75]).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o sqrt_approx_err sqrt_approx_err.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

__global__ void k_err(uint32_t lo, uint32_t hi, unsigned long long* worst) {
  double m = 0.0;
  for (uint32_t b = lo + blockIdx.x * blockDim.x + threadIdx.x; b < hi; b += gridDim.x * blockDim.x) {
    const float y = __uint_as_float(b);
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(y));
    const double t = sqrt((double)y);
    m = fmax(m, fabs((double)r - t) / t);
  }
  atomicMax(worst, (unsigned long long)__double_as_longlong(m));  // m >= 0: bits order as values
}

int main() {
  unsigned long long* w;
  cudaMalloc(&w, 8);
  cudaMemset(w, 0, 8);
  const float a = ldexpf(1.0f, -60), b = 80.0f;
  uint32_t lo, hi;
  memcpy(&lo, &a, 4);
  memcpy(&hi, &b, 4);
  k_err<<<148 * 8, 256>>>(lo, hi + 1, w);
  unsigned long long h = 0;
  cudaMemcpy(&h, w, 8, cudaMemcpyDeviceToHost);
  double m;
  memcpy(&m, &h, 8);
  printf("sqrt.approx.ftz.f32 max relative error on [2^-60, 80]: %.3e = 2^%.2f (%u inputs) %s\n", m,
         log2(m), hi + 1 - lo, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
