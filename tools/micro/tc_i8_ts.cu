// Smoke test: A operand written into TMEM by tcgen05.st (lane m = row m, 8 x 32-bit columns
// = the row's 32 K-bytes), B in shared memory (SWIZZLE_NONE K-major canonical layout),
// D[128x64] s32 = A * B^T via tcgen05.mma.kind::i8 with A from TMEM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_i8_ts tc_i8_ts.cu && ./tc_i8_ts
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int M = 128, N = 64, K = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(const void* p) {
  return (uint64_t)((smem_u32(p) >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(256 >> 4) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ int coff(int r, int k) {
  return (r >> 3) * 256 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15);
}

__global__ void k(const uint8_t* A, const uint8_t* B, int* D) {
  __shared__ __align__(1024) uint8_t sb[N * K];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t taddr_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < N * K; e += blockDim.x) sb[coff(e / K, e % K)] = B[e];
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&taddr_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t taddr = taddr_sh;
  // A row m = 32*warp + lane -> TMEM lane m, columns 64..71 (after the 64 D columns)
  {
    const int m = warp * 32 + lane;
    uint32_t w[8];
    for (int j = 0; j < 8; ++j)
      w[j] = (uint32_t)A[m * K + 4 * j] | ((uint32_t)A[m * K + 4 * j + 1] << 8) |
             ((uint32_t)A[m * K + 4 * j + 2] << 16) | ((uint32_t)A[m * K + 4 * j + 3] << 24);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                     taddr + ((uint32_t)(warp * 32) << 16) + 64u),
                 "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint64_t db = make_desc(sb);
    const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}\n"
        ::"r"(taddr), "r"(taddr + 64u), "l"(db), "r"(idesc), "r"(0), "r"(0), "r"(0), "r"(0), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  asm volatile("{\n\t.reg .pred P1;\n\tWAIT:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra WAIT;\n\t}\n" ::"r"(smem_u32(&mbar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
          "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
          "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * N + c0 + j] = (int)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(taddr));
}

int main() {
  uint8_t hA[M * K], hB[N * K];
  srand(7);
  for (int i = 0; i < M * K; ++i) hA[i] = rand() & 255;
  for (int i = 0; i < N * K; ++i) hB[i] = rand() & 255;
  uint8_t *dA, *dB;
  int* dD;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  k<<<1, 128>>>(dA, dB, dD);
  printf("kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  static int hD[M * N];
  cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      int s = 0;
      for (int kk = 0; kk < K; ++kk) s += hA[m * K + kk] * hB[n * K + kk];
      if (s != hD[m * N + n] && bad++ < 5) printf("mismatch m=%d n=%d got %d want %d\n", m, n, hD[m * N + n], s);
    }
  printf("tcgen05 kind::i8 A from TMEM (tcgen05.st) 128x64x32: %s (%d mismatches)\n", bad ? "FAIL" : "OK", bad);
  return bad != 0;
}
