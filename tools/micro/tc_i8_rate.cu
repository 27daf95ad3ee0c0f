// Throughput of tcgen05.mma.kind::i8 (M = 128, cta_group::1) by N, A from TMEM (TS) or from
// shared memory (SS): one CTA per SM issues `stages` x (kMMA MMAs) back to back on fixed
// operands (contents irrelevant), committing to an mbarrier every stage and waiting 4
// stages behind.  Prints the achieved dense int8 TOPS for each N -- the ceiling of the
// limb-Hessian kernels' inner loop (csrc/hessian_i8.cu).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_i8_rate tc_i8_rate.cu && ./tc_i8_rate
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(const void* p, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((smem_u32(p) >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
               "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

template <int N, bool kTS>
__global__ void __launch_bounds__(128, 1) k_rate(int stages, int mmas, int* sink) {
  __shared__ __align__(1024) uint8_t a[128 * 32];
  __shared__ __align__(1024) uint8_t b[256 * 32];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t taddr_sh;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 32; i += 128) a[i] = (uint8_t)(i * 7);
  for (int i = tid; i < 256 * 32; i += 128) b[i] = (uint8_t)(i * 3);
  if (tid == 0) {
    for (int q = 0; q < 4; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[q])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t taddr = taddr_sh;
  if (tid == 0) {
    const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = make_desc(a, 128, 256), db = make_desc(b, 128, 256);
    const uint32_t ta = taddr + 480;
    if (kTS) asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(ta), "l"(da));
    for (int t = 0; t < stages; ++t) {
      if (t >= 4) mbar_wait(&bar[t & 3], (uint32_t)(((t - 4) >> 2) & 1));
      for (int k = 0; k < mmas; ++k) {
        constexpr int nacc = (480 / N) < 5 ? (480 / N) : 5;  // distinct accumulators, as the 5 limbs
        const uint32_t dcol = taddr + (uint32_t)((k % nacc) * N);
        if (kTS)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}\n"
                       ::"r"(dcol), "r"(ta), "l"(db), "r"(idesc), "r"(1), "r"(0), "r"(0), "r"(0), "r"(0));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
                       ::"r"(dcol), "l"(da), "l"(db), "r"(idesc), "r"(1));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&bar[t & 3])));
    }
    for (int t = stages - 4 > 0 ? stages - 4 : 0; t < stages; ++t) mbar_wait(&bar[t & 3], (uint32_t)((t >> 2) & 1));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr));
  if (tid == 0 && stages < 0) *sink = 1;
}

template <int N, bool kTS>
void run(int sms) {
  const int stages = 20000, mmas = 10;
  int* sink;
  cudaMalloc(&sink, 4);
  k_rate<N, kTS><<<sms, 128>>>(10, mmas, sink);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_rate<N, kTS><<<sms, 128>>>(stages, mmas, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * 128 * N * 32 * (double)mmas * stages * sms;
  printf("N=%3d %s: %.3f ms, %.1f TOPS, %.1f ns per MMA per SM  (%s)\n", N, kTS ? "TS" : "SS", ms,
         ops / (ms * 1e-3) / 1e12, ms * 1e6 / ((double)mmas * stages), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, true>(sms);
  run<80, true>(sms);
  run<96, true>(sms);
  run<128, true>(sms);
  run<256, true>(sms);
  run<96, false>(sms);
  run<256, false>(sms);
  return 0;
}
