// Throughput of tcgen05.mma.cta_group::2.kind::i8 (M = 256 over a CTA pair, SS operands)
// by N: one cluster of 2 CTAs per TPC, the leader issues `stages` x 4 MMAs back to back,
// committing (multicast to both CTAs) every stage and waiting 4 stages behind.  Compare
// with tools/micro/tc_i8_rate.cu (cta_group::1).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_i8_pair_rate tc_i8_pair_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw64(const void* p) {
  return (uint64_t)((smem_u32(p) >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
               "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_rate2(int stages, int* sink) {
  __shared__ __align__(1024) uint8_t a[128 * 64];
  __shared__ __align__(1024) uint8_t b[128 * 64];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t taddr_sh;
  const int tid = threadIdx.x, warp = tid >> 5;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = tid; i < 128 * 64; i += 128) { a[i] = (uint8_t)i; b[i] = (uint8_t)(3 * i); }
  if (tid == 0) {
    for (int q = 0; q < 4; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[q])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t taddr = taddr_sh;
  if (tid == 0 && rank == 0) {
    const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    for (int t = 0; t < stages; ++t) {
      if (t >= 4) mbar_wait(&bar[t & 3], (uint32_t)(((t - 4) >> 2) & 1));
      for (int k = 0; k < 4; ++k) {
        const uint32_t dcol = taddr + (uint32_t)((k & 1) * N);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
                     ::"r"(dcol), "l"(desc_sw64(a + (k & 1) * 32)), "l"(desc_sw64(b + (k & 1) * 32)), "r"(idesc), "r"(1));
      }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   ::"r"(smem_u32(&bar[t & 3])), "h"((uint16_t)3));
    }
  }
  if (tid == 0) {
    for (int t = stages - 4 > 0 ? stages - 4 : 0; t < stages; ++t) mbar_wait(&bar[t & 3], (uint32_t)((t >> 2) & 1));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(taddr));
  if (tid == 0 && stages < 0) *sink = 1;
}

template <int N>
void run(int sms) {
  const int stages = 20000;
  int* sink;
  cudaMalloc(&sink, 4);
  k_rate2<N><<<sms, 128>>>(10, sink);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_rate2<N><<<sms, 128>>>(stages, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * 256 * N * 32 * 4.0 * stages * (sms / 2);
  printf("pair N=%3d: %.3f ms, %.1f TOPS, %.1f ns per MMA per pair (%s)\n", N, ms, ops / (ms * 1e-3) / 1e12,
         ms * 1e6 / (4.0 * stages), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<128>(sms);
  run<160>(sms);
  run<240>(sms);
  run<256>(sms);
  return 0;
}
