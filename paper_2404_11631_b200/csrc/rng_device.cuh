// Device-side stream addressing shared by every sampling kernel.
#pragma once
#include "glibc_math.cuh"
#include "glibc_tables.h"
#include "philox.cuh"

// Philox counter of block b of a uniform01 draw at stream counter (chi:clo).
// The reference fills 65536-double spans from a fresh numpy generator whose
// counter is (counter + span_start/4) mod 2^128 (RngStream._generator_at masks
// to two words, sampling.py:74-80); numpy pre-increments the 256-bit counter
// before each block.  For counters below 2^128 - 2^14 this is counter + b + 1.
__device__ __forceinline__ phx4 stream_block_counter(uint64_t clo, uint64_t chi, uint64_t b) {
  const uint64_t span_off = (b >> 14) << 14;  // blocks per span = 65536/4
  const uint64_t blo = clo + span_off;
  const uint64_t bhi = chi + (blo < clo ? 1ULL : 0ULL);  // mod 2^128
  return phx_block_counter(blo, bhi, b & 16383ULL);
}

__device__ __forceinline__ void load_sincostab(double* tab) {
  const double* src = reinterpret_cast<const double*>(simopt_sincostab_dev);
  for (int i = threadIdx.x; i < SIMOPT_SINCOSTAB_N; i += blockDim.x) tab[i] = src[i];
  __syncthreads();
}

// Normals 4b..4b+3 of standard_normal: Box-Muller on uniforms (4b,4b+1), (4b+2,4b+3).
__device__ __forceinline__ void normals4(uint64_t seed, uint64_t sid, uint64_t clo, uint64_t chi,
                                         uint64_t b, const double* tab, double z[4]) {
  const phx4 w = philox4x64_10(stream_block_counter(clo, chi, b), seed, sid);
  glibc_boxmuller_fast(phx_u01(w.v[0]), phx_u01(w.v[1]), tab, &z[0], &z[1]);
  glibc_boxmuller_fast(phx_u01(w.v[2]), phx_u01(w.v[3]), tab, &z[2], &z[3]);
}
