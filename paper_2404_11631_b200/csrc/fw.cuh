// Deterministic first-argmin used by the LMOs (np.argmin semantics: the first
// index among equal minima; lmo.py:62, :85).
#pragma once
#include <stdint.h>

struct ArgMin {
  double v;
  int64_t i;
};

__device__ __forceinline__ ArgMin amin(ArgMin a, ArgMin b) {
  if (b.v < a.v) return b;
  if (a.v < b.v) return a;
  return (b.i < a.i) ? b : a;
}

__device__ __forceinline__ ArgMin warp_amin(ArgMin b) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMin t{__shfl_xor_sync(0xffffffffu, b.v, o),
             (int64_t)__shfl_xor_sync(0xffffffffu, (long long)b.i, o)};
    b = amin(b, t);
  }
  return b;
}
