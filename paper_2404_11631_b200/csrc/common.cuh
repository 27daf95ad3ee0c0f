// Shared helpers for the sm_100a kernels of libsimopt_b200.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/simopt_b200.h"

// Streaming multiprocessors of the current device (queried once per device and
// cached; 148 on B200).  Grids of persistent and grid-stride kernels are sized
// from it.
int simopt_num_sms();
#define SIMOPT_NUM_SMS (simopt_num_sms())

// Thread-local last-error text (simopt_last_error()).
void simopt_set_error(const char* fmt, ...);

#define SIMOPT_CHECK_LAUNCH(name)                                                    \
  do {                                                                               \
    cudaError_t _e = cudaGetLastError();                                             \
    if (_e != cudaSuccess) {                                                         \
      simopt_set_error("%s: %s", name, cudaGetErrorString(_e));                      \
      return SIMOPT_E_CUDA;                                                          \
    }                                                                                \
  } while (0)

#define SIMOPT_CUDA(call)                                                            \
  do {                                                                               \
    cudaError_t _e = (call);                                                         \
    if (_e != cudaSuccess) {                                                         \
      simopt_set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(_e)); \
      return SIMOPT_E_CUDA;                                                          \
    }                                                                                \
  } while (0)

#define SIMOPT_REQUIRE(cond, code, ...)                                              \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      simopt_set_error(__VA_ARGS__);                                                 \
      return code;                                                                   \
    }                                                                                \
  } while (0)

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Per-(stream, host thread) scratch.  Every ABI call that needs scratch (chunk
// partials, argmin partials) takes it from its buffer: one thread's uses are
// stream-ordered, and two threads enqueueing on one stream get separate buffers, and no allocation happens on the hot path or
// inside a captured CUDA graph.  Buffers only grow; a superseded buffer is kept
// alive (graphs captured earlier may still reference it).  Returns nullptr and
// sets the error text on failure.
void* simopt_scratch(cudaStream_t st, size_t bytes);

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Pairwise fold of a[0..m) in index order, odd tail carried (_kernels.py:30-42),
// executed by one CTA, ping-ponging between shared buffers a and b (each >= m).
// Call with all threads of the block; returns the root.
__device__ __forceinline__ double block_fold_pairwise(double* a, double* b, int m) {
  __syncthreads();
  while (m > 1) {
    const int h = m >> 1;
    for (int i = threadIdx.x; i < h; i += blockDim.x) b[i] = a[2 * i] + a[2 * i + 1];
    if ((m & 1) && threadIdx.x == 0) b[h] = a[m - 1];
    __syncthreads();
    double* t = a; a = b; b = t;
    m = (m & 1) ? h + 1 : h;
  }
  const double r = (m == 0) ? 0.0 : a[0];
  __syncthreads();
  return r;
}

// Serial fold by a single thread (for small m held in registers/local arrays).
__device__ __forceinline__ double serial_fold_pairwise(double* p, int m) {
  if (m == 0) return 0.0;
  while (m > 1) {
    const int h = m >> 1;
    for (int i = 0; i < h; ++i) p[i] = p[2 * i] + p[2 * i + 1];
    if (m & 1) { p[h] = p[m - 1]; m = h + 1; } else { m = h; }
  }
  return p[0];
}
