// ABI bookkeeping: version + thread-local error text.
#include <stdarg.h>
#include <stdio.h>

#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.cuh"

static thread_local char g_err[512] = "";

void simopt_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" const char* simopt_last_error(void) { return g_err; }
extern "C" int simopt_abi_version(void) { return 4; }

int simopt_num_sms() {
  static std::mutex mu;
  static std::unordered_map<int, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  cache[dev] = n;
  return n;
}

namespace {
__global__ void k_stamp(int64_t* out) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = (int64_t)t;
}
}  // namespace

extern "C" int simopt_timestamp(void* stream, int64_t* out) {
  k_stamp<<<1, 1, 0, as_stream(stream)>>>(out);
  SIMOPT_CHECK_LAUNCH("k_stamp");
  return SIMOPT_OK;
}

namespace {
struct Scratch {
  void* ptr = nullptr;
  size_t bytes = 0;
};
struct ScratchKey {
  cudaStream_t stream;
  std::thread::id thread;
  bool operator==(const ScratchKey& o) const { return stream == o.stream && thread == o.thread; }
};
struct ScratchKeyHash {
  size_t operator()(const ScratchKey& k) const {
    return std::hash<void*>()(reinterpret_cast<void*>(k.stream)) ^
           (std::hash<std::thread::id>()(k.thread) * 0x9e3779b97f4a7c15ULL);
  }
};
std::mutex g_scratch_mu;
// keyed by (stream, host thread): a multi-kernel op (partials, then fold) enqueued by
// one thread must not share its buffer with another thread's op on the same stream
// (the reference's kernels are reentrant on disjoint data, backend.py:12-14)
std::unordered_map<ScratchKey, Scratch, ScratchKeyHash> g_scratch;
std::vector<void*> g_retired;  // superseded buffers, kept alive for captured graphs
}  // namespace

void* simopt_scratch(cudaStream_t st, size_t bytes) {
  std::lock_guard<std::mutex> lock(g_scratch_mu);
  Scratch& s = g_scratch[ScratchKey{st, std::this_thread::get_id()}];
  if (s.bytes >= bytes) return s.ptr;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
    simopt_set_error("scratch for this stream must be warmed up (an eager call of the same "
                     "sizes) before CUDA-graph capture: need %zu bytes, have %zu", bytes, s.bytes);
    return nullptr;
  }
  size_t want = bytes < (1u << 20) ? (1u << 20) : bytes;
  want = (want + 4095) & ~size_t(4095);
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, want);
  if (e != cudaSuccess) {
    simopt_set_error("scratch allocation of %zu bytes: %s", want, cudaGetErrorString(e));
    return nullptr;
  }
  if (s.ptr) g_retired.push_back(s.ptr);
  s.ptr = p;
  s.bytes = want;
  return p;
}
