// ABI bookkeeping: version + thread-local error text.
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"

static thread_local char g_err[512] = "";

void simopt_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" const char* simopt_last_error(void) { return g_err; }
extern "C" int simopt_abi_version(void) { return 1; }

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
