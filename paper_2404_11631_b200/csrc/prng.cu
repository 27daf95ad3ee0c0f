// Per-stream generators for the multi-PRNG tests (BASELINE.json north star: Philox4x32,
// SFC64, Xoshiro256++ "provided as per-stream kernels").  The reference's own draws
// use numpy Philox4x64-10 (rng.cu); these three back the reference's orphaned
// pkg/test_multi_prng_*.json fixtures, whose generating code is absent,
// so they follow the published algorithms (oracle/prng.c restates them):
//   Philox4x32-10  counter-based: one thread per block of 4 words, coalesced stores;
//   SFC64, xoshiro256++  one thread per stream holding the 256-bit state in
//                  registers; a warp generates 32 outputs per lane into a shared tile
//                  and writes each stream's row with 256-byte coalesced stores
//                  (out is stream-major [n_streams][n]); the advanced state is
//                  written back so successive calls continue each stream.
// out_kind 0 = raw 64-bit words, 1 = doubles (w >> 11) * 2^-53 (numpy's next_double).
#include "common.cuh"

namespace {

__device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

__global__ void __launch_bounds__(256) k_philox4x32(uint32_t k0, uint32_t k1, uint32_t c0,
                                                    uint32_t c1, uint32_t c2, uint32_t c3,
                                                    int64_t nblocks, uint32_t* __restrict__ out) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nblocks;
       b += (int64_t)gridDim.x * blockDim.x) {
    // 128-bit counter + b
    const uint64_t lo = ((uint64_t)c1 << 32 | c0), add = (uint64_t)b;
    const uint64_t nlo = lo + add;
    const uint64_t hi = ((uint64_t)c3 << 32 | c2) + (nlo < lo ? 1ULL : 0ULL);
    uint32_t x0 = (uint32_t)nlo, x1 = (uint32_t)(nlo >> 32), x2 = (uint32_t)hi, x3 = (uint32_t)(hi >> 32);
    uint32_t a0 = k0, a1 = k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const uint32_t hi0 = __umulhi(0xD2511F53u, x0), lo0 = 0xD2511F53u * x0;
      const uint32_t hi1 = __umulhi(0xCD9E8D57u, x2), lo1 = 0xCD9E8D57u * x2;
      const uint32_t n0 = hi1 ^ x1 ^ a0, n2 = hi0 ^ x3 ^ a1;
      x0 = n0; x1 = lo1; x2 = n2; x3 = lo0;
      a0 += 0x9E3779B9u;
      a1 += 0xBB67AE85u;
    }
    reinterpret_cast<uint4*>(out)[b] = make_uint4(x0, x1, x2, x3);
  }
}

struct Sfc64 {
  uint64_t a, b, c, w;
  __device__ __forceinline__ uint64_t next() {
    const uint64_t tmp = a + b + w++;
    a = b ^ (b >> 11);
    b = c + (c << 3);
    c = rotl64(c, 24) + tmp;
    return tmp;
  }
};

struct Xoshiro256pp {
  uint64_t a, b, c, w;  // s[0..3]
  __device__ __forceinline__ uint64_t next() {
    const uint64_t r = rotl64(a + w, 23) + a;
    const uint64_t t = b << 17;
    c ^= a;
    w ^= b;
    b ^= c;
    a ^= w;
    c ^= t;
    w = rotl64(w, 45);
    return r;
  }
};

template <class G>
__global__ void __launch_bounds__(128) k_streams(uint64_t* __restrict__ state, int64_t nstreams,
                                                 int64_t n, int out_kind, void* __restrict__ out) {
  __shared__ uint64_t tile[4][32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t s0 = (blockIdx.x * 4LL + warp) * 32;  // this warp's 32 streams
  if (s0 >= nstreams) return;
  const int64_t s = s0 + lane;
  const bool live = s < nstreams;
  G g{0, 0, 0, 0};
  if (live) {
    const uint4* st = reinterpret_cast<const uint4*>(state + 4 * s);
    const uint4 p = st[0], q = st[1];
    g.a = (uint64_t)p.y << 32 | p.x;
    g.b = (uint64_t)p.w << 32 | p.z;
    g.c = (uint64_t)q.y << 32 | q.x;
    g.w = (uint64_t)q.w << 32 | q.z;
  }
  const int rows = (int)(nstreams - s0 < 32 ? nstreams - s0 : 32);
  for (int64_t i0 = 0; i0 < n; i0 += 32) {
    const int cnt = (int)(n - i0 < 32 ? n - i0 : 32);
    for (int k = 0; k < cnt; ++k) tile[warp][lane][k] = g.next();
    __syncwarp();
    for (int r = 0; r < rows; ++r) {
      if (lane < cnt) {
        const uint64_t v = tile[warp][r][lane];
        const int64_t o = (s0 + r) * n + i0 + lane;
        if (out_kind == 0)
          static_cast<uint64_t*>(out)[o] = v;
        else
          static_cast<double*>(out)[o] = (double)(v >> 11) * (1.0 / 9007199254740992.0);
      }
    }
    __syncwarp();
  }
  if (live) {
    uint64_t* st = state + 4 * s;
    st[0] = g.a;
    st[1] = g.b;
    st[2] = g.c;
    st[3] = g.w;
  }
}

void xoshiro_step(uint64_t s[4]) {
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = (s[3] << 45) | (s[3] >> 19);
}

}  // namespace

extern "C" int simopt_philox4x32(void* stream, uint32_t key0, uint32_t key1, const uint32_t* ctr,
                                 int64_t nblocks, uint32_t* out) {
  SIMOPT_REQUIRE(nblocks >= 0, SIMOPT_E_CONFIG, "negative block count");
  SIMOPT_REQUIRE((reinterpret_cast<uintptr_t>(out) & 15) == 0, SIMOPT_E_CONFIG,
                 "philox4x32 output must be 16-byte aligned");
  if (nblocks == 0) return SIMOPT_OK;
  const int64_t want = ceil_div(nblocks, 256), cap = (int64_t)SIMOPT_NUM_SMS * 16;
  k_philox4x32<<<(int)(want < cap ? want : cap), 256, 0, as_stream(stream)>>>(
      key0, key1, ctr[0], ctr[1], ctr[2], ctr[3], nblocks, out);
  SIMOPT_CHECK_LAUNCH("k_philox4x32");
  return SIMOPT_OK;
}

static int launch_streams(int which, void* stream, uint64_t* state, int64_t nstreams, int64_t n,
                          int out_kind, void* out) {
  SIMOPT_REQUIRE(nstreams >= 0 && n >= 0, SIMOPT_E_CONFIG, "negative extent");
  SIMOPT_REQUIRE(out_kind == 0 || out_kind == 1, SIMOPT_E_CONFIG, "out_kind must be 0 or 1");
  SIMOPT_REQUIRE((reinterpret_cast<uintptr_t>(state) & 15) == 0, SIMOPT_E_CONFIG,
                 "state must be 16-byte aligned");
  if (nstreams == 0 || n == 0) return SIMOPT_OK;
  const int grid = (int)ceil_div(nstreams, 128);
  if (which == 0)
    k_streams<Sfc64><<<grid, 128, 0, as_stream(stream)>>>(state, nstreams, n, out_kind, out);
  else
    k_streams<Xoshiro256pp><<<grid, 128, 0, as_stream(stream)>>>(state, nstreams, n, out_kind, out);
  SIMOPT_CHECK_LAUNCH("k_streams");
  return SIMOPT_OK;
}

extern "C" int simopt_sfc64(void* stream, uint64_t* state, int64_t nstreams, int64_t n,
                            int out_kind, void* out) {
  return launch_streams(0, stream, state, nstreams, n, out_kind, out);
}

extern "C" int simopt_xoshiro256pp(void* stream, uint64_t* state, int64_t nstreams, int64_t n,
                                   int out_kind, void* out) {
  return launch_streams(1, stream, state, nstreams, n, out_kind, out);
}

// Host: nstreams states for parallel streams, state[k] = jump^k(seed_state) (each jump
// advances 2^128 steps: non-overlapping subsequences).
extern "C" int simopt_xoshiro256pp_streams(const uint64_t* seed_state, int64_t nstreams,
                                           uint64_t* states) {
  static const uint64_t J[4] = {0x180ec6d33cfd0abaULL, 0xd5a61266f0c9392cULL,
                                0xa9582618e03fc9aaULL, 0x39abdc4529b1661cULL};
  SIMOPT_REQUIRE(nstreams >= 0, SIMOPT_E_CONFIG, "negative stream count");
  uint64_t s[4] = {seed_state[0], seed_state[1], seed_state[2], seed_state[3]};
  SIMOPT_REQUIRE(s[0] | s[1] | s[2] | s[3], SIMOPT_E_CONFIG, "xoshiro256++ state must be nonzero");
  for (int64_t k = 0; k < nstreams; ++k) {
    for (int i = 0; i < 4; ++i) states[4 * k + i] = s[i];
    uint64_t t[4] = {0, 0, 0, 0};
    for (int i = 0; i < 4; ++i)
      for (int b = 0; b < 64; ++b) {
        if (J[i] & (1ULL << b))
          for (int q = 0; q < 4; ++q) t[q] ^= s[q];
        xoshiro_step(s);
      }
    for (int q = 0; q < 4; ++q) s[q] = t[q];
  }
  return SIMOPT_OK;
}
