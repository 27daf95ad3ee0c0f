// Philox4x64-10 (Random123; numpy.random.Philox), host+device.
//
// The reference's RngStream (sobench/sampling.py:51-80) keys numpy's Philox
// with key=(seed, stream_id) and a 256-bit counter whose two low words hold the
// stream's 128-bit block counter.  numpy pre-increments the counter before every
// block, so block b of a stream at counter c is Philox(ctr = c + b + 1, key)
// (carry propagating through all four words).  uniform01 (sampling.py:87-102)
// turns word w into (w >> 11) * 2^-53.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define PHX_HD __host__ __device__ __forceinline__
#else
#define PHX_HD static inline
#endif

#define PHILOX_M0 0xD2E7470EE14C6C93ULL
#define PHILOX_M1 0xCA5A826395121157ULL
#define PHILOX_W0 0x9E3779B97F4A7C15ULL
#define PHILOX_W1 0xBB67AE8584CAA73BULL

PHX_HD void phx_mulhilo(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
#if defined(__CUDA_ARCH__)
  *lo = a * b;
  *hi = __umul64hi(a, b);
#else
  const unsigned __int128 p = (unsigned __int128)a * b;
  *lo = (uint64_t)p;
  *hi = (uint64_t)(p >> 64);
#endif
}

typedef struct phx4 { uint64_t v[4]; } phx4;

PHX_HD phx4 philox4x64_10(phx4 c, uint64_t k0, uint64_t k1) {
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, lo0, hi1, lo1;
    phx_mulhilo(PHILOX_M0, c.v[0], &hi0, &lo0);
    phx_mulhilo(PHILOX_M1, c.v[2], &hi1, &lo1);
    phx4 o;
    o.v[0] = hi1 ^ c.v[1] ^ k0;
    o.v[1] = lo1;
    o.v[2] = hi0 ^ c.v[3] ^ k1;
    o.v[3] = lo0;
    c = o;
    k0 += PHILOX_W0;
    k1 += PHILOX_W1;
  }
  return c;
}

// Counter of block `b` (0-based) of a stream positioned at 128-bit counter
// (clo, chi): the 256-bit value (chi:clo) + b + 1.
PHX_HD phx4 phx_block_counter(uint64_t clo, uint64_t chi, uint64_t b) {
  phx4 c;
  const uint64_t add = b + 1;  // b < 2^62 in practice; +1 cannot wrap
  c.v[0] = clo + add;
  const uint64_t carry0 = (c.v[0] < clo) ? 1ULL : 0ULL;
  c.v[1] = chi + carry0;
  const uint64_t carry1 = (carry0 && c.v[1] == 0) ? 1ULL : 0ULL;
  c.v[2] = carry1;
  c.v[3] = 0;
  return c;
}

PHX_HD double phx_u01(uint64_t w) { return (double)(w >> 11) * (1.0 / 9007199254740992.0); }

// Round keys of Philox4x64-10 for key (k0, k1): rk[2r], rk[2r+1] = key after r bumps.
// Precomputed once on the host and passed by value, so every round's XOR takes
// its key straight from the constant bank (no per-round key arithmetic).
typedef struct phx_keys { uint64_t k[20]; } phx_keys;

static inline phx_keys phx_round_keys(uint64_t k0, uint64_t k1) {
  phx_keys r;
  for (int i = 0; i < 10; ++i) {
    r.k[2 * i] = k0;
    r.k[2 * i + 1] = k1;
    k0 += PHILOX_W0;
    k1 += PHILOX_W1;
  }
  return r;
}

PHX_HD phx4 philox4x64_10_rk(phx4 c, const phx_keys& rk) {
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, lo0, hi1, lo1;
    phx_mulhilo(PHILOX_M0, c.v[0], &hi0, &lo0);
    phx_mulhilo(PHILOX_M1, c.v[2], &hi1, &lo1);
    phx4 o;
    o.v[0] = hi1 ^ c.v[1] ^ rk.k[2 * r];
    o.v[1] = lo1;
    o.v[2] = hi0 ^ c.v[3] ^ rk.k[2 * r + 1];
    o.v[3] = lo0;
    c = o;
  }
  return c;
}

// Counter (c0, hi, 0, 0) with a launch-constant high word `hi`: the first two rounds
// carry known values (round 0 multiplies word 2 = 0; round 1 multiplies the constant
// hi ^ k0), so those two 64x64 products are skipped / precomputed on the host.
// Valid whenever the launch's counters c0 = clo + b + 1 do not carry into word 1
// (phx_no_carry).  Bit-identical to philox4x64_10_rk on such counters.
typedef struct phx_pre {
  uint64_t a;       // hi ^ k0 (word 0 after round 0)
  uint64_t h1, l1;  // mulhilo(M0, a): round 1's first product
} phx_pre;

static inline phx_pre phx_precompute(uint64_t hi, const phx_keys& rk) {
  phx_pre p;
  p.a = hi ^ rk.k[0];
#if defined(__CUDA_ARCH__)
  p.l1 = PHILOX_M0 * p.a;
  p.h1 = __umul64hi(PHILOX_M0, p.a);
#else
  const unsigned __int128 q = (unsigned __int128)PHILOX_M0 * p.a;
  p.l1 = (uint64_t)q;
  p.h1 = (uint64_t)(q >> 64);
#endif
  return p;
}

// True when clo + 1 .. clo + nblocks stays below 2^64 (no carry into word 1).
static inline bool phx_no_carry(uint64_t clo, uint64_t nblocks) {
  return nblocks <= ~clo;
}

// Rounds 1-9 of the counter (c0, hi, 0, 0) given round 0's product (hi0, lo0) = M0 * c0
// (word 2 == 0, so round 0 has no second product).  Split out so a caller walking
// counters c0, c0 + s, c0 + 2s, ... can carry M0 * c0 forward by a 128-bit add
// (phx_r0_advance) instead of a product.
PHX_HD phx4 philox4x64_10_rk_r0(uint64_t hi0, uint64_t lo0, const phx_keys& rk, const phx_pre& pre) {
  uint64_t hi1, lo1;
  phx4 c;                                          // round 1
  phx_mulhilo(PHILOX_M1, hi0 ^ rk.k[1], &hi1, &lo1);
  c.v[0] = hi1 ^ rk.k[2];
  c.v[1] = lo1;
  c.v[2] = pre.h1 ^ lo0 ^ rk.k[3];
  c.v[3] = pre.l1;
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int r = 2; r < 10; ++r) {
    phx_mulhilo(PHILOX_M0, c.v[0], &hi0, &lo0);
    phx_mulhilo(PHILOX_M1, c.v[2], &hi1, &lo1);
    phx4 o;
    o.v[0] = hi1 ^ c.v[1] ^ rk.k[2 * r];
    o.v[1] = lo1;
    o.v[2] = hi0 ^ c.v[3] ^ rk.k[2 * r + 1];
    o.v[3] = lo0;
    c = o;
  }
  return c;
}

PHX_HD phx4 philox4x64_10_rk_c0(uint64_t c0, const phx_keys& rk, const phx_pre& pre) {
  uint64_t hi0, lo0;
  phx_mulhilo(PHILOX_M0, c0, &hi0, &lo0);          // round 0
  return philox4x64_10_rk_r0(hi0, lo0, rk, pre);
}

#if defined(__CUDACC__)
// (hi0, lo0) <- M0 * (c0 + S) from M0 * c0, for a compile-time stride S: a 128-bit
// add of the constant M0 * S (exact mod 2^128, so equal to the product whenever
// c0 + S < 2^64, which phx_no_carry guarantees for the launch).
template <uint64_t S>
__device__ __forceinline__ void phx_r0_advance(uint64_t& hi0, uint64_t& lo0) {
  constexpr uint64_t kLo = PHILOX_M0 * S;
  constexpr uint64_t kHi = (uint64_t)(((unsigned __int128)PHILOX_M0 * S) >> 64);
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo0), "+l"(hi0) : "n"(kLo), "n"(kHi));
}
#endif
