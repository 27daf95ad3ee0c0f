/* CPU oracle for the multi-PRNG kernels (csrc/prng.cu) -- TEST INFRASTRUCTURE ONLY.
 *
 * The reference ships three orphaned fixture files
 * (pkg/test_multi_prng_{philox4x32,sfc64,xoshiro256pp}.json) that no source or
 * test consumes and that could not be reproduced: parity
 * with them is UNPINNED.  The generators are restated here from their published
 * definitions and pinned instead to
 *   Philox4x32-10  -- Random123 (Salmon et al., SC'11) known-answer vectors
 *                     (tests/test_oracle.py) and cuRAND's curand_Philox4x32_10
 *                     (tests/test_gpu_prng.py);
 *   SFC64          -- numpy.random.SFC64.random_raw (live, given the state);
 *   xoshiro256++   -- Blackman & Vigna's reference (xoshiro256plusplus.c):
 *                     next() and jump(); known first outputs from state {1,2,3,4}.
 */
#include <stdint.h>

static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* Philox4x32-10: out[4b + k] = word k of Philox(ctr + b, key), 128-bit counter. */
void orc_philox4x32(const uint32_t ctr[4], const uint32_t key[2], int64_t nblocks, uint32_t* out) {
  uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
  for (int64_t b = 0; b < nblocks; ++b) {
    uint32_t x0 = c[0], x1 = c[1], x2 = c[2], x3 = c[3], k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
      const uint64_t p0 = (uint64_t)0xD2511F53u * x0, p1 = (uint64_t)0xCD9E8D57u * x2;
      const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
      const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
      x0 = hi1 ^ x1 ^ k0; x1 = lo1; x2 = hi0 ^ x3 ^ k1; x3 = lo0;
      k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    out[4 * b] = x0; out[4 * b + 1] = x1; out[4 * b + 2] = x2; out[4 * b + 3] = x3;
    if (++c[0] == 0 && ++c[1] == 0 && ++c[2] == 0) ++c[3];
  }
}

/* SFC64 (Doty-Humphrey; numpy _sfc64.h): state = {a, b, c, counter}. */
void orc_sfc64(uint64_t s[4], int64_t n, uint64_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t tmp = s[0] + s[1] + s[3]++;
    s[0] = s[1] ^ (s[1] >> 11);
    s[1] = s[2] + (s[2] << 3);
    s[2] = rotl64(s[2], 24) + tmp;
    out[i] = tmp;
  }
}

/* xoshiro256++ 1.0 (Blackman & Vigna). */
void orc_xoshiro256pp(uint64_t s[4], int64_t n, uint64_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    out[i] = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
  }
}

/* jump(): advances by 2^128 steps (non-overlapping subsequences for parallel streams). */
void orc_xoshiro256pp_jump(uint64_t s[4]) {
  static const uint64_t J[4] = {0x180ec6d33cfd0abaULL, 0xd5a61266f0c9392cULL,
                                0xa9582618e03fc9aaULL, 0x39abdc4529b1661cULL};
  uint64_t t[4] = {0, 0, 0, 0}, dummy;
  for (int i = 0; i < 4; ++i)
    for (int b = 0; b < 64; ++b) {
      if (J[i] & (1ULL << b)) { t[0] ^= s[0]; t[1] ^= s[1]; t[2] ^= s[2]; t[3] ^= s[3]; }
      orc_xoshiro256pp(s, 1, &dummy);
    }
  s[0] = t[0]; s[1] = t[1]; s[2] = t[2]; s[3] = t[3];
}
