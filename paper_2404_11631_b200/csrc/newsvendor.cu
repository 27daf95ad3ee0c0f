// Multi-product newsvendor on sm_100a: fused demand resample + ECDF-count gradient,
// single-budget LMO and Frank-Wolfe update (reference: sobench/tasks.py:141-188,
// sampling.py:173-193, lmo.py:68-89, frank_wolfe.py:62-82, _kernels.py:210-259).
//
// Epoch layout (keyed ECDF, see newsvendor.cuh):
//   keys  [d][S] u32   row j = product j's S draws in segments of NV_SEG = 4096;
//                      key = q << 12 | local, counting-sorted by bucket (q >> 10).
//   off   [d][nseg][NV_B] u16   start of each bucket inside its segment.
// The reference sorts every row (sampling.py:192) and binary-searches it
// (_kernels.py:245-259).  Here the resample evaluates only an fp32 approximation
// per draw (plus the exact Philox stream), and a gradient query resolves the
// handful of draws whose approximation is within the guaranteed error of the
// threshold with the exact glibc Box-Muller -- the count is the reference's
// integer, bit for bit, for every query.
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "common.cuh"
#include "fw.cuh"
#include "glibc_math.cuh"
#include "glibc_tables.h"
#include "newsvendor.cuh"
#include "philox.cuh"
#include "reduce_device.cuh"
#include "rng_device.cuh"

namespace {

constexpr int kResampleThreads = 256;
constexpr int kResampleMinBlocks = 6;  // = the shared-memory limit (6 x 36.9 KB); 32 registers

// Persistent CTAs walk (product j, segment s) pairs: generate the segment's keys
// (Philox4x64-10 + fp32 Box-Muller approximation), histogram them by bucket in
// shared memory, scan, scatter into bucket order and stream keys + bucket starts out.
template <bool kNoCarry>
__global__ void __launch_bounds__(kResampleThreads, kResampleMinBlocks)
    k_nv_resample(const phx_keys rk, const phx_pre pre, uint64_t clo, uint64_t chi, int64_t d,
                  int64_t S, int nseg, uint32_t* __restrict__ keys, uint16_t* __restrict__ off) {
  __shared__ __align__(16) uint32_t raw[NV_SEG];
  __shared__ __align__(16) uint32_t sorted_[NV_SEG];
  __shared__ int hist[NV_B];
  __shared__ int wsum[kResampleThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nblk = d * nseg;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int64_t j = blk / nseg;
    const int s = (int)(blk - j * nseg);
    const int64_t e0 = (int64_t)s * NV_SEG;
    const int len = (int)((S - e0) < NV_SEG ? (S - e0) : NV_SEG);
    for (int i = threadIdx.x; i < NV_B; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    // 1) keys for normals i0 .. i0+len-1 of the epoch's standard_normal(d*S) draw
    const int64_t i0 = j * S + e0;
    const int64_t q0 = i0 >> 2, q1 = (i0 + len - 1) >> 2;
    const bool aligned = ((i0 & 3) == 0) && ((len & 3) == 0);
    const int nq = (int)(q1 - q0);             // <= NV_SEG / 4: 32-bit loop arithmetic
    const uint64_t c0 = clo + (uint64_t)q0 + 1;
    const int lbase = (int)((q0 << 2) - i0);   // local index of block q0's first normal
    for (int t = threadIdx.x; t <= nq; t += kResampleThreads) {
      const int64_t q = q0 + t;
      // kNoCarry: no carry into the counter's word 1 within this launch (checked on the
      // host), so block q's counter is (clo + q + 1, chi, 0, 0) -- see stream_block_counter
      const phx4 w = kNoCarry ? philox4x64_10_rk_c0(c0 + (uint64_t)t, rk, pre)
                              : philox4x64_10_rk(stream_block_counter(clo, chi, (uint64_t)q), rk);
      float z[4];
      nv_approx_pair(w.v[0], w.v[1], &z[0], &z[1]);
      nv_approx_pair(w.v[2], w.v[3], &z[2], &z[3]);
      const int l0 = lbase + (t << 2);
      if (aligned) {
        uint32_t kk[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          kk[k] = nv_key(z[k], (uint32_t)(l0 + k));
          atomicAdd(&hist[kk[k] >> (12 + NV_QBITS - 10)], 1);
        }
        reinterpret_cast<uint4*>(raw)[l0 >> 2] = make_uint4(kk[0], kk[1], kk[2], kk[3]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int l = l0 + k;
          if (l >= 0 && l < len) {
            const uint32_t key = nv_key(z[k], (uint32_t)l);
            raw[l] = key;
            atomicAdd(&hist[key >> (12 + NV_QBITS - 10)], 1);
          }
        }
      }
    }
    __syncthreads();
    // 2) exclusive scan of the histogram (NV_B entries, kPer per thread)
    {
      constexpr int kPer = NV_B / kResampleThreads;
      static_assert(kPer == 4, "bucket starts are stored as one u64 per thread");
      int v[kPer];
      int run = 0;
#pragma unroll
      for (int k = 0; k < kPer; ++k) { v[k] = hist[threadIdx.x * kPer + k]; run += v[k]; }
      int incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) wsum[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        int w = lane < kResampleThreads / 32 ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, w, o);
          if (lane >= o) w += t;
        }
        if (lane < kResampleThreads / 32) wsum[lane] = w;  // inclusive warp prefix
      }
      __syncthreads();
      int base = incl - run + (warp > 0 ? wsum[warp - 1] : 0);
      uint64_t packed = 0;
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        packed |= (uint64_t)(uint16_t)base << (16 * k);
        hist[threadIdx.x * kPer + k] = base;  // becomes the scatter cursor
        base += v[k];
      }
      reinterpret_cast<uint64_t*>(off + (j * nseg + s) * (int64_t)NV_B)[threadIdx.x] = packed;
    }
    __syncthreads();
    // 3) scatter into bucket order (order inside a bucket is irrelevant to every count)
    constexpr int kBucketShift = 12 + NV_QBITS - 10;
    if (aligned) {  // four keys per 16-byte shared load
      for (int l4 = threadIdx.x; l4 < (len >> 2); l4 += kResampleThreads) {
        const uint4 k4 = reinterpret_cast<const uint4*>(raw)[l4];
        sorted_[atomicAdd(&hist[k4.x >> kBucketShift], 1)] = k4.x;
        sorted_[atomicAdd(&hist[k4.y >> kBucketShift], 1)] = k4.y;
        sorted_[atomicAdd(&hist[k4.z >> kBucketShift], 1)] = k4.z;
        sorted_[atomicAdd(&hist[k4.w >> kBucketShift], 1)] = k4.w;
      }
    } else {
      for (int l = threadIdx.x; l < len; l += kResampleThreads) {
        const uint32_t key = raw[l];
        sorted_[atomicAdd(&hist[key >> kBucketShift], 1)] = key;
      }
    }
    __syncthreads();
    uint32_t* dst = keys + j * S + e0;
    if (aligned) {  // 16-byte stores (row offset j*S + e0 is a multiple of 4 here)
      for (int l4 = threadIdx.x; l4 < (len >> 2); l4 += blockDim.x)
        reinterpret_cast<uint4*>(dst)[l4] = reinterpret_cast<const uint4*>(sorted_)[l4];
    } else {
      for (int l = threadIdx.x; l < len; l += blockDim.x) dst[l] = sorted_[l];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Warp-specialised resample.  Generation is bound by the heavy FMA pipe (the Philox
// 64x64->128 products); the scan, scatter and store use the ALU and LSU.  Eight producer
// warps only generate: segment k's keys into raw[k&1] and its bucket counts into
// hist[k&1]; four consumer warps scan, scatter into bucket order and store.  The two
// roles meet at named barriers (full[slot]: producers arrive, consumers wait; empty[slot]:
// consumers arrive once they have read raw[slot] and re-zeroed hist[slot], producers
// wait), so producer warps never stop at a CTA-wide barrier and the heavy pipe keeps a
// steady supply of multiplies while the consumers' memory work runs beside it.
// Measured at C2 (tools/nv_resample_ab.py): 8 producer + 4 consumer warps, 3 CTAs per SM
// (48 registers) 3.76 ms; 12 + 4 warps 3.88; 16 + 4 at 2 CTAs per SM 3.97; consumers also
// counting the buckets 3.88; the single-role k_nv_resample 4.12; a software-pipelined
// variant (generate i || scatter i-1 in one phase) 4.38-4.62.
constexpr int kWsProd = 256, kWsCons = 128, kWsPerSm = 3;
// ring depth of raw segments between producers and consumers; named barriers 1..S (full),
// S+1..2S (empty), 2S+1 (consumers only)
#ifndef NV_WS_SLOTS
#define NV_WS_SLOTS 2
#endif
constexpr int kWsSlots = NV_WS_SLOTS, kWsConsBar = 2 * kWsSlots + 1;

struct WsSmem {
  uint32_t raw[kWsSlots][NV_SEG];
  uint32_t sorted[NV_SEG];
  int hist[kWsSlots][NV_B];
  int wsum[kWsCons / 32];
};  // 56 KB: up to three CTAs per SM
static_assert(sizeof(int) * NV_B == 4096, "ws_counter: hist[p] at +4 KB * p");

// The bucket counter of key k in hist[p]: hist[0] and hist[1] are adjacent 4 KB arrays, so
// the byte offset is ((k >> 20) & 0xffc) | (p << 12) -- one LOP3 after the shift, and the
// struct offset becomes the shared-memory instruction's immediate (no IMAD.IADD per key on
// the heavy pipe, which the Philox products saturate).
__device__ __forceinline__ int* ws_counter(unsigned char* smem, uint32_t k, uint32_t pbase);

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

#ifndef NV_WS_STREAM_STORES
#define NV_WS_STREAM_STORES 1
#endif
__device__ __forceinline__ void ws_store(uint4* p, uint4 v) {
  if (NV_WS_STREAM_STORES) __stcs(p, v);
  else *p = v;
}

__device__ __forceinline__ int* ws_counter(unsigned char* smem, uint32_t k, uint32_t pbase) {
  constexpr int kBucketByteShift = 12 + NV_QBITS - 10 - 2;  // bucket index * 4 bytes
  return reinterpret_cast<int*>(smem + offsetof(WsSmem, hist) +
                                (((k >> kBucketByteShift) & 0xffcu) | pbase));
}

// kRegCap: launch-bound blocks per SM used only to cap registers (3: 48 registers;
// 4: 40 registers, leaving room on the SM for the step kernel that runs beside it)
template <bool kNoCarry, int kRegCap>
__global__ void __launch_bounds__(kWsProd + kWsCons, kRegCap)
    k_nv_resample_ws(const phx_keys rk, const phx_pre pre, uint64_t clo, uint64_t chi, int64_t d,
                     int64_t S, int nseg, uint32_t* __restrict__ keys, uint16_t* __restrict__ off) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WsSmem& sm = *reinterpret_cast<WsSmem*>(smem_raw);
  constexpr int kBucketShift = 12 + NV_QBITS - 10;
  constexpr int kWsThreads = kWsProd + kWsCons;
  const int tid = threadIdx.x;
  const int64_t nblk = d * nseg;
  for (int i = tid; i < kWsSlots * NV_B; i += kWsThreads) (&sm.hist[0][0])[i] = 0;
  __syncthreads();
  const int64_t gq = gridDim.x / nseg;
  const int gr = (int)(gridDim.x - gq * nseg);
  int64_t j = blockIdx.x / nseg;
  int s = (int)(blockIdx.x - j * nseg);
  if (tid < kWsProd) {
    // ---- producers: Philox4x64-10 + fp32 key + bucket count, segment after segment
    for (int64_t blk = blockIdx.x, k = 0; blk < nblk; blk += gridDim.x, ++k) {
      const int p = (int)(k % kWsSlots);
      if (k >= kWsSlots) named_sync(1 + kWsSlots + p, kWsThreads);  // consumers are done with slot p
      const int64_t e0 = (int64_t)s * NV_SEG;
      const int len = (int)((S - e0) < NV_SEG ? (S - e0) : NV_SEG);
      const int64_t i0 = j * S + e0;
      const bool aligned = ((i0 & 3) == 0) && ((len & 3) == 0);
      const int64_t q0 = i0 >> 2, q1 = (i0 + len - 1) >> 2;
      const int nq = (int)(q1 - q0);
      const uint64_t c0 = clo + (uint64_t)q0 + 1;
      const int lbase = (int)((q0 << 2) - i0);
      uint32_t* raw = sm.raw[p];
      int* hist = sm.hist[p];
      const uint32_t pbase = (uint32_t)p << 12;
      // kNoCarry: round 0's product M0 * (c0 + t) is carried from t to t + kWsProd by a
      // 128-bit add (phx_r0_advance): 17 products per block instead of 18
      uint64_t r0h = 0, r0l = 0;
      if (kNoCarry) phx_mulhilo(PHILOX_M0, c0 + (uint64_t)tid, &r0h, &r0l);
      for (int t = tid; t <= nq; t += kWsProd) {
        phx4 w;
        if (kNoCarry) {
          w = philox4x64_10_rk_r0(r0h, r0l, rk, pre);
          phx_r0_advance<kWsProd>(r0h, r0l);
        } else {
          w = philox4x64_10_rk(stream_block_counter(clo, chi, (uint64_t)(q0 + t)), rk);
        }
        float z[4];
        nv_approx_pair(w.v[0], w.v[1], &z[0], &z[1]);
        nv_approx_pair(w.v[2], w.v[3], &z[2], &z[3]);
        const int l0 = lbase + (t << 2);
        if (aligned) {
          uint32_t kk[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            kk[u] = nv_key(z[u], (uint32_t)(l0 + u));
            atomicAdd(ws_counter(smem_raw, kk[u], pbase), 1);
          }
          reinterpret_cast<uint4*>(raw)[l0 >> 2] = make_uint4(kk[0], kk[1], kk[2], kk[3]);
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int l = l0 + u;
            if (l >= 0 && l < len) {
              const uint32_t key = nv_key(z[u], (uint32_t)l);
              raw[l] = key;
              atomicAdd(&hist[key >> kBucketShift], 1);
            }
          }
        }
      }
      named_arrive(1 + p, kWsThreads);  // slot p holds segment blk
      j += gq;
      s += gr;
      if (s >= nseg) {
        s -= nseg;
        ++j;
      }
    }
    return;
  }
  // ---- consumers: scan, scatter into bucket order, store
  const int ct = tid - kWsProd, lane = ct & 31, cw = ct >> 5;
  constexpr int kPer = NV_B / kWsCons;  // 8 buckets per thread
  for (int64_t blk = blockIdx.x, k = 0; blk < nblk; blk += gridDim.x, ++k) {
    const int p = (int)(k % kWsSlots);
    const int64_t e0 = (int64_t)s * NV_SEG;
    const int len = (int)((S - e0) < NV_SEG ? (S - e0) : NV_SEG);
    const bool aligned = (((j * S + e0) & 3) == 0) && ((len & 3) == 0);
    named_sync(1 + p, kWsThreads);  // segment blk is in slot p
    int* hist = sm.hist[p];
    const uint32_t* raw = sm.raw[p];
    int v[kPer];
    {
      const int4 a = reinterpret_cast<const int4*>(hist)[2 * ct];
      const int4 b = reinterpret_cast<const int4*>(hist)[2 * ct + 1];
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
    int run = 0;
#pragma unroll
    for (int u = 0; u < kPer; ++u) run += v[u];
    int incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) sm.wsum[cw] = incl;
    named_sync(kWsConsBar, kWsCons);
    int wpre = lane < cw ? sm.wsum[lane] : 0;
#pragma unroll
    for (int o = 2; o; o >>= 1) wpre += __shfl_xor_sync(0xffffffffu, wpre, o);  // lanes < 4
    int base = incl - run + __shfl_sync(0xffffffffu, wpre, 0);
    int st[kPer];
    uint32_t pk[kPer / 2];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      st[u] = base;
      base += v[u];
    }
#pragma unroll
    for (int u = 0; u < kPer / 2; ++u) pk[u] = (uint32_t)st[2 * u] | ((uint32_t)st[2 * u + 1] << 16);
    reinterpret_cast<int4*>(hist)[2 * ct] = make_int4(st[0], st[1], st[2], st[3]);
    reinterpret_cast<int4*>(hist)[2 * ct + 1] = make_int4(st[4], st[5], st[6], st[7]);
    // streaming stores (evict-first): the layout is read an epoch later, and the previous
    // epoch's FW steps, running beside this resample, keep their windows in L2
    ws_store(reinterpret_cast<uint4*>(off + (j * nseg + s) * (int64_t)NV_B) + ct,
             make_uint4(pk[0], pk[1], pk[2], pk[3]));
    named_sync(kWsConsBar, kWsCons);  // cursors complete
    if (aligned) {
      const uint32_t pbase = (uint32_t)p << 12;
      for (int l4 = ct; l4 < (len >> 2); l4 += kWsCons) {
        const uint4 k4 = reinterpret_cast<const uint4*>(raw)[l4];
        sm.sorted[atomicAdd(ws_counter(smem_raw, k4.x, pbase), 1)] = k4.x;
        sm.sorted[atomicAdd(ws_counter(smem_raw, k4.y, pbase), 1)] = k4.y;
        sm.sorted[atomicAdd(ws_counter(smem_raw, k4.z, pbase), 1)] = k4.z;
        sm.sorted[atomicAdd(ws_counter(smem_raw, k4.w, pbase), 1)] = k4.w;
      }
    } else {
      for (int l = ct; l < len; l += kWsCons) {
        const uint32_t key = raw[l];
        sm.sorted[atomicAdd(&hist[key >> kBucketShift], 1)] = key;
      }
    }
    named_sync(kWsConsBar, kWsCons);  // scatter complete: raw[p] read, cursors final, sorted full
    reinterpret_cast<int4*>(hist)[2 * ct] = make_int4(0, 0, 0, 0);
    reinterpret_cast<int4*>(hist)[2 * ct + 1] = make_int4(0, 0, 0, 0);
    named_arrive(1 + kWsSlots + p, kWsThreads);  // slot p free for the producers
    uint32_t* dst = keys + j * S + e0;
    if (aligned) {  // pointer walk: one 64-bit add per 16-byte store, no per-store IMAD.WIDE
      uint4* dp = reinterpret_cast<uint4*>(dst) + ct;
      const uint4* sp = reinterpret_cast<const uint4*>(sm.sorted) + ct;
      const uint4* se = reinterpret_cast<const uint4*>(sm.sorted) + (len >> 2);
#pragma unroll 4
      for (; sp < se; sp += kWsCons, dp += kWsCons) ws_store(dp, *sp);
    } else {
      for (int l = ct; l < len; l += kWsCons) dst[l] = sm.sorted[l];
    }
    named_sync(kWsConsBar, kWsCons);  // sorted stored: the next scatter may overwrite it
    j += gq;
    s += gr;
    if (s >= nseg) {
      s -= nseg;
      ++j;
    }
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// ECDF count #{D[j,:] <= x} for one product, one warp: lanes take segments.
struct NvStreamPos {
  uint64_t seed, sid, clo, chi;
};

// Exact resolve of one ambiguous draw, kept out of line so the rare glibc
// Box-Muller path does not inflate the register budget of the scan.
__device__ __noinline__ int nv_resolve(NvStreamPos sp, int64_t i, double mu, double sigma,
                                       double x) {
  const double* tab = reinterpret_cast<const double*>(simopt_sincostab_dev);
  const double z = nv_exact_z(sp.seed, sp.sid, sp.clo, sp.chi, i, tab);
  const double dv = mu + sigma * z;  // sampling.py:191
  return (dv <= x) ? 1 : 0;
}

#ifndef NV_KEY_BATCH
#define NV_KEY_BATCH 8
#endif
constexpr int kBatch = NV_KEY_BATCH;  // window keys per lane per round (loads in flight)
constexpr int kQueue = 32 * kBatch;   // ambiguous draws buffered per warp (>= one round)

// Lanes scan segments and count certain-below draws; ambiguous draws are queued in
// shared memory and then resolved with the exact glibc Box-Muller, one per lane.
__device__ __forceinline__ int64_t nv_count_warp(const uint32_t* __restrict__ keys,
                                                 const uint16_t* __restrict__ off, int64_t j,
                                                 int64_t S, int nseg, double x, double mu,
                                                 double sigma, NvStreamPos sp, int64_t* queue) {
  const int lane = threadIdx.x & 31;
  const NvWindow w = nv_window(x, mu, sigma);
  const int blo = (int)(w.qlo >> (NV_QBITS - 10)), bhi = (int)(w.qhi >> (NV_QBITS - 10));
  int64_t cnt = 0;
  int nq = 0;  // warp-uniform queue length
  auto drain = [&]() {
    for (int e = lane; e < nq; e += 32) cnt += nv_resolve(sp, queue[e], mu, sigma, x);
    __syncwarp();
    nq = 0;
  };
  for (int s0 = 0; s0 < nseg; s0 += 32) {
    const int s = s0 + lane;
    int start = 0, end = 0, c = 0;
    const uint32_t* seg = keys;
    int64_t base = 0;
    if (s < nseg) {
      const int64_t e0 = (int64_t)s * NV_SEG;
      const int len = (int)((S - e0) < NV_SEG ? (S - e0) : NV_SEG);
      const uint16_t* o = off + (j * nseg + s) * (int64_t)NV_B;
      start = o[blo];
      end = (bhi + 1 < NV_B) ? o[bhi + 1] : len;
      seg = keys + j * S + e0;
      base = j * S + e0;
      c = start;
    }
    // walk the window buckets in lock-step batches of kBatch keys per lane (all loads of a
    // batch in flight together); ambiguous draws are queued warp-wide
    const int span = end - start;
    int maxspan = span;
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) maxspan = max(maxspan, __shfl_xor_sync(0xffffffffu, maxspan, o2));
    for (int p0 = 0; p0 < maxspan; p0 += kBatch) {
      uint32_t kv[kBatch];
#pragma unroll
      for (int k = 0; k < kBatch; ++k) kv[k] = (p0 + k < span) ? seg[start + p0 + k] : 0u;
      unsigned amb = 0;
#pragma unroll
      for (int k = 0; k < kBatch; ++k) {
        if (p0 + k < span) {
          const int cls = nv_classify(kv[k] >> 12, w);
          c += (cls < 0) ? 1 : 0;
          amb |= (cls == 0) ? (1u << k) : 0u;
        }
      }
      const int na = __popc(amb);
      int pre = na;  // inclusive warp prefix of the ambiguous counts
#pragma unroll
      for (int o2 = 1; o2 < 32; o2 <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, pre, o2);
        if (lane >= o2) pre += t;
      }
      const int total = __shfl_sync(0xffffffffu, pre, 31);
      if (total) {
        if (nq + total > kQueue) drain();
        int pos = nq + pre - na;
        for (int k = 0; k < kBatch; ++k)
          if (amb & (1u << k)) queue[pos++] = base + (int64_t)(kv[k] & 4095u);
        __syncwarp();
        nq += total;
      }
    }
    cnt += c;
  }
  drain();
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o2);
  return cnt;
}

// gradient (tasks.py:158-160): g = (k - v) + ((h + v) * (count / S))
__device__ __forceinline__ double nv_grad_value(int64_t cnt, int64_t S, double k, double h,
                                                double v) {
  const double frac = (double)cnt / (double)S;
  return (k - v) + ((h + v) * frac);
}

namespace {


// Fused product-shard LMO exchange over NVLink peer memory (one thread of the step's
// last block): publish (value, global index, vertex value) into slot `rank` of every
// peer's mailbox, release the sequence word, then acquire all `world` entries of this
// sequence from the own mailbox and keep the global first-argmin -- the allgather +
// simopt_nv_lmo_apply of the NCCL path in one kernel, no host round trip.  Mailboxes are
// double-buffered by sequence parity (a rank cannot run two exchanges ahead).  A peer
// that never arrives ends the wait after 10 s with NV_FLAG_EXCHANGE_TIMEOUT, and every later
// exchange of the run then skips its wait (sticky NvState.exchange_failed): fail fast.
__device__ __forceinline__ void st_release_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// The fields of NvIterArgs the exchange needs, by value: taking the address of the kernel
// parameter block (a reference into a noinline call) made every thread copy it to the
// stack at kernel entry.
struct NvPeerArgs {
  double* const* peer_mb;
  int64_t world, rank, j0, d, grad_step;
  uint64_t seq;
  uint64_t* seq_ptr;
  int* flags;
};

__device__ __noinline__ void nv_peer_exchange(const NvPeerArgs a, ArgMin r, double sval, NvState* st) {
  uint64_t seq = a.seq;
  if (a.seq_ptr) {  // device-resident sequence (graph replay): this exchange's number
    seq = *a.seq_ptr + 1;
    *a.seq_ptr = seq;
  }
  const int64_t par = (int64_t)(seq & 1ULL), W = a.world;
  for (int64_t q = 0; q < W; ++q) {
    double* slot = a.peer_mb[q] + (par * W + a.rank) * 4;
    volatile double* vs = slot;
    vs[0] = r.v;
    vs[1] = (double)(r.i + a.j0);  // exact: product indices < 2^53
    vs[2] = sval;
    __threadfence_system();
    st_release_u64(reinterpret_cast<uint64_t*>(slot + 3), seq);
  }
  const double* mb = a.peer_mb[a.rank] + par * W * 4;
  ArgMin best{INFINITY, INT64_MAX};
  double bs = 0.0;
  const uint64_t t0 = globaltimer();
  bool timed_out = st->exchange_failed != 0;  // sticky: after one failure, never wait again
  for (int64_t q = 0; q < W && !timed_out; ++q) {
    const double* e = mb + q * 4;
    while (ld_acquire_u64(reinterpret_cast<const uint64_t*>(e + 3)) != seq) {
      if (globaltimer() - t0 > 10000000000ULL) { timed_out = true; break; }
    }
    if (timed_out) break;
    const volatile double* ve = e;
    const ArgMin c{ve[0], (int64_t)ve[1]};
    const ArgMin m = amin(best, c);
    if (m.i != best.i || m.v != best.v) bs = ve[2];
    best = m;
  }
  if (timed_out) {
    st->exchange_failed = 1;
    atomicOr(&a.flags[a.grad_step], NV_FLAG_EXCHANGE_TIMEOUT);
    best = ArgMin{r.v, r.i + a.j0};
    bs = sval;
  }
  st->jstar = (best.i >= a.j0 && best.i < a.j0 + a.d) ? best.i - a.j0 : -1;
  st->sval = bs;
  st->best_val = best.v;
}

// Integer form of nv_classify for one query: a key with code q is certainly below iff
// q < qb, certainly above iff q >= qa, ambiguous otherwise.  The thresholds are the
// real-number solutions of nv_classify's two inequalities in q, formed once per query
// in double; their rounding (~1e-15 z) is far inside the 0.1-code margin nv_classify's
// slack leaves, so every key either test calls certain is certain, and the count --
// certain-below keys plus the exactly resolved ambiguous ones -- is the same integer.
struct NvThresh {
  int qb, qa;
};
__device__ __forceinline__ NvThresh nv_thresh(const NvWindow& w) {
  // below: (q + 1.25) W - Z0 + eps < t  <=>  q < B;  q = QMAX is never below
  const double B = (w.t - w.eps + NV_Z0) * NV_QSCALE - 1.25;
  // above: (q - 0.25) W - Z0 - eps > t  <=>  q > A;  q = 0 is never above
  const double A = (w.t + w.eps + NV_Z0) * NV_QSCALE + 0.25;
  NvThresh r;
  r.qb = !(B > 0.0) ? 0 : (B >= (double)NV_QMAX ? NV_QMAX : (int)ceil(B));
  r.qa = !(A >= 0.0) ? (A < 0.0 ? 1 : NV_QMAX + 1)  // NaN: nothing certain (as nv_classify)
                     : (A >= (double)NV_QMAX ? NV_QMAX + 1 : max((int)floor(A) + 1, 1));
  return r;
}

// Fused FW step for the newsvendor:
//   (1) if do_update: x_j <- (gamma * ((-1 * x_j) + s_j)) + x_j with the vertex of the
//       previous LMO (frank_wolfe.py:69-82), record x_j < -FEAS_TOL, objective term;
//   (2) if do_grad: g_j at the (new) x_j, LMO values g_j * (C / c_j), argmin over all
//       products (last-block reduction), NaN flag.
// Gradient steps run in CTA rounds:
//  (A) each warp takes up to kSlotsPerWarp (8) products, one at a time from a device
//      counter (the counter read for the product after the next is in flight while the
//      current one is processed; the next product's iterate and parameters are loaded as
//      soon as its index is known); lanes = the product's segments: bucket starts of the
//      query window, then the window's keys in 16-byte loads (several in flight per lane),
//      integer thresholds count the certainly-below keys and the few ambiguous draws are
//      appended to one CTA-wide queue;
//  (B) all threads of the CTA resolve the queue with the exact glibc Box-Muller (full
//      warps instead of one partly filled pass per product);
//  (C) one thread per product forms the gradient and its LMO value.
// Ambiguous draws that do not fit the queue are resolved by the warp that found them.
constexpr int kCtaQueue = 1024;
// usable queue entries (tests shrink it through SIMOPT_NV_QCAP to drive the overflow path)
__device__ int g_nv_qcap = kCtaQueue;

// One ambiguous draw of a step (rare): appended to the CTA queue, or resolved here when the
// queue is full (returns the draw's count then, 0 when queued).  Out of line so the scan
// loops keep their register budget.
__device__ __noinline__ int nv_amb_push(uint32_t key, int sg, int slot, int64_t j, int64_t S,
                                        double mu, double sigma, double x, NvStreamPos sp,
                                        uint64_t* queue, int* q_len, int qcap) {
  const uint64_t idx = (uint64_t)(sg * NV_SEG) + (key & 4095u);
  const int pos = atomicAdd(q_len, 1);
  if (pos < qcap) {
    queue[pos] = (uint64_t)slot << 40 | idx;
    return 0;
  }
  return nv_resolve(sp, j * S + (int64_t)idx, mu, sigma, x);
}

struct NvStepCtx {
  int64_t jstar;
  double sval, gamma;
};

// (1) for product j from its current iterate x; `writer` stores the new iterate, flags and
// objective term
__device__ __forceinline__ double nv_update(const NvIterArgs& a, const NvStepCtx& cx, int64_t j,
                                           double x, bool writer) {
  if (a.do_update) {
    const double sj = (j == cx.jstar) ? cx.sval : 0.0;
    const double dir = (-1.0 * x) + sj;
    x = cx.gamma * dir + x;
    if (writer) {
      a.x[j] = x;
      if (x < -1e-10) atomicOr(&a.flags[a.step], NV_FLAG_NEGATIVE);
      if (a.terms) a.terms[j] = nv_cost_term(x, a.mu[j], a.sigma[j], a.k[j], a.h[j], a.v[j]);
    }
  }
  return x;
}

// One product's window in one segment (a lane's share of a gradient step): the keys in
// [start, end) -- bucket order, so [0, start) are the keys of lower buckets, counted by the
// caller -- certainly-below keys counted, ambiguous draws queued (nv_amb_push).  Returns the
// count on top of `start`.
//  vec (16-byte aligned rows): the 16-byte words from the one holding `start` to the one
//  holding end - 1, every key tested, no masks: the head word's keys before `start` lie in
//  buckets below the window, i.e. below qlo < qb (certainly below: counted by the test, so
//  taken out of `start`), and the tail word's keys from `end` on lie above qhi > qa
//  (certainly above, never ambiguous).  Per key one compare for the count; ambiguity is one
//  unsigned min per key and one compare per batch (key - kb <= kspan for any key), the
//  per-key mask only formed when the batch holds an ambiguous draw.
//  otherwise: the window itself, 8 single keys per batch.
template <int kVecBatch>
__device__ __forceinline__ int nv_scan_window(const uint32_t* seg, int start, int end, bool vec,
                                              uint32_t kb, uint32_t kspan, int sg, int slot,
                                              int64_t j, int64_t S, double mu, double sigma,
                                              double x, const NvStreamPos& sp, uint64_t* queue,
                                              int* q_len, int qcap) {
  int c = 0;
  if (!vec) {
    for (int p0 = start; p0 < end; p0 += 8) {
      uint32_t kv[8];
      unsigned amb = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const bool v = p0 + i < end;
        kv[i] = v ? seg[p0 + i] : 0u;
        c += (v && kv[i] < kb) ? 1 : 0;
        amb |= (v && kv[i] - kb <= kspan) ? 1u << i : 0u;
      }
      while (amb) {  // ambiguous draws: rare
        const int bit = __ffs(amb) - 1;
        amb &= amb - 1;
        uint32_t key = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) key = (bit == i) ? kv[i] : key;
        c += nv_amb_push(key, sg, slot, j, S, mu, sigma, x, sp, queue, q_len, qcap);
      }
    }
    return c;
  }
  if (end <= start) return 0;
  const int hb = start & ~3;
  const int nw = (((end - 1) & ~3) - hb) / 4 + 1;  // 16-byte words of the window
  c = hb - start;
  const uint4* vrow = reinterpret_cast<const uint4*>(seg + hb);
  for (int v0 = 0; v0 < nw; v0 += kVecBatch) {
    uint4 t[kVecBatch];
#pragma unroll
    for (int v = 0; v < kVecBatch; ++v)
      if (v0 + v < nw) t[v] = vrow[v0 + v];
    uint32_t m = 0xffffffffu;  // min over the batch of key - kb (unsigned)
#pragma unroll
    for (int v = 0; v < kVecBatch; ++v) {
      if (v0 + v < nw) {
        const uint32_t k4[4] = {t[v].x, t[v].y, t[v].z, t[v].w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          c += k4[u] < kb ? 1 : 0;
          m = min(m, k4[u] - kb);
        }
      }
    }
    if (m > kspan) continue;  // no ambiguous draw in the batch: the common case
    unsigned amb = 0;
#pragma unroll
    for (int v = 0; v < kVecBatch; ++v) {
      if (v0 + v < nw) {
        const uint32_t k4[4] = {t[v].x, t[v].y, t[v].z, t[v].w};
#pragma unroll
        for (int u = 0; u < 4; ++u) amb |= (k4[u] - kb <= kspan) ? 1u << (4 * v + u) : 0u;
      }
    }
    while (amb) {
      const int bit = __ffs(amb) - 1;
      amb &= amb - 1;
      uint32_t key = 0;
#pragma unroll
      for (int v = 0; v < kVecBatch; ++v) {
        key = (bit == 4 * v) ? t[v].x : key;
        key = (bit == 4 * v + 1) ? t[v].y : key;
        key = (bit == 4 * v + 2) ? t[v].z : key;
        key = (bit == 4 * v + 3) ? t[v].w : key;
      }
      c += nv_amb_push(key, sg, slot, j, S, mu, sigma, x, sp, queue, q_len, qcap);
    }
  }
  return c;
}

// the window [start, end) of product j in segment sg: its first and one-past-last bucket's starts
__device__ __forceinline__ void nv_bounds(const NvIterArgs& a, int64_t j, int sg, int nseg, int S32,
                                          int blo, int bhi, int& start, int& end) {
  const int e0 = sg * NV_SEG;
  const int len = (S32 - e0) < NV_SEG ? (S32 - e0) : NV_SEG;
  const uint16_t* o = a.off + (j * nseg + sg) * (int64_t)NV_B;
  start = o[blo];
  end = (bhi + 1 < NV_B) ? o[bhi + 1] : len;
}

// kVecBatch: 16-byte key loads per lane per pass.  (Measured and not kept: loading the next
// product's iterate and parameters before this product's scan, 4.03 vs 4.02 ms per pipelined
// C2 epoch; preparing the next product's window and bucket starts a product ahead, 4.24 ms --
// 80 registers leave no room for a second product's state.)
// kSlotsPerWarp: products per warp per CTA round
template <int kIterWarps, int kMinBlocks, int kVecBatch, int kSlotsPerWarp = 8>
__global__ void __launch_bounds__(kIterWarps * 32, kMinBlocks)
    k_nv_iter(NvIterArgs a) {
  constexpr int kSlots = kIterWarps * kSlotsPerWarp;
  __shared__ ArgMin warp_best[kIterWarps];
  __shared__ uint64_t queue[kCtaQueue];   // slot << 40 | draw index within the product
  __shared__ int64_t slot_j[kSlots];       // -1: empty
  __shared__ double slot_x[kSlots], slot_mu[kSlots], slot_sigma[kSlots];
  __shared__ int slot_cnt[kSlots];
  __shared__ int q_len;
  __shared__ int nan_seen;
  __shared__ bool am_last;
  if (threadIdx.x == 0) {
    nan_seen = 0;
    q_len = 0;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  NvState* st = a.state;
  NvStepCtx cx;
  cx.jstar = st->jstar;
  cx.sval = st->sval;
  // frank_wolfe.py:62-66: gamma = 2 / (epoch * inner_iters + inner + 2), IEEE double division
  cx.gamma = a.epoch_ctr ? 2.0 / (double)(*a.epoch_ctr * a.inner_iters + a.m + 2) : a.gamma;
  if (!a.do_grad) {  // update-only step: a static split
    for (int64_t j = (int64_t)blockIdx.x * kIterWarps + warp; j < a.d; j += (int64_t)gridDim.x * kIterWarps)
      nv_update(a, cx, j, a.x_in[j], lane == 0);
    if (a.stamp) {  // the last block to finish stamps the step
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&st->blocks_done, 1u) == gridDim.x - 1) {
          __threadfence();
          *a.stamp = (int64_t)globaltimer();
          st->blocks_done = 0;
        }
      }
    }
    return;
  }
  const NvStreamPos sp = a.epoch_draw
                            ? NvStreamPos{a.epoch_draw[0], a.epoch_draw[1], a.epoch_draw[2], a.epoch_draw[3]}
                            : NvStreamPos{a.seed, a.sid, a.ctr_lo, a.ctr_hi};
  __syncthreads();
  // products: warp g of the grid takes product g first, then products nwarps + n in the
  // order of a device counter n (NvState.pad, reset by the last block) -- a product's cost
  // varies with its window and ambiguous draws.  The counter is read one product ahead
  // (lane 0's atomic is in flight while the current product is processed) and the next
  // product's iterate and parameters are loaded one product ahead.
  unsigned* next = &st->pad;
  const int64_t nwarps = (int64_t)gridDim.x * kIterWarps;
  const int64_t gw = (int64_t)blockIdx.x * kIterWarps + warp;
  ArgMin best{INFINITY, INT64_MAX};
  const int S32 = (int)a.S;  // S < 2^31 (checked on the host)
  const int nseg = (int)a.nseg;
  const int qcap = min(g_nv_qcap, kCtaQueue);
  const bool vec = (a.S & 3) == 0;  // rows start 16-byte aligned: vector key loads
  unsigned pend = 0;  // lane 0: the counter value of the product after jn
  if (lane == 0 && gw < a.d) pend = atomicAdd(next, 1u);
  int64_t jn = gw;
  double xn = 0.0, mun = 0.0, sgn = 1.0;  // the next product's iterate and parameters
  if (jn < a.d) {
    xn = a.x_in[jn];
    mun = a.mu[jn];
    sgn = a.sigma[jn];
  }
  for (;;) {
    // ---- (A) count certain keys, queue ambiguous draws
    for (int k = 0; k < kSlotsPerWarp; ++k) {
      const int slot = warp * kSlotsPerWarp + k;
      const int64_t j = jn;
      if (j >= a.d) {
        if (lane == 0) slot_j[slot] = -1;
        continue;
      }
      const double x = nv_update(a, cx, j, xn, lane == 0);
      const double mu = mun, sigma = sgn;
      const unsigned got = pend;
      if (lane == 0) pend = atomicAdd(next, 1u);  // the product after the next one
      const NvWindow w = nv_window(x, mu, sigma);
      const NvThresh th = nv_thresh(w);
      // as raw keys (q << 12 | local): key < kb <=> q < qb (certainly below);
      // key - kb <= kspan (unsigned) <=> qb <= q < qa (ambiguous); qa > qb always
      const uint32_t kb = (uint32_t)th.qb << 12;
      const uint32_t kspan = (uint32_t)((((uint64_t)th.qa) << 12) - 1 - kb);
      const int blo = (int)(w.qlo >> (NV_QBITS - 10)), bhi = (int)(w.qhi >> (NV_QBITS - 10));
      int c = 0;  // per lane: certain-below (+ locally resolved) draws
      for (int s0 = 0; s0 < nseg; s0 += 32) {
        const int sg = s0 + lane;
        int start = 0, end = 0;
        const uint32_t* seg = a.keys;
        if (sg < nseg) {
          nv_bounds(a, j, sg, nseg, S32, blo, bhi, start, end);
          seg = a.keys + j * a.S + sg * NV_SEG;
          c += start;
        }
        c += nv_scan_window<kVecBatch>(seg, start, end, vec, kb, kspan, sg, slot, j, a.S, mu, sigma,
                                       x, sp, queue, &q_len, qcap);
      }
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o2);
      jn = nwarps + (int64_t)__shfl_sync(0xffffffffu, got, 0);
      if (jn < a.d) {
        xn = a.x_in[jn];
        mun = a.mu[jn];
        sgn = a.sigma[jn];
      }
      if (lane == 0) {
        slot_j[slot] = j;
        slot_x[slot] = x;
        slot_mu[slot] = mu;
        slot_sigma[slot] = sigma;
        slot_cnt[slot] = c;
      }
    }
    __syncthreads();
    // ---- (B) resolve the queued draws exactly, all threads
    const int nq = min(q_len, qcap);
    for (int e = threadIdx.x; e < nq; e += kIterWarps * 32) {
      const uint64_t v = queue[e];
      const int slot = (int)(v >> 40);
      const int64_t j = slot_j[slot];
      if (nv_resolve(sp, j * a.S + (int64_t)(v & ((1ULL << 40) - 1)), slot_mu[slot], slot_sigma[slot],
                     slot_x[slot]))
        atomicAdd(&slot_cnt[slot], 1);
    }
    __syncthreads();
    // ---- (C) gradient and LMO value per product
    if (threadIdx.x < kSlots) {
      const int64_t j = slot_j[threadIdx.x];
      if (j >= 0) {
        const double g = nv_grad_value((int64_t)slot_cnt[threadIdx.x], a.S, a.k[j], a.h[j], a.v[j]);
        a.g[j] = g;
        if (g != g) nan_seen = 1;
        const double val = g * (a.budget / a.c[j]);  // lmo.py:84
        best = amin(best, ArgMin{val, j});
      }
    }
    if (threadIdx.x == 0) q_len = 0;
    // another round while any warp holds a product
    if (!__syncthreads_or(jn < a.d)) break;
  }
  // the last counter read must have returned before this block reports done (the last
  // block resets the counter)
  if (lane == 0) asm volatile("" ::"r"(pend));
  best = warp_amin(best);
  if (lane == 0) warp_best[warp] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    ArgMin b = warp_best[0];
    for (int w = 1; w < kIterWarps; ++w) b = amin(b, warp_best[w]);
    a.part_v[blockIdx.x] = b.v;
    a.part_i[blockIdx.x] = b.i;
    if (nan_seen) atomicOr(&a.flags[a.grad_step], NV_FLAG_NAN_GRADIENT);
    __threadfence();
    const unsigned prev = atomicAdd(&st->blocks_done, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  // last block: reduce the per-block partials (deterministic: lexicographic min).
  ArgMin b{INFINITY, INT64_MAX};
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x)
    b = amin(b, ArgMin{((volatile double*)a.part_v)[i], ((volatile int64_t*)a.part_i)[i]});
  b = warp_amin(b);
  if (lane == 0) warp_best[warp] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    ArgMin r = warp_best[0];
    for (int w = 1; w < kIterWarps; ++w) r = amin(r, warp_best[w]);
    // lmo_single_budget (lmo.py:84-89): s_j* = C / c_j* iff g_j* < 0
    const double gj = a.g[r.i];
    const double sval = (gj < 0.0) ? a.budget / a.c[r.i] : 0.0;
    st->blocks_done = 0;
    st->pad = 0;  // the product counter of the next gradient step
    if (a.peer_mb == nullptr) {
      st->jstar = r.i;
      st->sval = sval;
      st->best_val = r.v;
    } else {
      nv_peer_exchange(NvPeerArgs{a.peer_mb, a.world, a.rank, a.j0, a.d, a.grad_step, a.seq,
                                  a.seq_ptr, a.flags},
                       r, sval, st);
    }
    if (a.stamp) *a.stamp = (int64_t)globaltimer();
  }
}

// Gradient steps on small product shards (d <= the grid's warps, e.g. one rank of an 8-way
// C2 run): one product per warp, statically assigned, so a step is one pass of dependent
// loads per warp with no product counter, no CTA rounds and no block barrier before the
// argmin; the few ambiguous draws of the product are queued per warp and resolved by its
// lanes (overflow resolved in place).  Same counts and LMO as k_nv_iter.
constexpr int kWarpQueue = 64;

// kMinBlocks: launch-bound blocks per SM (register cap).  The 4-warp default uses 7 (72
// registers): two blocks then sit beside the 40-register resample the small shards use, and
// the 8-way shard's pipelined epoch is 0.666 vs 0.677-0.688 ms at 80 registers (16-way:
// 0.485 vs 0.488-0.496)
template <int kIterWarps, int kVecBatch = 4, int kMinBlocks = 24 / kIterWarps>
__global__ void __launch_bounds__(kIterWarps * 32, kMinBlocks) k_nv_iter_small(NvIterArgs a) {
  __shared__ ArgMin warp_best[kIterWarps];
  __shared__ uint64_t wq[kIterWarps][kWarpQueue];
  __shared__ int wql[kIterWarps];
  __shared__ int nan_seen;
  __shared__ bool am_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) nan_seen = 0;
  if (lane == 0) wql[warp] = 0;
  NvState* st = a.state;
  NvStepCtx cx;
  cx.jstar = st->jstar;
  cx.sval = st->sval;
  cx.gamma = a.epoch_ctr ? 2.0 / (double)(*a.epoch_ctr * a.inner_iters + a.m + 2) : a.gamma;
  const NvStreamPos sp = a.epoch_draw
                            ? NvStreamPos{a.epoch_draw[0], a.epoch_draw[1], a.epoch_draw[2], a.epoch_draw[3]}
                            : NvStreamPos{a.seed, a.sid, a.ctr_lo, a.ctr_hi};
  __syncthreads();
  ArgMin best{INFINITY, INT64_MAX};
  const int S32 = (int)a.S;  // S < 2^31 (checked on the host)
  const int nseg = (int)a.nseg;
  const bool vec = (a.S & 3) == 0;
  const int64_t j = (int64_t)blockIdx.x * kIterWarps + warp;
  if (j < a.d) {
    // every per-product load issued up front (the gradient's k, h, v, c too): one round trip
    const double x0 = a.x_in[j], mu = a.mu[j], sigma = a.sigma[j];
    const double pk = a.k[j], ph = a.h[j], pv = a.v[j], pc = a.c[j];
    const double x = nv_update(a, cx, j, x0, lane == 0);
    const NvWindow w = nv_window(x, mu, sigma);
    const NvThresh th = nv_thresh(w);
    const uint32_t kb = (uint32_t)th.qb << 12;
    const uint32_t kspan = (uint32_t)((((uint64_t)th.qa) << 12) - 1 - kb);
    const int blo = (int)(w.qlo >> (NV_QBITS - 10)), bhi = (int)(w.qhi >> (NV_QBITS - 10));
    int c = 0;
    for (int s0 = 0; s0 < nseg; s0 += 32) {
      const int sg = s0 + lane;
      int start = 0, end = 0;
      const uint32_t* seg = a.keys;
      if (sg < nseg) {
        nv_bounds(a, j, sg, nseg, S32, blo, bhi, start, end);
        seg = a.keys + j * a.S + sg * NV_SEG;
        c += start;
      }
      c += nv_scan_window<kVecBatch>(seg, start, end, vec, kb, kspan, sg, 0, j, a.S, mu, sigma, x, sp,
                                     wq[warp], &wql[warp], kWarpQueue);
    }
    __syncwarp();
    const int nq = min(wql[warp], kWarpQueue);
    for (int e = lane; e < nq; e += 32)
      c += nv_resolve(sp, j * a.S + (int64_t)(wq[warp][e] & ((1ULL << 40) - 1)), mu, sigma, x);
#pragma unroll
    for (int o2 = 16; o2 > 0; o2 >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o2);
    if (lane == 0) {
      const double g = nv_grad_value((int64_t)c, a.S, pk, ph, pv);
      a.g[j] = g;
      if (g != g) nan_seen = 1;
      best = ArgMin{g * (a.budget / pc), j};  // lmo.py:84
    }
  }
  best = warp_amin(best);
  if (lane == 0) warp_best[warp] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    ArgMin b = warp_best[0];
    for (int w = 1; w < kIterWarps; ++w) b = amin(b, warp_best[w]);
    a.part_v[blockIdx.x] = b.v;
    a.part_i[blockIdx.x] = b.i;
    if (nan_seen) atomicOr(&a.flags[a.grad_step], NV_FLAG_NAN_GRADIENT);
    __threadfence();
    const unsigned prev = atomicAdd(&st->blocks_done, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return;
  __threadfence();
  // last block: reduce the per-block partials (deterministic: lexicographic min).
  ArgMin b{INFINITY, INT64_MAX};
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x)
    b = amin(b, ArgMin{((volatile double*)a.part_v)[i], ((volatile int64_t*)a.part_i)[i]});
  b = warp_amin(b);
  if (lane == 0) warp_best[warp] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    ArgMin r = warp_best[0];
    for (int w = 1; w < kIterWarps; ++w) r = amin(r, warp_best[w]);
    // lmo_single_budget (lmo.py:84-89): s_j* = C / c_j* iff g_j* < 0
    const double gj = a.g[r.i];
    const double sval = (gj < 0.0) ? a.budget / a.c[r.i] : 0.0;
    st->blocks_done = 0;
    st->pad = 0;  // the product counter of the next gradient step
    if (a.peer_mb == nullptr) {
      st->jstar = r.i;
      st->sval = sval;
      st->best_val = r.v;
    } else {
      nv_peer_exchange(NvPeerArgs{a.peer_mb, a.world, a.rank, a.j0, a.d, a.grad_step, a.seq,
                                  a.seq_ptr, a.flags},
                       r, sval, st);
    }
    if (a.stamp) *a.stamp = (int64_t)globaltimer();
  }
}

__global__ void k_nv_counts(const uint32_t* __restrict__ keys, const uint16_t* __restrict__ off,
                            const double* __restrict__ mu, const double* __restrict__ sigma,
                            int64_t d, int64_t S, int nseg, NvStreamPos sp,
                            const double* __restrict__ x, int64_t* __restrict__ counts) {
  const int warp = threadIdx.x >> 5;
  __shared__ int64_t queues[8][kQueue];
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; j < d;
       j += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const int64_t c = nv_count_warp(keys, off, j, S, nseg, x[j], mu[j], sigma[j], sp, queues[warp]);
    if ((threadIdx.x & 31) == 0) counts[j] = c;
  }
}

// Materialise the exact demand of every stored key (test/diagnostic path).
__global__ void k_nv_decode(const uint32_t* __restrict__ keys, const double* __restrict__ mu,
                            const double* __restrict__ sigma, int64_t d, int64_t S, NvStreamPos sp,
                            double* __restrict__ out) {
  const double* tab = reinterpret_cast<const double*>(simopt_sincostab_dev);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < d * S;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / S, pos = e - j * S;
    const int64_t seg0 = pos - (pos % NV_SEG);
    const int64_t i = j * S + seg0 + (int64_t)(keys[e] & 4095u);
    out[e] = mu[j] + sigma[j] * nv_exact_z(sp.seed, sp.sid, sp.clo, sp.chi, i, tab);
  }
}

}  // namespace

extern "C" int simopt_nv_geometry(int64_t* seg, int64_t* buckets) {
  if (seg) *seg = NV_SEG;
  if (buckets) *buckets = NV_B;
  return SIMOPT_OK;
}

extern "C" int simopt_nv_layout(int64_t d, int64_t S, int64_t* nseg, int64_t* key_elems,
                                int64_t* off_elems) {
  SIMOPT_REQUIRE(d >= 1 && S >= 1, SIMOPT_E_EMPTY, "need d >= 1 products and S >= 1 samples");
  const int64_t ns = ceil_div(S, NV_SEG);
  if (nseg) *nseg = ns;
  if (key_elems) *key_elems = d * S;
  if (off_elems) *off_elems = d * ns * NV_B;
  return SIMOPT_OK;
}

extern "C" int simopt_nv_resample(void* stream, uint64_t seed, uint64_t sid, uint64_t clo,
                                  uint64_t chi, int64_t d, int64_t S, uint32_t* keys,
                                  uint16_t* off) {
  SIMOPT_REQUIRE(d >= 1 && S >= 1, SIMOPT_E_EMPTY, "need at least one demand sample per product");
  const int64_t nseg = ceil_div(S, NV_SEG);
  const int64_t nblk = d * nseg;
  SIMOPT_REQUIRE(nblk < (1LL << 31), SIMOPT_E_CONFIG, "too many segments");
  const phx_keys rk = phx_round_keys(seed, sid);
  // blocks q = 0 .. ceil(d*S/4)-1 use counters clo+1 ..; when they stay within word 0
  // (the span resets of stream_block_counter then add no carry either) the first two
  // Philox rounds are partly constant (philox4x64_10_rk_c0)
  const phx_pre pre = phx_precompute(chi, rk);
  const bool no_carry = phx_no_carry(clo, (uint64_t)ceil_div(d * S, 4));
  // SIMOPT_NV_RESAMPLE=1: the single-role kernel k_nv_resample (comparison); default: the
  // warp-specialised k_nv_resample_ws (3.72 vs 4.12 ms at C2).  Both are persistent grids
  // of one full wave.  The previous epoch's step kernels (high stream priority) share the
  // SMs with it: a 4-warp step block (10 K registers, 9 KB shared) fits beside the three
  // resample CTAs (46 K registers at the default cap, 3 x 57 KB); further step blocks take an SM slot whenever
  // the scheduler has one, which costs the resample ~0.3 ms per epoch (4,3,4 is the best
  // measured trade-off, tools/nv_iter_ab.py).
  const char* ev = getenv("SIMOPT_NV_RESAMPLE");
  if (!(ev && atoi(ev) == 1)) {
    const int64_t g = nblk < (int64_t)SIMOPT_NUM_SMS * kWsPerSm ? nblk : (int64_t)SIMOPT_NUM_SMS * kWsPerSm;
    const size_t smem = sizeof(WsSmem);
    // Registers: the pipelined epoch is set by whichever of the resample and the previous
    // epoch's steps beside it ends last (tools/nv_timeline.py).  At C2 the steps' share is
    // small enough for the 48-register resample (3.70 ms alone): resample 3.79, steps 3.80 ms
    // beside each other (bench 6.55k vs 6.45k FW it/s at 40 registers).  On small product
    // shards (the one-product-per-warp step kernel, d <= 12 x SMs) the steps dominate, and
    // 40 registers leave them more issue slots: 0.689 vs 0.711 ms at the 8-way shard size.
    const int64_t small_shard = (int64_t)4 * 3 * SIMOPT_NUM_SMS;  // as simopt_nv_iter
    int regcap = d <= small_shard ? 4 : 3;
    if (const char* rc = getenv("SIMOPT_NV_WS_REGCAP")) regcap = atoi(rc) == 3 ? 3 : 4;
    static std::mutex mu;
    static std::vector<int> ready;  // devices whose shared-memory limit is raised
    int dev = 0;
    SIMOPT_CUDA(cudaGetDevice(&dev));
    cudaError_t attr_err = cudaSuccess;
    {
      std::lock_guard<std::mutex> lock(mu);
      bool have = false;
      for (int x : ready) have |= x == dev;
      if (!have) {
        const void* fns[4] = {(const void*)k_nv_resample_ws<true, 3>, (const void*)k_nv_resample_ws<false, 3>,
                              (const void*)k_nv_resample_ws<true, 4>, (const void*)k_nv_resample_ws<false, 4>};
        for (const void* f : fns)
          if (attr_err == cudaSuccess)
            attr_err = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (attr_err == cudaSuccess) ready.push_back(dev);
      }
    }
    SIMOPT_CUDA(attr_err);
    auto k = no_carry ? (regcap == 4 ? k_nv_resample_ws<true, 4> : k_nv_resample_ws<true, 3>)
                      : (regcap == 4 ? k_nv_resample_ws<false, 4> : k_nv_resample_ws<false, 3>);
    k<<<(unsigned)g, kWsProd + kWsCons, smem, as_stream(stream)>>>(rk, pre, clo, chi, d, S, (int)nseg,
                                                                   keys, off);
    SIMOPT_CHECK_LAUNCH("k_nv_resample_ws");
    return SIMOPT_OK;
  }
  const int64_t cap = (int64_t)SIMOPT_NUM_SMS * kResampleMinBlocks;
  const int64_t grid = nblk < cap ? nblk : cap;
  if (no_carry)
    k_nv_resample<true><<<(unsigned)grid, kResampleThreads, 0, as_stream(stream)>>>(
        rk, pre, clo, chi, d, S, (int)nseg, keys, off);
  else
    k_nv_resample<false><<<(unsigned)grid, kResampleThreads, 0, as_stream(stream)>>>(
        rk, pre, clo, chi, d, S, (int)nseg, keys, off);
  SIMOPT_CHECK_LAUNCH("k_nv_resample");
  return SIMOPT_OK;
}

extern "C" int simopt_nv_counts(void* stream, const uint32_t* keys, const uint16_t* off,
                                const double* mu, const double* sigma, int64_t d, int64_t S,
                                uint64_t seed, uint64_t sid, uint64_t clo, uint64_t chi,
                                const double* x, int64_t* counts) {
  const int64_t nseg = ceil_div(S, NV_SEG);
  const int grid = (int)(ceil_div(d, 8) < 8 * SIMOPT_NUM_SMS ? ceil_div(d, 8) : 8 * SIMOPT_NUM_SMS);
  k_nv_counts<<<grid, 256, 0, as_stream(stream)>>>(keys, off, mu, sigma, d, S, (int)nseg,
                                                   NvStreamPos{seed, sid, clo, chi}, x, counts);
  SIMOPT_CHECK_LAUNCH("k_nv_counts");
  return SIMOPT_OK;
}

extern "C" int simopt_nv_decode(void* stream, const uint32_t* keys, const double* mu,
                                const double* sigma, int64_t d, int64_t S, uint64_t seed,
                                uint64_t sid, uint64_t clo, uint64_t chi, double* out) {
  k_nv_decode<<<8 * SIMOPT_NUM_SMS, 256, 0, as_stream(stream)>>>(keys, mu, sigma, d, S,
                                                                 NvStreamPos{seed, sid, clo, chi},
                                                                 out);
  SIMOPT_CHECK_LAUNCH("k_nv_decode");
  return SIMOPT_OK;
}

extern "C" int simopt_nv_iter(void* stream, const NvIterArgs* args) {
  NvIterArgs a = *args;
  SIMOPT_REQUIRE(a.S < (1LL << 31), SIMOPT_E_CONFIG, "S >= 2^31 samples per product");
  {  // test hook: SIMOPT_NV_QCAP shrinks the ambiguous-draw queue (set once per process)
    static std::once_flag once;
    static cudaError_t qerr = cudaSuccess;
    std::call_once(once, [] {
      if (const char* qc = getenv("SIMOPT_NV_QCAP")) {
        const int v = atoi(qc);
        qerr = cudaMemcpyToSymbol(g_nv_qcap, &v, sizeof(int));
      }
    });
    SIMOPT_CUDA(qerr);
  }
  // gradient steps: one resident wave of blocks pulling products from a counter; update-only
  // steps: a static split.  SIMOPT_NV_ITER=W,B,V (A/B): W warps per block, B blocks per SM,
  // V 16-byte key loads per lane per pass.  Measured on the pipelined C2 epoch (the steps
  // run beside the next epoch's resample; tools/nv_iter_ab.py, interleaved medians):
  // 4,3,4 3.88 ms; 4,3,8 3.94; 4,6,4 3.94; 8,3,4 3.95; 8,3,8 4.03; 8,2,4 4.15.  Fewer,
  // smaller blocks take fewer issue slots from the resample; 72 or 64 registers (more step
  // blocks beside it) and a single block per SM were slower still.  A fourth field P sets
  // the products per warp per CTA round: 8 (default) 3.84-3.85 ms, 16 the same, 4 3.88-3.93,
  // 2 3.95 (fewer block barriers and fuller resolve passes per product).
  int kw = 4, bps = 3, vb = 4, spw = 8;
  if (const char* ev = getenv("SIMOPT_NV_ITER")) sscanf(ev, "%d,%d,%d,%d", &kw, &bps, &vb, &spw);
  const int64_t cap = a.do_grad ? (int64_t)bps * SIMOPT_NUM_SMS : 16 * SIMOPT_NUM_SMS;
  const int grid = (int)(ceil_div(a.d, kw) < cap ? ceil_div(a.d, kw) : cap);
  SIMOPT_REQUIRE(grid <= a.part_capacity, SIMOPT_E_CONFIG, "partials buffer too small");
  cudaStream_t s = as_stream(stream);
  // small shards (one product per warp fits in one wave): k_nv_iter_small
  const char* sm_env = getenv("SIMOPT_NV_ITER_SMALL");
  const int64_t small_max = (int64_t)4 * 3 * SIMOPT_NUM_SMS;
  const int sw = sm_env ? atoi(sm_env) : 4;  // warps per block (0: off)
  if (a.do_grad && a.d <= small_max && sw > 0) {
    const int ws = sw >= 16 ? 16 : (sw >= 8 ? 8 : 4);
    const int gs = (int)ceil_div(a.d, ws);
    SIMOPT_REQUIRE(gs <= a.part_capacity, SIMOPT_E_CONFIG, "partials buffer too small");
    if (ws == 16) k_nv_iter_small<16><<<gs, 16 * 32, 0, s>>>(a);
    else if (ws == 8) k_nv_iter_small<8><<<gs, 8 * 32, 0, s>>>(a);
    else k_nv_iter_small<4, 4, 7><<<gs, 4 * 32, 0, s>>>(a);
    SIMOPT_CHECK_LAUNCH("k_nv_iter_small");
    return SIMOPT_OK;
  }
  if (kw == 4 && spw != 8)
    (spw >= 16 ? k_nv_iter<4, 6, 4, 16> : spw >= 4 ? k_nv_iter<4, 6, 4, 4> : k_nv_iter<4, 6, 4, 2>)<<<grid, 4 * 32, 0, s>>>(a);
  else if (kw == 4)
    (vb == 4 ? k_nv_iter<4, 6, 4> : k_nv_iter<4, 6, 8>)<<<grid, 4 * 32, 0, s>>>(a);
  else if (bps <= 2)
    (vb == 4 ? k_nv_iter<8, 2, 4> : k_nv_iter<8, 2, 8>)<<<grid, 8 * 32, 0, s>>>(a);
  else
    (vb == 4 ? k_nv_iter<8, 3, 4> : k_nv_iter<8, 3, 8>)<<<grid, 8 * 32, 0, s>>>(a);
  SIMOPT_CHECK_LAUNCH("k_nv_iter");
  return SIMOPT_OK;
}

namespace {
__global__ void k_nv_lmo_pack(const NvState* st, int64_t j0, double* send) {
  send[0] = st->best_val;
  send[1] = (double)(st->jstar + j0);  // exact: product indices < 2^53
  send[2] = st->sval;
}

__global__ void k_nv_lmo_apply(const double* recv, int64_t world, int64_t j0, int64_t d_local,
                               NvState* st) {
  ArgMin b{recv[0], (int64_t)recv[1]};
  double sv = recv[2];
  for (int64_t r = 1; r < world; ++r) {
    const ArgMin c{recv[3 * r], (int64_t)recv[3 * r + 1]};
    const ArgMin m = amin(b, c);
    if (m.i != b.i || m.v != b.v) sv = recv[3 * r + 2];
    b = m;
  }
  st->jstar = (b.i >= j0 && b.i < j0 + d_local) ? b.i - j0 : -1;
  st->sval = sv;
  st->best_val = b.v;
}
}  // namespace

extern "C" int simopt_nv_lmo_pack(void* stream, const NvState* state, int64_t j0, double* send) {
  k_nv_lmo_pack<<<1, 1, 0, as_stream(stream)>>>(state, j0, send);
  SIMOPT_CHECK_LAUNCH("k_nv_lmo_pack");
  return SIMOPT_OK;
}

extern "C" int simopt_nv_lmo_apply(void* stream, const double* recv, int64_t world, int64_t j0,
                                   int64_t d_local, NvState* state) {
  SIMOPT_REQUIRE(world >= 1, SIMOPT_E_CONFIG, "world size must be >= 1");
  k_nv_lmo_apply<<<1, 1, 0, as_stream(stream)>>>(recv, world, j0, d_local, state);
  SIMOPT_CHECK_LAUNCH("k_nv_lmo_apply");
  return SIMOPT_OK;
}

namespace {
__global__ void k_nv_cost(const double* __restrict__ x, const double* __restrict__ mu,
                          const double* __restrict__ sigma, const double* __restrict__ unit,
                          const double* __restrict__ hold, const double* __restrict__ sell,
                          int64_t d, double* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < d;
       j += (int64_t)gridDim.x * blockDim.x)
    out[j] = nv_cost_term(x[j], mu[j], sigma[j], unit[j], hold[j], sell[j]);
}

// One epoch's records (simopt_nv_epoch_records), two launches:
//  k_nv_records_terms  newsvendor_cost_block of every (step, product), all threads;
//  k_nv_records        warp g takes unit (m, job, chunk), job 0 = dot(c, x_m), job 1 = sum
//                      of step m's terms; lane 0 adds the chunk in index order from 0.0
//                      (_kernels.py:45-68, the dot_partials / sum_partials chains) from
//                      256-element tiles the warp stages in shared memory; the warp that
//                      completes a unit's last chunk folds its partials pairwise (the tree
//                      of k_fold_strided).
__global__ void k_nv_records_terms(const double* __restrict__ xs, int64_t H, int64_t r0, int64_t M,
                                   const double* __restrict__ mu, const double* __restrict__ sigma,
                                   const double* __restrict__ unit, const double* __restrict__ hold,
                                   const double* __restrict__ sell, int64_t d,
                                   double* __restrict__ terms) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < M * d;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = e / d, i = e - m * d;
    const double x = xs[((r0 + m) % H) * d + i];
    terms[e] = nv_cost_term(x, mu[i], sigma[i], unit[i], hold[i], sell[i]);
  }
}

constexpr int kRecWarps = 4, kRecTile = 256;
__global__ void __launch_bounds__(kRecWarps * 32)
    k_nv_records(const double* __restrict__ xs, int64_t H, int64_t r0, int64_t M,
                 const double* __restrict__ c, const double* __restrict__ terms, int64_t d,
                 int64_t chunk, int64_t nch, double* __restrict__ part, unsigned* __restrict__ cnt,
                 double* __restrict__ spent, double* __restrict__ objs) {
  __shared__ double buf[kRecWarps][2][kRecTile];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t total = M * 2 * nch;
  for (int64_t g = (int64_t)blockIdx.x * kRecWarps + warp; g < total;
       g += (int64_t)gridDim.x * kRecWarps) {
    const int64_t ch = g % nch, u = g / nch;  // u = m * 2 + job
    const int job = (int)(u & 1);
    const int64_t m = u >> 1;
    const double* x = xs + ((r0 + m) % H) * d;
    const double* y = terms + m * d;
    const int64_t lo = ch * chunk, hi = lo + chunk < d ? lo + chunk : d;
    constexpr int kPer = kRecTile / 32;
    double v[kPer];
    auto load = [&](int64_t base) {  // raw loads, consumed one tile later (in flight meanwhile)
#pragma unroll
      for (int t = 0; t < kPer; ++t) {
        const int64_t i = base + lane + 32 * t;
        v[t] = i < hi ? (job == 0 ? c[i] * x[i] : y[i]) : 0.0;
      }
    };
    double s = 0.0;
    load(lo);
    int par = 0;
    for (int64_t base = lo; base < hi; base += kRecTile) {
      double* b = buf[warp][par];
#pragma unroll
      for (int t = 0; t < kPer; ++t) b[lane + 32 * t] = v[t];
      __syncwarp();
      if (base + kRecTile < hi) load(base + kRecTile);
      if (lane == 0) {
        const int n = (int)(hi - base < kRecTile ? hi - base : kRecTile);
        if (n == kRecTile) {  // 16-element register batches: the chain runs at DADD latency
          double w[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) w[k] = b[k];
          for (int t = 0; t < kRecTile; t += 16) {
            double z[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) z[k] = w[k];
            if (t + 16 < kRecTile) {
#pragma unroll
              for (int k = 0; k < 16; ++k) w[k] = b[t + 16 + k];
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) s = s + z[k];
          }
        } else {
          for (int t = 0; t < n; ++t) s = s + b[t];
        }
      }
      par ^= 1;
    }
    __syncwarp();
    if (lane == 0) {
      part[u * nch + ch] = s;
      __threadfence();
      if (atomicAdd(&cnt[u], 1u) == (unsigned)(nch - 1)) {
        __threadfence();
        volatile double* q = part + u * nch;
        int64_t n = nch;
        while (n > 1) {  // pairwise levels, odd tail carried (k_fold_strided's tree)
          const int64_t h = n >> 1;
          for (int64_t i = 0; i < h; ++i) q[i] = q[2 * i] + q[2 * i + 1];
          if (n & 1) { q[h] = q[n - 1]; n = h + 1; } else { n = h; }
        }
        (job == 0 ? spent : objs)[m] = q[0];
      }
    }
  }
}
}  // namespace

extern "C" int simopt_nv_epoch_records(void* stream, const double* xs, int64_t H, int64_t r0,
                                       int64_t M, const double* c, const double* mu,
                                       const double* sigma, const double* unit, const double* hold,
                                       const double* sell, int64_t d, int64_t chunk, double* spent,
                                       double* objs) {
  SIMOPT_REQUIRE(chunk >= 1, SIMOPT_E_CONFIG, "chunk_size must be >= 1, got %lld", (long long)chunk);
  SIMOPT_REQUIRE(H >= 1 && M >= 0 && r0 >= 0, SIMOPT_E_CONFIG, "bad iterate ring");
  if (M == 0) return SIMOPT_OK;
  cudaStream_t st = as_stream(stream);
  if (d == 0) {  // empty sums are 0.0
    SIMOPT_CUDA(cudaMemsetAsync(spent, 0, M * sizeof(double), st));
    SIMOPT_CUDA(cudaMemsetAsync(objs, 0, M * sizeof(double), st));
    return SIMOPT_OK;
  }
  const int64_t nch = ceil_div(d, chunk);
  const int64_t units = M * 2;
  const size_t tbytes = (size_t)(M * d) * sizeof(double);
  unsigned char* ws = static_cast<unsigned char*>(
      simopt_scratch(st, tbytes + units * nch * sizeof(double) + units * sizeof(unsigned) + 64));
  SIMOPT_REQUIRE(ws != nullptr, SIMOPT_E_CUDA, "%s", simopt_last_error());
  double* terms = reinterpret_cast<double*>(ws);
  double* part = reinterpret_cast<double*>(ws + tbytes);
  unsigned* cnt = reinterpret_cast<unsigned*>(ws + tbytes + units * nch * sizeof(double));
  SIMOPT_CUDA(cudaMemsetAsync(cnt, 0, units * sizeof(unsigned), st));
  const int64_t tg = ceil_div(M * d, 256);
  k_nv_records_terms<<<(int)(tg < 16 * SIMOPT_NUM_SMS ? tg : 16 * SIMOPT_NUM_SMS), 256, 0, st>>>(
      xs, H, r0, M, mu, sigma, unit, hold, sell, d, terms);
  SIMOPT_CHECK_LAUNCH("k_nv_records_terms");
  const int64_t g = ceil_div(units * nch, kRecWarps);
  const int grid = (int)(g < 8 * SIMOPT_NUM_SMS ? g : 8 * SIMOPT_NUM_SMS);
  k_nv_records<<<grid, kRecWarps * 32, 0, st>>>(xs, H, r0, M, c, terms, d, chunk, nch, part, cnt,
                                                spent, objs);
  SIMOPT_CHECK_LAUNCH("k_nv_records");
  return SIMOPT_OK;
}

extern "C" int simopt_nv_cost_terms(void* stream, const double* x, const double* mu,
                                    const double* sigma, const double* unit, const double* hold,
                                    const double* sell, int64_t d, double* out) {
  if (d == 0) return SIMOPT_OK;
  k_nv_cost<<<(int)(ceil_div(d, 256) < 2048 ? ceil_div(d, 256) : 2048), 256, 0,
              as_stream(stream)>>>(x, mu, sigma, unit, hold, sell, d, out);
  SIMOPT_CHECK_LAUNCH("k_nv_cost");
  return SIMOPT_OK;
}

namespace {
// ecdf_count_block (_kernels.py:245-259): upper-bound binary search on sorted rows.
__global__ void k_ecdf_sorted(const double* __restrict__ samples, int64_t rows, int64_t s,
                              const double* __restrict__ x, int64_t* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < rows;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double xj = x[j];
    const double* row = samples + j * s;
    int64_t lo = 0, hi = s;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (row[mid] <= xj) lo = mid + 1; else hi = mid;
    }
    out[j] = lo;
  }
}

__global__ void k_nv_grad_counts(const int64_t* __restrict__ cnt, int64_t S,
                                 const double* __restrict__ k, const double* __restrict__ h,
                                 const double* __restrict__ v, int64_t d, double* __restrict__ g) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < d;
       j += (int64_t)gridDim.x * blockDim.x)
    g[j] = nv_grad_value(cnt[j], S, k[j], h[j], v[j]);
}

// nv_gradient_exact (tasks.py:163-171): z = (x - mu)/sigma, cdf = 0.5 (1 + erf(z SQRT1_2))
// (normal_cdf_block, _kernels.py:204-207, glibc erf), g = (k - v) + ((h + v) cdf)
__global__ void k_nv_grad_exact(const double* __restrict__ x, const double* __restrict__ mu,
                                const double* __restrict__ sigma, const double* __restrict__ k,
                                const double* __restrict__ h, const double* __restrict__ v, int64_t d,
                                double* __restrict__ g) {
  const double SQRT1_2 = 0.7071067811865476;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < d;
       j += (int64_t)gridDim.x * blockDim.x) {
    const double z = (x[j] - mu[j]) / sigma[j];
    const double cdf = 0.5 * (1.0 + glibc_erf(z * SQRT1_2, simopt_exptab_dev));
    g[j] = (k[j] - v[j]) + ((h[j] + v[j]) * cdf);
  }
}
}  // namespace

extern "C" int simopt_nv_grad_exact(void* stream, const double* x, const double* mu, const double* sigma,
                                    const double* k, const double* h, const double* v, int64_t d,
                                    double* g) {
  if (d == 0) return SIMOPT_OK;
  k_nv_grad_exact<<<(int)(ceil_div(d, 256) < 4096 ? ceil_div(d, 256) : 4096), 256, 0,
                    as_stream(stream)>>>(x, mu, sigma, k, h, v, d, g);
  SIMOPT_CHECK_LAUNCH("k_nv_grad_exact");
  return SIMOPT_OK;
}

extern "C" int simopt_ecdf_count_sorted(void* stream, const double* samples, int64_t rows,
                                        int64_t s, const double* x, int64_t* counts) {
  if (rows == 0) return SIMOPT_OK;
  k_ecdf_sorted<<<(int)(ceil_div(rows, 128) < 4096 ? ceil_div(rows, 128) : 4096), 128, 0,
                  as_stream(stream)>>>(samples, rows, s, x, counts);
  SIMOPT_CHECK_LAUNCH("k_ecdf_sorted");
  return SIMOPT_OK;
}

extern "C" int simopt_nv_grad_from_counts(void* stream, const int64_t* counts, int64_t S,
                                          const double* k, const double* h, const double* v,
                                          int64_t d, double* g) {
  if (d == 0) return SIMOPT_OK;
  k_nv_grad_counts<<<(int)(ceil_div(d, 256) < 4096 ? ceil_div(d, 256) : 4096), 256, 0,
                     as_stream(stream)>>>(counts, S, k, h, v, d, g);
  SIMOPT_CHECK_LAUNCH("k_nv_grad_counts");
  return SIMOPT_OK;
}

namespace {
// max |z~ - z| over the first n normals of a draw (evidence for NV_EPSZ).
__global__ void k_nv_approx_error(const phx_keys rk, uint64_t seed, uint64_t sid, uint64_t clo,
                                  uint64_t chi, int64_t nblk, unsigned long long* __restrict__ out) {
  __shared__ double tab[SIMOPT_SINCOSTAB_N];
  load_sincostab(tab);
  double m = 0.0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nblk;
       q += (int64_t)gridDim.x * blockDim.x) {
    const phx4 w = philox4x64_10_rk(stream_block_counter(clo, chi, (uint64_t)q), rk);
    float za[4];
    nv_approx_pair(w.v[0], w.v[1], &za[0], &za[1]);
    nv_approx_pair(w.v[2], w.v[3], &za[2], &za[3]);
    double ze[4];
    glibc_boxmuller_fast(phx_u01(w.v[0]), phx_u01(w.v[1]), tab, &ze[0], &ze[1]);
    glibc_boxmuller_fast(phx_u01(w.v[2]), phx_u01(w.v[3]), tab, &ze[2], &ze[3]);
    for (int k = 0; k < 4; ++k) m = fmax(m, fabs((double)za[k] - ze[k]));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}
}  // namespace

extern "C" int simopt_nv_approx_error(void* stream, uint64_t seed, uint64_t sid, uint64_t clo,
                                      uint64_t chi, int64_t n, double* out_max, double* eps) {
  if (eps) *eps = NV_EPSZ;
  SIMOPT_REQUIRE(n >= 4, SIMOPT_E_EMPTY, "need n >= 4");
  cudaStream_t st = as_stream(stream);
  SIMOPT_CUDA(cudaMemsetAsync(out_max, 0, sizeof(double), st));
  k_nv_approx_error<<<8 * SIMOPT_NUM_SMS, 256, 0, st>>>(phx_round_keys(seed, sid), seed, sid, clo,
                                                         chi, n / 4,
                                                         reinterpret_cast<unsigned long long*>(out_max));
  SIMOPT_CHECK_LAUNCH("k_nv_approx_error");
  return SIMOPT_OK;
}

extern "C" int simopt_peer_alloc(int64_t bytes, void** ptr, void* handle64) {
  SIMOPT_REQUIRE(bytes > 0, SIMOPT_E_CONFIG, "mailbox size must be > 0");
  SIMOPT_CUDA(cudaMalloc(ptr, (size_t)bytes));
  SIMOPT_CUDA(cudaMemset(*ptr, 0xff, (size_t)bytes));  // sequence words never match at start
  cudaIpcMemHandle_t h;
  SIMOPT_CUDA(cudaIpcGetMemHandle(&h, *ptr));
  memcpy(handle64, &h, sizeof(h));
  return SIMOPT_OK;
}

extern "C" int simopt_peer_open(const void* handle64, void** ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  SIMOPT_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return SIMOPT_OK;
}

extern "C" int simopt_peer_close(void* ptr) {
  SIMOPT_CUDA(cudaIpcCloseMemHandle(ptr));
  return SIMOPT_OK;
}

extern "C" int simopt_peer_free(void* ptr) {
  SIMOPT_CUDA(cudaFree(ptr));
  return SIMOPT_OK;
}
