// kernels.cu -- hand-written sm_100a kernels for the cascade-hashing hot path.
//
//   K1 row_mean_kernel        engine.cpp:446-461   exact sequential FP64 chain
//   K2 project_kernel         hashmatch.cpp:71-100 FP32 projections d.p per image residency
//      codes_kernel                                per row: d.p - m.p + certified sign
//      codes_fixup_kernel                          FP64 reference-order recompute of
//      codes_overflow_kernel                       the uncertified signs
//   K3 tables_{hist,scan,scatter}  hashmatch.cpp:120-145 bucket index per (image,row)
//   K4 match_kernel           hashmatch.cpp:147-208 bucket union + Hamming top-K +
//                                                  certified Euclidean re-rank + ratio
//   K6 scan_counts / compact  engine.cpp:475-487   ascending-query match lists
//
// Exactness contract: every decision equals the
// reference's IEEE-754 double computation.  FP32 is only used as a certified
// filter: a result is accepted when a rigorous forward error bound proves the
// FP64 result has the same sign / ordering; otherwise the FP64 path recomputes
// it with __dadd_rn/__dmul_rn/__dsub_rn/__dsqrt_rn in the reference order.
#include <cuda_runtime.h>
#include <climits>
#include <cstdint>
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "bmg_internal.h"

namespace bmg {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr uint32_t kEmpty = 0xffffffffu;

// Gate (uniform across the grid): the kernel is a no-op when *gate == 0 (the
// chain fallback runs only when the exact parallel mean gave up).
__device__ __forceinline__ bool gated_off(const uint32_t* gate) {
  return gate != nullptr && *reinterpret_cast<const volatile uint32_t*>(gate) == 0u;
}

// ---------------------------------------------------------------------------
// K1: row centering mean (engine.cpp:446-461): acc[c] += (double)d.v[c] over
// the row's images in ascending id order, descriptors in index order, then
// mean[c] = float(acc[c] / (double)total).
//
// Reproduced bit for bit without running the 128 dependent FP64 chains.
// Descriptor values in (-2^7, 2^7) whose lowest set bit is >= 2^-96 are exact
// in 128-bit fixed point with 96 fractional bits ("F96"), and so is every
// prefix sum S_k of up to 2^23 of them (|S_k| < 2^30, i128 holds 2^31).  The chain's state is
// acc_k = RN(acc_{k-1} + x_k); when the exact value acc_{k-1} + x_k fits a
// binary64 (its F96 bit span is <= 53 bits) the add is exact.  Hence
// acc_k = S_k + delta, where delta changes only at the steps whose exact sum
// needs rounding ("events", a few per channel in a BASELINE row), and there
// delta' = RN(S_k + delta) - S_k.
//   mean_sums     per 128-descriptor tile and channel: the F96 tile sum, the
//                 range of its partial sums and the lowest set bit of any x
//   mean_resolve  one CTA per channel: exclusive scan of the tile sums, then
//                 a tile certificate -- every partial sum of tile t is a
//                 multiple of 2^low inside [P_t + delta + lo, P_t + delta + hi],
//                 so its bit span is bounded without walking it.  All tiles
//                 are certified in parallel against the current delta; the
//                 first one that is not is walked by one warp (warp scan of
//                 its 128 steps, every event replayed in order), delta is
//                 updated and certification resumes after it.
// A row outside the F96 range, or with more than kMeanMaxWalks uncertified
// tiles in a channel, falls back to mean_chain_kernel, the literal chain.
// ---------------------------------------------------------------------------
using i128 = __int128;
using u128 = unsigned __int128;
constexpr uint32_t kNoLow = 0xffffu;          // tile of zeros: adds nothing
constexpr int kMeanMaxWalks = 1024;

// x * 2^96 as an integer; ok = false when that is not exact or |x| >= 2^7
__device__ __forceinline__ i128 to_f96(float x, bool& ok) {
  const uint32_t u = __float_as_uint(x);
  const int e = (u >> 23) & 0xff;
  const uint32_t m = (u & 0x7fffffu) | 0x800000u;
  u128 mag = 0;
  if (e >= 54 && e < 127 + 7) {
    mag = (u128)m << (e - 54);  // x = m * 2^(e-150) = m << (e-54) F96 units
  } else if (e == 0) {
    ok &= (u & 0x7fffffu) == 0u;  // +-0 (subnormals are below 2^-96)
  } else if (e < 54 && e > 54 - 24) {
    const int sh = 54 - e;
    ok &= (m & ((1u << sh) - 1u)) == 0u;
    mag = m >> sh;
  } else {
    ok = false;
  }
  return (u >> 31) ? -(i128)mag : (i128)mag;
}

__device__ __forceinline__ u128 abs128(i128 v) { return v < 0 ? (u128)(-v) : (u128)v; }

__device__ __forceinline__ int top_bit(u128 a) {  // a != 0
  const uint64_t hi = (uint64_t)(a >> 64), lo = (uint64_t)a;
  return hi ? 127 - __clzll((long long)hi) : 63 - __clzll((long long)lo);
}

__device__ __forceinline__ int low_bit(u128 a) {  // a != 0
  const uint64_t hi = (uint64_t)(a >> 64), lo = (uint64_t)a;
  return lo ? __ffsll((long long)lo) - 1 : 63 + __ffsll((long long)hi);
}

// is the F96 value v exactly representable as a binary64?
__device__ __forceinline__ bool fits_double(i128 v) {
  const u128 a = abs128(v);
  return a == 0 || top_bit(a) - low_bit(a) <= 52;
}

// round-to-nearest-even of v to 53 significant bits (the FP64 add's rounding)
__device__ __forceinline__ i128 round53(i128 v) {
  u128 a = abs128(v);
  if (a == 0) return v;
  const int sh = top_bit(a) - 52;
  if (sh > 0) {
    u128 q = a >> sh;
    const u128 rem = a - (q << sh), half = (u128)1 << (sh - 1);
    if (rem > half || (rem == half && (q & 1))) q += 1;
    a = q << sh;
  }
  return v < 0 ? -(i128)a : (i128)a;
}

// v fits a double (checked): exact conversion
__device__ __forceinline__ double f96_to_double(i128 v) {
  const u128 a = abs128(v);
  const double hi = __ull2double_rn((unsigned long long)(a >> 64));
  const double lo = __ull2double_rn((unsigned long long)a);
  const double r = __dmul_rn(__dadd_rn(__dmul_rn(hi, 18446744073709551616.0), lo), 0x1p-96);
  return v < 0 ? -r : r;
}

__device__ __forceinline__ i128 shfl_i128(i128 v, int src) {
  const uint64_t lo = __shfl_sync(kFull, (unsigned long long)(uint64_t)v, src);
  const uint64_t hi = __shfl_sync(kFull, (unsigned long long)(uint64_t)((u128)v >> 64), src);
  return (i128)(((u128)hi << 64) | lo);
}

__device__ __forceinline__ i128 shfl_up_i128(i128 v, int d) {
  const uint64_t lo = __shfl_up_sync(kFull, (unsigned long long)(uint64_t)v, d);
  const uint64_t hi = __shfl_up_sync(kFull, (unsigned long long)(uint64_t)((u128)v >> 64), d);
  return (i128)(((u128)hi << 64) | lo);
}

constexpr uint32_t kBadTile = 0xfffffffeu;  // tile_low: a value outside F96 (row takes the chain)

struct TileRange {
  i128 lo, hi;
};

// Statistics of rows [r0, r1) of one channel (ld(r) = the value): the F96
// sum, the range [lo, hi] of the partial sums and the lowest set F96 bit.
// A check pass finds the lowest set bit and whether every value is a
// multiple of 2^-49 below 2^7: then the sums run exactly in int64 at scale
// 2^49 (|partial sum| < 64 * 2^56), one add and two compares per value
// instead of the int128 ones.
struct HalfStats {
  i128 s, lo, hi;
  uint32_t low;
  bool ok;
};
template <typename Ld>
__device__ __forceinline__ HalfStats half_tile_stats(int r0, int r1, Ld&& ld) {
  HalfStats o;
  o.low = kNoLow;
  o.ok = true;
  bool fast = true;
#pragma unroll 16
  for (int r = r0; r < r1; ++r) {
    const uint32_t u = __float_as_uint(ld(r));
    const int e = (int)((u >> 23) & 0xff);
    const uint32_t lb = (uint32_t)(e - 54 + (__ffs((int)((u & 0x7fffffu) | 0x800000u)) - 1));
    const bool nz = (u & 0x7fffffffu) != 0u;
    o.low = nz ? min(o.low, lb) : o.low;
    fast &= !nz || (e >= 1 && e < 127 + 7 && (int)lb >= 96 - 49);
  }
  o.s = o.lo = o.hi = 0;
  if (fast) {
    long long s6 = 0, lo6 = 0, hi6 = 0;
#pragma unroll 16
    for (int r = r0; r < r1; ++r) {
      const uint32_t u = __float_as_uint(ld(r));
      const int e = (int)((u >> 23) & 0xff);
      const long long m = (long long)((u & 0x7fffffu) | 0x800000u);
      const int sh = e - 101;  // x * 2^49 = m * 2^(e - 101), exact by the fast-path test
      long long v = sh >= 0 ? m << sh : m >> min(-sh, 63);
      v = (u & 0x7fffffffu) ? ((u >> 31) ? -v : v) : 0;
      s6 += v;
      lo6 = min(lo6, s6);
      hi6 = max(hi6, s6);
    }
    o.s = (i128)s6 * ((i128)1 << 47);  // F96 = (x * 2^49) * 2^47
    o.lo = (i128)lo6 * ((i128)1 << 47);
    o.hi = (i128)hi6 * ((i128)1 << 47);
  } else {
#pragma unroll 16
    for (int r = r0; r < r1; ++r) {
      o.s += to_f96(ld(r), o.ok);
      o.lo = o.s < o.lo ? o.s : o.lo;
      o.hi = o.s > o.hi ? o.s : o.hi;
    }
  }
  return o;
}

// Tile statistics of one 128-descriptor tile, 128 P threads: thread (h, c)
// covers rows [128h/P, 128(h+1)/P) of channel c; the parts meet in shared
// memory and the result goes to the image's arrays (ImgDev::tsum / trng /
// tlow) at tile index ti.  Contains __syncthreads (call from every thread).
template <int P>
struct TileStatsSmem {
  i128 sum[P][kDim], lo[P][kDim], hi[P][kDim];
  uint32_t low[P][kDim];
};
template <int P, typename Ld>
__device__ __forceinline__ void tile_stats(const ImgDev& im, uint32_t ti, int nd, TileStatsSmem<P>& sm, Ld&& ld) {
  const int c = threadIdx.x & (kDim - 1), h = threadIdx.x >> 7;
  const int r0 = h * (kCodesTile / P), r1 = min(nd, r0 + kCodesTile / P);
  const HalfStats hs = half_tile_stats(r0, r1, [&](int r) { return ld(r, c); });
  sm.sum[h][c] = hs.s;
  sm.lo[h][c] = hs.lo;
  sm.hi[h][c] = hs.hi;
  sm.low[h][c] = hs.low;
  const int bad = __syncthreads_or(!hs.ok);
  if (h == P - 1) {
    // part q's partial sums are offset by the parts before it
    i128 s0 = 0, lo = 0, hi = 0;
    uint32_t low = kNoLow;
#pragma unroll
    for (int q = 0; q < P; ++q) {
      const i128 l = s0 + sm.lo[q][c], u = s0 + sm.hi[q][c];
      lo = l < lo ? l : lo;
      hi = u > hi ? u : hi;
      s0 += sm.sum[q][c];
      low = min(low, sm.low[q][c]);
    }
    const size_t o = (size_t)ti * kDim + c;
    static_cast<i128*>(im.tsum)[o] = s0;
    TileRange rg;
    rg.lo = lo;
    rg.hi = hi;
    static_cast<TileRange*>(im.trng)[o] = rg;
    im.tlow[o] = bad ? kBadTile : low;
  }
}

// Tile statistics for a row's tiles whose images do not carry them yet
// (the SIMT projection path): one CTA per tile.
constexpr int kSumsThreads = 256;
__global__ void __launch_bounds__(kSumsThreads) mean_sums_kernel(const ImgDev* __restrict__ imgs,
                                                                 const uint32_t* __restrict__ tile_img,
                                                                 const uint32_t* __restrict__ tile_start) {
  __shared__ TileStatsSmem<kSumsThreads / kDim> sm;
  const ImgDev im = imgs[tile_img[blockIdx.x]];
  const uint32_t i0 = tile_start[blockIdx.x];
  const int nd = min(kCodesTile, (int)(im.n - i0));
  const float* d = im.desc + (size_t)i0 * kDim;
  tile_stats(im, i0 / kCodesTile, nd, sm, [&](int r, int c) { return __ldg(d + (size_t)r * kDim + c); });
}

// Certificate for tile t with the accumulator v = P_t + delta at its start:
// every partial sum v + p_k is a multiple of 2^low and lies in
// [v + lo, v + hi], so its magnitude is at most the larger end's; no step
// needs rounding when that bit span is <= 52.
__device__ __forceinline__ bool tile_certified(i128 v, const TileRange& rg, uint32_t lowx) {
  if (lowx == kNoLow) return true;  // all zeros: the accumulator stays v
  const u128 a = abs128(v);
  int low = (int)lowx;
  if (a) low = min(low, low_bit(a));
  const u128 m0 = abs128(v + rg.lo), m1 = abs128(v + rg.hi);
  const u128 m = m0 > m1 ? m0 : m1;
  return m == 0 || top_bit(m) - low <= 52;
}

#ifndef BMG_RESOLVE_THREADS
#define BMG_RESOLVE_THREADS 256
#endif
constexpr int kResolveThreads = BMG_RESOLVE_THREADS;

// exclusive block scan of one i128 per thread (warp shuffles, then the warp
// totals in shared memory); returns the block total in *total
__device__ __forceinline__ i128 block_excl_scan_i128(i128 v, i128* s_w, i128* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
  i128 incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const i128 y = shfl_up_i128(incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    i128 w = lane < nw ? s_w[lane] : (i128)0;
    i128 wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const i128 y = shfl_up_i128(wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < nw) s_w[lane] = wi - w;  // exclusive warp offsets
    if (lane == 31) s_w[32] = wi;
  }
  __syncthreads();
  const i128 out = s_w[warp] + incl - v;
  *total = s_w[32];
  __syncthreads();
  return out;
}

// tile t of the row -> its statistics' offset in its image's arrays
__device__ __forceinline__ const ImgDev& tile_of(const ImgDev* imgs, const uint32_t* tile_img,
                                                 const uint32_t* tile_start, int t, int c, size_t& o) {
  const ImgDev& im = imgs[tile_img[t]];
  o = (size_t)(tile_start[t] / kCodesTile) * kDim + c;
  return im;
}

__global__ void __launch_bounds__(kResolveThreads) mean_resolve_kernel(
    const ImgDev* __restrict__ imgs, const uint32_t* __restrict__ tile_img,
    const uint32_t* __restrict__ tile_start, i128* __restrict__ tile_sum, int n_tiles, unsigned long long total,
    MeanState* st, float* __restrict__ mean_out, double* __restrict__ acc_out) {
  __shared__ i128 part[33];
  __shared__ i128 s_delta;
  __shared__ int s_fail;
  const int c = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  // ---- exclusive scan of the tile sums of channel c (into tile_sum, the
  // row's prefix scratch); a tile with a value outside F96 sends the row to
  // the chain
  const int per = (n_tiles + kResolveThreads - 1) / kResolveThreads;
  const int t0 = min(n_tiles, tid * per), t1 = min(n_tiles, t0 + per);
  i128 loc = 0;
  bool bad = false;
  for (int t = t0; t < t1; ++t) {
    size_t o;
    const ImgDev& im = tile_of(imgs, tile_img, tile_start, t, c, o);
    loc += static_cast<const i128*>(im.tsum)[o];
    bad |= im.tlow[o] == kBadTile;
  }
  if (__syncthreads_or(bad)) {
    if (tid == 0) {
      st->bad = 1u;
      st->need_chain = 1u;
    }
    return;
  }
  i128 row_total;
  {
    i128 run = block_excl_scan_i128(loc, part, &row_total);
    for (int t = t0; t < t1; ++t) {
      size_t o;
      const ImgDev& im = tile_of(imgs, tile_img, tile_start, t, c, o);
      tile_sum[(size_t)t * kDim + c] = run;
      run += static_cast<const i128*>(im.tsum)[o];
    }
  }
  if (tid == 0) s_delta = 0;
  __syncthreads();  // the prefixes in tile_sum are read by other threads below

  // ---- certify / walk
  i128 delta = 0;
  int cur = 0, walked = 0, events = 0;
  bool give_up = false;
  for (;;) {
    // certify forward from `cur`, one tile per thread per window, stopping
    // at the first window holding an uncertified tile (so a row costs about
    // one pass over its tiles plus one window per walked tile)
    int f = 0x7fffffff;
    for (int w0 = cur; w0 < n_tiles; w0 += kResolveThreads) {
      const int t = w0 + tid;
      bool fail = false;
      if (t < n_tiles) {
        size_t o;
        const ImgDev& im = tile_of(imgs, tile_img, tile_start, t, c, o);
        fail = !tile_certified(tile_sum[(size_t)t * kDim + c] + delta, static_cast<const TileRange*>(im.trng)[o],
                               im.tlow[o]);
      }
      // one barrier per certified window; the first failing tile only when
      // there is one
      if (__syncthreads_or(fail)) {
        if (tid == 0) s_fail = 0x7fffffff;
        __syncthreads();
        if (fail) atomicMin(&s_fail, t);
        __syncthreads();
        f = s_fail;
        break;
      }
    }
    if (f == 0x7fffffff) break;
    if (walked >= kMeanMaxWalks) {
      give_up = true;
      break;
    }
    if (tid < 32) {
      // walk tile f: lane l takes step b + l of each 32-step batch; the warp
      // scan gives every S_k, the ballot the first step that needs rounding
      const uint32_t img = tile_img[f], i0 = tile_start[f];
      const int nd = min(kCodesTile, (int)(imgs[img].n - i0));
      const float* col = imgs[img].desc + (size_t)i0 * kDim + c;
      i128 V = tile_sum[(size_t)f * kDim + c];
      i128 dl = delta;
      for (int b = 0; b < nd; b += 32) {
        const int r = b + lane;
        bool ok = true;
        const i128 x = r < nd ? to_f96(__ldg(col + (size_t)r * kDim), ok) : (i128)0;
        i128 incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const i128 y = shfl_up_i128(incl, o);
          if (lane >= o) incl += y;
        }
        const i128 S = V + incl;
        int start = 0;
        for (;;) {
          const bool fail = r < nd && lane >= start && !fits_double(S + dl);
          const unsigned m = __ballot_sync(kFull, fail);
          if (!m) break;
          const int fl = __ffs(m) - 1;
          dl = shfl_i128(round53(S + dl) - S, fl);
          start = fl + 1;
          ++events;
        }
        V = shfl_i128(S, 31);
      }
      if (tid == 0) s_delta = dl;
    }
    __syncthreads();
    delta = s_delta;
    cur = f + 1;
    ++walked;
  }
  if (tid == 0) {
    atomicMax(&st->rounds, (uint32_t)walked + 1u);
    atomicAdd(&st->events, (uint32_t)events);
    if (give_up) {
      st->need_chain = 1u;
    } else {
      const double acc = f96_to_double(row_total + delta);
      mean_out[c] = total ? __double2float_rn(__ddiv_rn(acc, (double)total)) : 0.0f;
      if (acc_out) acc_out[c] = acc;
    }
  }
}

// The literal chain (fallback and test reference): 4 CTAs x 32 channels, one
// thread per channel; the loads of the next 32 descriptors are in flight
// while the current 32 dependent DADDs issue, with an L2 prefetch stream 8
// batches ahead.
constexpr int kChainBatch = 32;

__global__ void __launch_bounds__(32, 1) mean_chain_kernel(const ImgDev* __restrict__ imgs, int n_imgs,
                                                           const uint32_t* gate, float* __restrict__ mean_out,
                                                           double* __restrict__ acc_out) {
  if (gated_off(gate)) return;
  const int lane = threadIdx.x;
  const int c = blockIdx.x * 32 + lane;
  double acc = 0.0;
  unsigned long long total = 0;
  for (int im = 0; im < n_imgs; ++im) {
    const uint32_t n = imgs[im].n;
    total += n;
    const float* d = imgs[im].desc + c;
    const uint32_t nb = n / kChainBatch;
    float cur[kChainBatch], nxt[kChainBatch];
    if (nb) {
#pragma unroll
      for (int r = 0; r < kChainBatch; ++r) cur[r] = __ldcg(d + (size_t)r * kDim);
    }
    for (uint32_t b = 0; b < nb; ++b) {
      const size_t row = (size_t)(b + 1) * kChainBatch;
      if (b + 1 < nb) {
#pragma unroll
        for (int r = 0; r < kChainBatch; ++r) nxt[r] = __ldcg(d + (row + r) * kDim);
      }
      const size_t pf = row + 8 * kChainBatch + lane;
      if (pf < n) asm volatile("prefetch.global.L2 [%0];" ::"l"(imgs[im].desc + pf * kDim + blockIdx.x * 32));
#pragma unroll
      for (int r = 0; r < kChainBatch; ++r) acc = __dadd_rn(acc, (double)cur[r]);
#pragma unroll
      for (int r = 0; r < kChainBatch; ++r) cur[r] = nxt[r];
    }
    for (uint32_t i = nb * kChainBatch; i < n; ++i) acc = __dadd_rn(acc, (double)__ldcg(d + (size_t)i * kDim));
  }
  mean_out[c] = total ? __double2float_rn(__ddiv_rn(acc, (double)total)) : 0.0f;
  if (acc_out) acc_out[c] = acc;
}

// ---------------------------------------------------------------------------
// K2: projections, split into a mean-independent GEMM and a per-row certify.
//
//   project_kernel  per image, once per residency (right after its upload,
//                   overlapping the next uploads): D[i][p] = fl32(d_i . p)
//                   (packed FFMA2, one FMA chain over c = 0..127 in order) and
//                   ||d_i||_2 rounded up.  Persistent, TMA-fed: a CTA keeps
//                   its plane chunk in shared memory and walks descriptor
//                   tiles whose rows arrive by cp.async.bulk (528-byte smem
//                   stride, conflict-free LDS.128) into a double buffer.
//   codes_kernel    per row: s32 = fl32(D[i][p] - fl32(m . p)) and the sign
//                   certificate below; packs bucket ids and fine words.
//
// Certificate: with u = 2^-24, |fl(d.p) - d.p| <= gamma_128 ||d|| ||p||,
// |fl(m.p) - m.p| <= gamma_128 ||m|| ||p|| and the subtraction adds
// u(||d|| + ||m||)||p||, so |s32 - s_exact| <= gamma_130 (||d|| + ||m||) ||p||
// <= 8e-6 (||d|| + ||m||) ||p|| (Cauchy-Schwarz, norms rounded up), where
// s_exact = sum_c (d_c - m_c) p_c; the reference's FP64 value
// (hashmatch.cpp:27-33) is within 1.5e-14 ||d - m|| ||p|| of it.  So
// s32 > B => bit 1, s32 < -B => bit 0; anything in [-B, B] goes to the FP64
// fixup list (recomputed in the reference's order).
// ---------------------------------------------------------------------------
constexpr int kAStride = 132;
constexpr float kDotBound = 8.0e-6f;
constexpr float kDotBoundAbs = 1.0e-37f;

__device__ __forceinline__ uint64_t extract_bits(const uint32_t* w, int start, int len) {
  const int wi = start >> 5, sh = start & 31;
  const uint64_t lo = (uint64_t)w[wi] | ((uint64_t)w[wi + 1] << 32);
  const uint64_t hi = w[wi + 2];
  uint64_t v = (lo >> sh) | (sh ? (hi << (64 - sh)) : 0ull);
  return len >= 64 ? v : (v & ((1ull << len) - 1ull));
}

constexpr int kTileStride = kAStride;  // floats per staged row (528 B: conflict-free LDS.128)

__device__ __forceinline__ uint32_t cvta_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Tiles of the launch: tile_img == nullptr means one image (`one`), tile t =
// its descriptors [128t, 128t+128); otherwise the (image, start) lists.
struct ProjJob {
  const ImgDev* imgs;
  const uint32_t* tile_img;
  const uint32_t* tile_start;
  int n_tiles;
  ImgDev one;
};

__device__ __forceinline__ void job_tile(const ProjJob& j, int t, ImgDev& im, uint32_t& i0) {
  if (j.tile_img) {
    im = j.imgs[j.tile_img[t]];
    i0 = j.tile_start[t];
  } else {
    im = j.one;
    i0 = (uint32_t)t * kCodesTile;
  }
}

__global__ void __launch_bounds__(512, 1) project_kernel(HashDev h, ProjJob job, int pstride) {
  extern __shared__ __align__(128) float smem_f[];
  float* sT = smem_f;                                  // [2][128][132] staged tiles
  float* sP = sT + 2 * kCodesTile * kTileStride;       // [128][pstride]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + kDim * pstride);  // [2]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int p0 = blockIdx.y * kPlaneChunk;
  const int np = min(kPlaneChunk, h.n_planes - p0);
  const int n_groups = (np + 11) / 12;  // warps with planes to project
  const bool norms = blockIdx.y == 0;

  // stage tile t's rows into buffer k (warp 0)
  auto issue = [&](int t, int k) {
    ImgDev im;
    uint32_t i0;
    job_tile(job, t, im, i0);
    const int nd = min(kCodesTile, (int)(im.n - i0));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(cvta_smem(bars + k)),
                   "r"((uint32_t)nd * 512u)
                   : "memory");
    __syncwarp();
    for (int r = lane; r < nd; r += 32)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
              cvta_smem(sT + ((size_t)k * kCodesTile + r) * kTileStride)),
          "l"(im.desc + (size_t)(i0 + r) * kDim), "r"(cvta_smem(bars + k))
          : "memory");
  };

  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cvta_smem(bars + 0)) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cvta_smem(bars + 1)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if ((int)blockIdx.x < job.n_tiles) issue(blockIdx.x, 0);
    if ((int)(blockIdx.x + gridDim.x) < job.n_tiles) issue(blockIdx.x + gridDim.x, 1);
  }
  // planes chunk -> smem (row c: planes p0 .. p0+pstride; planes_t is zero
  // padded to a multiple of kPlaneChunk, pstride is a multiple of 4)
  {
    const int q4 = pstride / 4;
    for (int e = tid; e < kDim * q4; e += blockDim.x) {
      const int c = e / q4, q = e - c * q4;
      reinterpret_cast<float4*>(sP + c * pstride)[q] =
          __ldg(reinterpret_cast<const float4*>(h.planes_t + (size_t)c * h.n_planes_pad + p0) + q);
    }
  }
  __syncthreads();

  uint32_t ph0 = 0, ph1 = 0;
  int k = 0;
  for (int t = blockIdx.x; t < job.n_tiles; t += gridDim.x, k ^= 1) {
    ImgDev im;
    uint32_t i0;
    job_tile(job, t, im, i0);
    const int nd = min(kCodesTile, (int)(im.n - i0));
    const float* sA = sT + (size_t)k * kCodesTile * kTileStride;
    {
      const uint32_t par = k ? ph1 : ph0;
      const uint32_t a = cvta_smem(bars + k);
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(a), "r"(par)
            : "memory");
      }
      if (k) ph1 ^= 1u;
      else ph0 ^= 1u;
    }
    if (norms) {  // ||d||_2 rounded up: thread (row, quarter) covers 32 floats
      const int r = tid >> 2, qq = tid & 3;
      const float4* row = reinterpret_cast<const float4*>(sA + r * kTileStride + qq * 32);
      float ss = 0.f;
      if (r < nd) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 v = row[i];
          ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
        }
      }
      ss += __shfl_xor_sync(kFull, ss, 1);
      ss += __shfl_xor_sync(kFull, ss, 2);
      if (qq == 0 && r < nd) im.dnorm[i0 + r] = sqrtf(ss) * 1.00001f;
    }
    const int pg = warp;  // plane groups of 12 (warp 15 idles: 180 = 15 x 12)
    if (pg < n_groups) {
      // packed FP32x2 FMAs (FFMA2, the descriptor value broadcast to both
      // halves): plane pair jp of row r accumulates in acc[r][jp]; every
      // output is one FP32 FMA chain over c = 0..127 in order
      float2 acc[4][6];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int j = 0; j < 6; ++j) acc[r][j] = make_float2(0.f, 0.f);
#pragma unroll 2
      for (int c4 = 0; c4 < kDim / 4; ++c4) {
        float4 a[4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
          a[r] = *reinterpret_cast<const float4*>(sA + (r * 32 + lane) * kTileStride + c4 * 4);
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const float* prow = sP + (c4 * 4 + cc) * pstride + pg * 12;
          const float4 q0 = *reinterpret_cast<const float4*>(prow);
          const float4 q1 = *reinterpret_cast<const float4*>(prow + 4);
          const float4 q2 = *reinterpret_cast<const float4*>(prow + 8);
          const float2 pv[6] = {make_float2(q0.x, q0.y), make_float2(q0.z, q0.w), make_float2(q1.x, q1.y),
                                make_float2(q1.z, q1.w), make_float2(q2.x, q2.y), make_float2(q2.z, q2.w)};
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const float av = cc == 0 ? a[r].x : cc == 1 ? a[r].y : cc == 2 ? a[r].z : a[r].w;
#pragma unroll
            for (int j = 0; j < 6; ++j) acc[r][j] = __ffma2_rn(make_float2(av, av), pv[j], acc[r][j]);
          }
        }
      }
      // D[i][p0 + 12pg + j]
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int i = r * 32 + lane;
        if (i < nd) {
          float* out = im.proj + (size_t)(i0 + i) * h.proj_stride + p0 + pg * 12;
#pragma unroll
          for (int j = 0; j < 6; ++j)
            if (pg * 12 + 2 * j + 1 < np) *reinterpret_cast<float2*>(out + 2 * j) = acc[r][j];
            else if (pg * 12 + 2 * j < np) out[2 * j] = acc[r][j].x;
        }
      }
    }
    __syncthreads();  // the tile is consumed: its buffer takes the next-but-one tile
    if (warp == 0 && t + 2 * (int)gridDim.x < job.n_tiles) issue(t + 2 * gridDim.x, k);
  }
}

// ---------------------------------------------------------------------------
// K2 on the 5th-gen tensor cores (default when n_planes <= 192): the same
// mean-independent projections D[i][p] ~ d_i . p, computed EXACTLY in integer
// arithmetic on quantised operands, so the certificate keeps a rigorous bound.
//   * every descriptor row and every plane is scaled by its own power of two
//     (2^e > max|x|) and rounded to a 22-bit integer X = rint(x 2^(22-e));
//     X is split into balanced base-256 digits X = X2 2^16 + X1 2^8 + X0,
//     |Xk| <= 128 (int8);
//   * tcgen05.mma kind::i8 (s8 x s8 -> s32, M=128 rows x N planes, K=128
//     channels in 4 steps of 32) accumulates the 9 digit products into 5 TMEM
//     accumulators by digit weight s = k + l (|acc_s| < 2^21: no overflow);
//   * the epilogue (tcgen05.ld) forms sum_s acc_s 2^(8s) in int64 (< 2^53,
//     exact in FP64), scales by 2^(e+f-44) and rounds once to FP32.
// Error (Cauchy-Schwarz, |x - X 2^(e-22)| <= 2^(e-23) <= 2^-22 max|x|):
// |D - d.p| <= 2^-22 sqrt(128) (2 + 1e-6) ||d|| ||p|| + 2^-24 |D|
//           <= 5.5e-6 ||d|| ||p|| < gamma_128 ||d|| ||p||,
// inside the bound the codes certificate assumes for fl32(d.p) (K2 above).
// Rows with a non-finite value get NaN (-> FP64 fixup, as the FP32 chain
// would); ||d|| is computed on the 2^-e scaled row (no underflow), rounded up.
// Operands live in shared memory in the canonical K-major 128-byte-swizzle
// layout (8-row x 128 B atoms, 16-byte chunk j of row r stored at chunk
// j ^ (r & 7)); the planes' digit image is prepared once per context by the
// host (bmg_api.cpp build_hash) in exactly that layout.
// ---------------------------------------------------------------------------
#ifndef BMG_TC_THREADS
#define BMG_TC_THREADS 512
#endif
constexpr int kTcThreads = BMG_TC_THREADS;  // 256 or 512
constexpr int kTcParts = kTcThreads / 128;  // threads per tile row (quantise), warps per TMEM lane quadrant
constexpr int kTcRows = 128;                 // UMMA M
constexpr int kTcDigitBytes = kTcRows * 128; // one digit plane of the A tile
constexpr uint32_t kTcTmemCols = 512;

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  // SM100 shared-memory matrix descriptor: start address >> 4 [0,14),
  // leading byte offset (unused for swizzled K-major, 1) [16,30), stride
  // byte offset 1024 >> 4 [32,46), version 1 [46,48), SWIZZLE_128B (2) [61,64)
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ uint32_t umma_idesc_i8(int n) {
  // kind::i8: D s32 (2) [4,6), A s8 (1) [7,10), B s8 (1) [10,13), both
  // K-major, N >> 3 [17,23), M >> 4 [24,29)
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kTcRows >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}

// balanced base-256 digits of |x| <= 2^22
__device__ __forceinline__ void digits3(int x, int& d0, int& d1, int& d2) {
  d0 = (int)(int8_t)(x & 0xff);
  x = (x - d0) >> 8;
  d1 = (int)(int8_t)(x & 0xff);
  d2 = (x - d1) >> 8;
}

__global__ void __launch_bounds__(kTcThreads, 1) project_tc_kernel(HashDev h, ProjJob job) {
  extern __shared__ unsigned char smem_raw[];
  // 1024-aligned operand region (SWIZZLE_128B atoms)
  const uint32_t raw = cvta_smem(smem_raw);
  unsigned char* base = smem_raw + ((1024u - (raw & 1023u)) & 1023u);
  unsigned char* sA = base;                                  // [3][128 rows][128 B]
  unsigned char* sB = sA + 3 * kTcDigitBytes;                // [3][npad rows][128 B]
  const int npad = h.tc_npad;
  float* sRaw = reinterpret_cast<float*>(sB + 3 * npad * 128);  // [128][128] the next tile's rows (bulk copy)
  int* sExp = reinterpret_cast<int*>(sRaw + kTcRows * kDim);    // [128] row exponents (INT_MIN: non-finite)
  int* sF = sExp + kTcRows;                                     // [npad] plane exponents
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sF + ((npad + 1) & ~1));  // [3]: MMA done, raw tile, planes
  uint32_t* sTmem = reinterpret_cast<uint32_t*>(mbar + 3);
  // the row-mean tile statistics' half-tile exchange (16-byte aligned)
  TileStatsSmem<kTcParts>& sStats = *reinterpret_cast<TileStatsSmem<kTcParts>*>(
      (reinterpret_cast<uintptr_t>(sTmem + 1) + 15) & ~static_cast<uintptr_t>(15));

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // thread 0: tile t's rows (contiguous, nd x 512 B) -> sRaw
  auto issue_raw = [&](int t) {
    ImgDev im;
    uint32_t i0;
    job_tile(job, t, im, i0);
    const uint32_t bytes = (uint32_t)min(kTcRows, (int)(im.n - i0)) * 512u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(cvta_smem(mbar + 1)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            cvta_smem(sRaw)),
        "l"(im.desc + (size_t)i0 * kDim), "r"(bytes), "r"(cvta_smem(mbar + 1))
        : "memory");
  };
  auto wait_bar = [&](uint64_t* bar, uint32_t par) {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(cvta_smem(bar)), "r"(par)
          : "memory");
    }
  };
  if (tid == 0) {
    for (int q = 0; q < 3; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cvta_smem(mbar + q)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the planes' digit image (prepared once per context) and the first tile
    const uint32_t bbytes = (uint32_t)(3 * npad * 128);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(cvta_smem(mbar + 2)), "r"(bbytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            cvta_smem(sB)),
        "l"(h.tc_b), "r"(bbytes), "r"(cvta_smem(mbar + 2))
        : "memory");
    if ((int)blockIdx.x < job.n_tiles) issue_raw(blockIdx.x);
  }
  for (int i = tid; i < npad; i += kTcThreads) sF[i] = __ldg(h.tc_fexp + i);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(cvta_smem(sTmem)),
                 "n"(kTcTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *sTmem;
  uint32_t phase = 0, raw_phase = 0;
  const int n_pass = h.tc_pass0 < npad ? 2 : 1;
  if (tid == 0) wait_bar(mbar + 2, 0);  // the MMA issuer needs the planes

  for (int t = blockIdx.x; t < job.n_tiles; t += gridDim.x) {
    ImgDev im;
    uint32_t i0;
    job_tile(job, t, im, i0);
    const int nd = min(kTcRows, (int)(im.n - i0));
    wait_bar(mbar + 1, raw_phase);
    raw_phase ^= 1u;
    // ---- quantise from the staged rows: kTcParts threads per row (128 /
    // kTcParts channels each); float4 j of a part is read in a per-thread
    // rotation (the 8 threads of a quarter warp hit distinct 16-byte banks)
    {
      constexpr int kNf = 32 / kTcParts;  // float4s per thread
      const int r = tid / kTcParts, part = tid % kTcParts;
      const int rot = (r * kTcParts + part) & (kNf - 1);
      const float4* row = reinterpret_cast<const float4*>(sRaw + r * kDim) + part * kNf;
      float mx = 0.f;
      bool finite = true;
      if (r < nd) {
#pragma unroll
        for (int j = 0; j < kNf; ++j) {
          const float4 v = row[(j + rot) & (kNf - 1)];
          mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
          finite &= isfinite(v.x) & isfinite(v.y) & isfinite(v.z) & isfinite(v.w);
        }
      }
#pragma unroll
      for (int o = 1; o < kTcParts; o <<= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
        finite = __shfl_xor_sync(kFull, (int)finite, o) != 0 && finite;
      }
      int e = 0;
      if (mx > 0.f && finite) frexpf(mx, &e);  // 2^(e-1) <= max < 2^e
      const float sc = finite ? ldexpf(1.f, 22 - e) : 0.f;
      const float sn = finite ? ldexpf(1.f, -e) : 0.f;
      float ss = 0.f;
      const uint32_t rbase = (uint32_t)(r >> 3) * 1024u + (uint32_t)(r & 7) * 128u;
#pragma unroll
      for (int j = 0; j < kNf; ++j) {
        const int f4 = (j + rot) & (kNf - 1);  // channels part * 128 / kTcParts + 4 f4 ..
        const float4 v = r < nd ? row[f4] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float vv[4] = {v.x, v.y, v.z, v.w};
        uint32_t b0 = 0, b1 = 0, b2 = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float ys = vv[u] * sn;
          ss = fmaf(ys, ys, ss);
          int d0, d1, d2;
          digits3(__float2int_rn(vv[u] * sc), d0, d1, d2);
          b0 |= (uint32_t)(d0 & 0xff) << (8 * u);
          b1 |= (uint32_t)(d1 & 0xff) << (8 * u);
          b2 |= (uint32_t)(d2 & 0xff) << (8 * u);
        }
        // channel c = part * 128 / kTcParts + 4 f4: 16-byte chunk c / 16, byte c % 16
        const int chunk = part * (8 / kTcParts) + (f4 >> 2);
        const uint32_t off = rbase + (uint32_t)((chunk ^ (r & 7)) * 16 + (f4 & 3) * 4);
        *reinterpret_cast<uint32_t*>(sA + off) = b0;
        *reinterpret_cast<uint32_t*>(sA + kTcDigitBytes + off) = b1;
        *reinterpret_cast<uint32_t*>(sA + 2 * kTcDigitBytes + off) = b2;
      }
#pragma unroll
      for (int o = 1; o < kTcParts; o <<= 1) ss += __shfl_xor_sync(kFull, ss, o);
      if (part == 0) {
        sExp[r] = finite ? e : INT_MIN;
        // ||d||_2 rounded up, from the 2^-e scaled row
        if (r < nd) im.dnorm[i0 + r] = finite ? ldexpf(sqrtf(ss), e) * 1.00001f : __int_as_float(0x7f800000);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    auto issue_mma = [&](int pass) {
      const int p0 = pass ? h.tc_pass0 : 0;
      const int np = pass ? npad - h.tc_pass0 : min(h.tc_pass0, npad);
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t idesc = umma_idesc_i8(np);
        const uint32_t a0 = cvta_smem(sA), b0 = cvta_smem(sB) + (uint32_t)(p0 >> 3) * 1024u;
#pragma unroll
        for (int sw = 0; sw < 5; ++sw) {           // digit weight s = k + l
          bool first = true;
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const int l = sw - k;
            if (l < 0 || l > 2) continue;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {        // K = 128 channels in steps of 32 bytes
              const uint64_t da = umma_desc_sw128(a0 + (uint32_t)k * kTcDigitBytes + kk * 32);
              const uint64_t db = umma_desc_sw128(b0 + (uint32_t)(l * npad * 128) + kk * 32);
              umma_i8(tmem + (uint32_t)(sw * np), da, db, idesc, first ? 0u : 1u);
              first = false;
            }
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         cvta_smem(mbar))
                     : "memory");
      }
    };
    issue_mma(0);
    // while the first pass's MMAs run: the row-mean tile statistics (K1)
    // from the same staged rows, so the row's mean only resolves them
    // (uniform branch: one image per tile)
    if (im.tsum) {
      tile_stats(im, i0 / kCodesTile, nd, sStats, [&](int r, int c) { return sRaw[r * kDim + c]; });
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
    }
    // the staged rows are consumed: stream the next tile in under this one's
    // MMAs and epilogue
    if (tid == 0 && t + (int)gridDim.x < job.n_tiles) issue_raw(t + gridDim.x);

    for (int pass = 0; pass < n_pass; ++pass) {
      const int p0 = pass ? h.tc_pass0 : 0;
      const int np = pass ? npad - h.tc_pass0 : min(h.tc_pass0, npad);
      if (pass) issue_mma(pass);
      // wait for the accumulators
      {
        uint32_t done = 0;
        while (!done) {
          asm volatile(
              "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
              : "=r"(done)
              : "r"(cvta_smem(mbar)), "r"(phase)
              : "memory");
        }
        phase ^= 1u;
      }
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // ---- epilogue: warp w reads TMEM lanes 32(w&3).. (= tile rows) and
      // every kTcParts-th group of 8 columns of the pass's planes from (w >> 2)
      {
        const int rg = warp & 3, ch = warp >> 2;
        const int r = rg * 32 + lane;
        const int ex = sExp[r];
        const uint32_t tl = tmem + ((uint32_t)(rg * 32) << 16);
        for (int c = 8 * ch; c < np; c += 8 * kTcParts) {
          int32_t acc[5][8];
#pragma unroll
          for (int sw = 0; sw < 5; ++sw) tmem_ld8(tl + (uint32_t)(sw * np + c), acc[sw]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          float out[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const long long v = (long long)acc[0][u] + ((long long)acc[1][u] << 8) + ((long long)acc[2][u] << 16) +
                                ((long long)acc[3][u] << 24) + ((long long)acc[4][u] << 32);
            const int pe = ex + sF[p0 + c + u] - 44;
            const double sc = __longlong_as_double((long long)(1023 + max(-1022, min(1023, pe))) << 52);
            out[u] = ex == INT_MIN ? __int_as_float(0x7fc00000) : __double2float_rn((double)v * sc);
          }
          if (r < nd) {
            float* dst = im.proj + (size_t)(i0 + r) * h.proj_stride + p0 + c;
            const int valid = min(8, h.n_planes - (p0 + c));
            if (valid == 8) {
              reinterpret_cast<float4*>(dst)[0] = make_float4(out[0], out[1], out[2], out[3]);
              reinterpret_cast<float4*>(dst)[1] = make_float4(out[4], out[5], out[6], out[7]);
            } else {
#pragma unroll
              for (int u = 0; u < 8; ++u)
                if (u < valid) dst[u] = out[u];
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
    }
  }
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTcTmemCols));
}

// Per row: mproj[p] = fl32(m . p) as one FP32 FMA chain per plane (the
// certificate's model), mproj[n_planes] = ||m||_2 rounded up.
__global__ void __launch_bounds__(256) mproj_kernel(HashDev h, const float* __restrict__ mean,
                                                    float* __restrict__ mproj) {
  __shared__ float sm[kDim];
  const int tid = threadIdx.x;
  if (tid < kDim) sm[tid] = mean[tid];
  __syncthreads();
  for (int p = blockIdx.x * blockDim.x + tid; p < h.n_planes; p += gridDim.x * blockDim.x) {
    const float* pp = h.planes + (size_t)p * kDim;
    float acc = 0.f;
#pragma unroll 8
    for (int c = 0; c < kDim; ++c) acc = fmaf(sm[c], __ldg(pp + c), acc);
    mproj[p] = acc;
  }
  if (blockIdx.x == 0 && tid < 32) {
    float ss = 0.f;
    for (int c = tid; c < kDim; c += 32) ss = fmaf(sm[c], sm[c], ss);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(kFull, ss, o);
    if (tid == 0) mproj[h.n_planes] = sqrtf(ss) * 1.00001f;
  }
}

// Per row: thread (descriptor i of the tile, plane word w) certifies planes
// 32w .. 32w+31 from D and the row's m.p; words of a descriptor meet in a
// shared-memory mask that is then cut into bucket ids and fine words.
constexpr int kCodesThreads = 256;

__global__ void __launch_bounds__(kCodesThreads)
    codes_kernel(HashDev h, const ImgDev* __restrict__ imgs, const uint32_t* __restrict__ tile_img,
                 const uint32_t* __restrict__ tile_start, const float* __restrict__ mproj,
                 Fixup* __restrict__ fix, uint32_t* __restrict__ fix_count, uint32_t fix_cap,
                 uint32_t* __restrict__ overflow) {
  extern __shared__ __align__(16) uint32_t smem_u[];
  const int n_pw = (h.n_planes + 31) / 32, mw = n_pw + 2;  // mask words (+2 guards)
  uint32_t* sMask = smem_u;                                        // [128][mw]
  float* sMp = reinterpret_cast<float*>(sMask + kCodesTile * mw);  // [n_planes] m . p, then ||m||
  const int tid = threadIdx.x;
  const uint32_t img = tile_img[blockIdx.x];
  const ImgDev im = imgs[img];
  const uint32_t i0 = tile_start[blockIdx.x];
  const int nd = min(kCodesTile, (int)(im.n - i0));
  for (int p = tid; p <= h.n_planes; p += blockDim.x) sMp[p] = __ldg(mproj + p);
  for (int e = tid; e < kCodesTile * mw; e += blockDim.x) sMask[e] = 0u;
  __syncthreads();

  const float mn = sMp[h.n_planes];
  for (int e = tid; e < nd * n_pw; e += blockDim.x) {
    const int i = e % nd, w = e / nd;
    const float* drow = im.proj + (size_t)(i0 + i) * h.proj_stride + 32 * w;
    const float bn = kDotBound * (__ldg(im.dnorm + i0 + i) + mn);
    const int pn = min(32, h.n_planes - 32 * w);
    uint32_t bits = 0;
    for (int j0 = 0; j0 < pn; j0 += 4) {
      float4 dv;
      if (j0 + 3 < pn) {
        dv = __ldg(reinterpret_cast<const float4*>(drow + j0));
      } else {
        dv.x = __ldg(drow + j0);
        dv.y = j0 + 1 < pn ? __ldg(drow + j0 + 1) : 0.f;
        dv.z = j0 + 2 < pn ? __ldg(drow + j0 + 2) : 0.f;
        dv.w = 0.f;
      }
      const float dd[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = j0 + q, p = 32 * w + j;
        if (j < pn) {
          const float sv = dd[q] - sMp[p];
          const float B = fmaf(bn, __ldg(h.plane_norm + p), kDotBoundAbs);
          if (sv > B) {
            bits |= 1u << j;
          } else if (!(sv < -B)) {
            const uint32_t slot = atomicAdd(fix_count, 1u);
            if (slot < fix_cap) {
              Fixup f;
              f.img = img;
              f.desc = i0 + i;
              f.plane = p;
              f.pad = 0;
              fix[slot] = f;
            } else {
              atomicOr(overflow + img, 1u);
            }
          }
        }
      }
    }
    sMask[i * mw + w] = bits;
  }
  __syncthreads();

  // assemble coarse bucket ids and fine words
  const int L = h.tables, m = h.coarse_bits, fb = h.fine_bits, coarse_planes = L * m;
  const int n_words = L + h.fwp;
  for (int e = tid; e < nd * n_words; e += blockDim.x) {
    const int i = e / n_words, wd = e % n_words;
    const uint32_t* mk = sMask + i * mw;
    const size_t gi = i0 + i;
    if (wd < L) {
      im.coarse[gi * L + wd] = (uint32_t)extract_bits(mk, wd * m, m);
    } else {
      const int fwi = wd - L;
      const int b0 = coarse_planes + 64 * fwi;
      const int len = min(64, coarse_planes + fb - b0);
      im.fine[gi * h.fwp + fwi] = len > 0 ? extract_bits(mk, b0, len) : 0ull;
    }
  }
}

// codes_kernel with the tile's projections streamed into shared memory by
// one bulk copy per tile (the tile's rows of ImgDev::proj are contiguous),
// double-buffered, persistent over the row's tiles; one warp per descriptor,
// lane j certifies planes j, j+32, .. and the plane word is a warp ballot.
// Same arithmetic, bits and fixup list as codes_kernel (used when two tile
// buffers fit: proj_stride <= 192).
constexpr int kCodesTmaThreads = 1024;
__global__ void __launch_bounds__(kCodesTmaThreads, 1)
    codes_tma_kernel(HashDev h, const ImgDev* __restrict__ imgs, const uint32_t* __restrict__ tile_img,
                     const uint32_t* __restrict__ tile_start, int n_tiles, const float* __restrict__ mproj,
                     Fixup* __restrict__ fix, uint32_t* __restrict__ fix_count, uint32_t fix_cap,
                     uint32_t* __restrict__ overflow) {
  extern __shared__ __align__(128) unsigned char smem_c[];
  const int n_pw = (h.n_planes + 31) / 32, mw = n_pw + 2;
  const int ps = h.proj_stride;
  float* sD = reinterpret_cast<float*>(smem_c);                         // [2][128][ps]
  uint32_t* sMask = reinterpret_cast<uint32_t*>(sD + 2 * kCodesTile * ps);  // [128][mw]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sMask + ((kCodesTile * mw + 1) & ~1));  // [2], 8-byte aligned
  float* sN = reinterpret_cast<float*>(bars + 2);                       // [2][128] tile norms
  float* sMp = sN + 2 * kCodesTile;                                     // [n_planes + 1]
  float* sPn = sMp + h.n_planes + 1;                                    // [n_planes]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kWarps = kCodesTmaThreads / 32;

  auto issue = [&](int t, int k) {  // thread 0: tile t's projections -> buffer k
    const ImgDev im = imgs[tile_img[t]];
    const uint32_t i0 = tile_start[t];
    const uint32_t nd = min((uint32_t)kCodesTile, im.n - i0);
    const uint32_t bytes = nd * (uint32_t)ps * 4u;
    const uint32_t nbytes = (nd * 4u + 15u) & ~15u;  // the norms (ImgDev::dnorm is 16-byte aligned per tile)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(cvta_smem(bars + k)),
                 "r"(bytes + nbytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            cvta_smem(sD + (size_t)k * kCodesTile * ps)),
        "l"(im.proj + (size_t)i0 * ps), "r"(bytes), "r"(cvta_smem(bars + k))
        : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            cvta_smem(sN + k * kCodesTile)),
        "l"(im.dnorm + i0), "r"(nbytes), "r"(cvta_smem(bars + k))
        : "memory");
  };
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cvta_smem(bars + 0)) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cvta_smem(bars + 1)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int p = tid; p <= h.n_planes; p += blockDim.x) sMp[p] = __ldg(mproj + p);
  for (int p = tid; p < h.n_planes; p += blockDim.x) sPn[p] = __ldg(h.plane_norm + p);
  __syncthreads();
  if (tid == 0) {
    if ((int)blockIdx.x < n_tiles) issue(blockIdx.x, 0);
    if ((int)(blockIdx.x + gridDim.x) < n_tiles) issue(blockIdx.x + gridDim.x, 1);
  }
  const float mn = sMp[h.n_planes];
  const int L = h.tables, m = h.coarse_bits, fb = h.fine_bits, coarse_planes = L * m;
  const int n_words = L + h.fwp;
  uint32_t ph[2] = {0u, 0u};
  int k = 0;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, k ^= 1) {
    const uint32_t img = tile_img[t];
    const ImgDev im = imgs[img];
    const uint32_t i0 = tile_start[t];
    const int nd = min(kCodesTile, (int)(im.n - i0));
    {
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(cvta_smem(bars + k)), "r"(ph[k])
            : "memory");
      }
      ph[k] ^= 1u;
    }
    const float* D = sD + (size_t)k * kCodesTile * ps;
    for (int i = warp; i < nd; i += kWarps) {
      const float bn = kDotBound * (sN[k * kCodesTile + i] + mn);
      for (int w = 0; w < n_pw; ++w) {
        const int p = 32 * w + lane;
        bool bit = false;
        if (p < h.n_planes) {
          const float sv = D[i * ps + p] - sMp[p];
          const float B = fmaf(bn, sPn[p], kDotBoundAbs);
          bit = sv > B;
          if (!bit && !(sv < -B)) {
            const uint32_t slot = atomicAdd(fix_count, 1u);
            if (slot < fix_cap) {
              Fixup f;
              f.img = img;
              f.desc = i0 + i;
              f.plane = p;
              f.pad = 0;
              fix[slot] = f;
            } else {
              atomicOr(overflow + img, 1u);
            }
          }
        }
        const uint32_t word = __ballot_sync(kFull, bit);
        if (lane == 0) sMask[i * mw + w] = word;
      }
      if (lane < 2) sMask[i * mw + n_pw + lane] = 0u;  // guards
    }
    __syncthreads();  // masks complete; the D buffer is consumed
    if (tid == 0 && t + 2 * (int)gridDim.x < n_tiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(t + 2 * gridDim.x, k);
    }
    for (int e = tid; e < nd * n_words; e += blockDim.x) {
      const int i = e / n_words, wd = e % n_words;
      const uint32_t* mk = sMask + i * mw;
      const size_t gi = i0 + i;
      if (wd < L) {
        im.coarse[gi * L + wd] = (uint32_t)extract_bits(mk, wd * m, m);
      } else {
        const int fwi = wd - L;
        const int b0 = coarse_planes + 64 * fwi;
        const int len = min(64, coarse_planes + fb - b0);
        im.fine[gi * h.fwp + fwi] = len > 0 ? extract_bits(mk, b0, len) : 0ull;
      }
    }
    __syncthreads();  // sMask reused by the next tile
  }
}

__device__ __forceinline__ double centered_dot_ref(const float* __restrict__ d,
                                                   const float* __restrict__ mean,
                                                   const float* __restrict__ p) {
  // hashmatch.cpp:27-33: s += ((double)d - (double)mean) * (double)p, no contraction
  double s = 0.0;
#pragma unroll 8
  for (int c = 0; c < kDim; ++c)
    s = __dadd_rn(s, __dmul_rn(__dsub_rn((double)d[c], (double)mean[c]), (double)p[c]));
  return s;
}

__device__ __forceinline__ void set_code_bit(const HashDev& h, const ImgDev& im, uint32_t desc,
                                             uint32_t plane) {
  const uint32_t cp = (uint32_t)(h.tables * h.coarse_bits);
  if (plane < cp) {
    const uint32_t t = plane / h.coarse_bits, b = plane % h.coarse_bits;
    atomicOr(im.coarse + (size_t)desc * h.tables + t, 1u << b);
  } else {
    const uint32_t f = plane - cp;
    atomicOr(reinterpret_cast<unsigned long long*>(im.fine + (size_t)desc * h.fwp + (f >> 6)),
             1ull << (f & 63));
  }
}

constexpr int kFixupThreads = 256;
__global__ void __launch_bounds__(kFixupThreads) codes_fixup_kernel(HashDev h, const ImgDev* __restrict__ imgs,
                                   const float* __restrict__ mean, const Fixup* __restrict__ fix,
                                   const uint32_t* __restrict__ fix_count, uint32_t fix_cap,
                                   unsigned long long* fixed_bits) {
  // one warp per ambiguous bit: lane l loads channels 4l..4l+3 of the
  // descriptor, mean and plane (coalesced rows) and forms the products
  // fl(fl(d - m) * p) in FP64 exactly as the reference does per channel; the
  // reference's sequential sum over c = 0..127 (hashmatch.cpp:27-33) is then
  // replayed in order by lane 0 from shared memory
  __shared__ double s_t[kFixupThreads / 32][kDim];
  const uint32_t n = min(*fix_count, fix_cap);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const float4 mv = __ldg(reinterpret_cast<const float4*>(mean) + lane);
  for (uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < n; e += (gridDim.x * blockDim.x) >> 5) {
    const Fixup f = fix[e];
    const ImgDev im = imgs[f.img];
    const float4 dv = __ldg(reinterpret_cast<const float4*>(im.desc + (size_t)f.desc * kDim) + lane);
    const float4 pv = __ldg(reinterpret_cast<const float4*>(h.planes + (size_t)f.plane * kDim) + lane);
    const float dd[4] = {dv.x, dv.y, dv.z, dv.w}, mm[4] = {mv.x, mv.y, mv.z, mv.w},
                pp[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)
      s_t[wib][4 * lane + j] = __dmul_rn(__dsub_rn((double)dd[j], (double)mm[j]), (double)pp[j]);
    __syncwarp();
    if (lane == 0) {
      double acc = 0.0;
#pragma unroll 16
      for (int c = 0; c < kDim; ++c) acc = __dadd_rn(acc, s_t[wib][c]);
      if (acc > 0.0) set_code_bit(h, im, f.desc, f.plane);
    }
    __syncwarp();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && fixed_bits) atomicAdd(fixed_bits, (unsigned long long)n);
}

// Fixup-list overflow (pathological inputs, e.g. thousands of descriptors
// equal to the mean): recompute every projection of the flagged images in
// FP64 and OR in the positive ones (certified 1-bits are already set).
__global__ void codes_overflow_kernel(HashDev h, const ImgDev* __restrict__ imgs, int n_imgs,
                                      const float* __restrict__ mean,
                                      const uint32_t* __restrict__ overflow) {
  for (int ii = 0; ii < n_imgs; ++ii) {
    if (!overflow[ii]) continue;
    const ImgDev im = imgs[ii];
    const uint64_t total = (uint64_t)im.n * h.n_planes;
    for (uint64_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
      const uint32_t desc = (uint32_t)(e / h.n_planes), plane = (uint32_t)(e % h.n_planes);
      const double s = centered_dot_ref(im.desc + (size_t)desc * kDim, mean,
                                        h.planes + (size_t)plane * kDim);
      if (s > 0.0) set_code_bit(h, im, desc, plane);
    }
  }
}

// ---------------------------------------------------------------------------
// K3: bucket index per (image, row): histogram -> per-table scan -> scatter.
// The order of train indices inside a bucket is irrelevant to the result:
// candidates are ranked by the unique key (hamming, train_idx).
// ---------------------------------------------------------------------------
__global__ void tables_hist_kernel(HashDev h, const ImgDev* __restrict__ imgs,
                                   const uint32_t* __restrict__ tile_img,
                                   const uint32_t* __restrict__ tile_start) {
  const ImgDev im = imgs[tile_img[blockIdx.x]];
  const uint32_t i = tile_start[blockIdx.x] + threadIdx.x;
  if (i >= im.n) return;
  for (int t = 0; t < h.tables; ++t) {
    const uint32_t b = im.coarse[(size_t)i * h.tables + t];
    atomicAdd(im.offsets + (size_t)t * (h.n_buckets + 1) + b + 1, 1u);
  }
}

__device__ __forceinline__ uint32_t block_incl_scan(uint32_t v, uint32_t* s_warp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) s_warp[warp] = v;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    s_warp[lane] = w;
  }
  __syncthreads();
  if (warp > 0) v += s_warp[warp - 1];
  __syncthreads();
  return v;
}

// Buckets are laid out padded to whole 8-entry chunks (kBucketPad; also
// 16-byte aligned slot runs for the TMA-staged matcher's bulk copies); pad
// entries hold train index kEmpty, which makes their match key kEmpty.  The
// last chunk of each table's slot range is an all-pad sentinel: walk lanes
// past the end of a query's union read it instead of testing bounds.
__global__ void __launch_bounds__(1024) tables_scan_kernel(HashDev h, const ImgDev* __restrict__ imgs) {
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_carry;
  const ImgDev im = imgs[blockIdx.x];
  const int t = blockIdx.y;
  uint32_t* off = im.offsets + (size_t)t * (h.n_buckets + 1);
  uint32_t* cur = im.cursor + (size_t)t * h.n_buckets;
  uint32_t* slots = im.slots + (size_t)t * im.ns;
  uint64_t* bfine = im.bfine + (size_t)t * im.ns * h.fwp;
  uint32_t carry = 0;
  for (int base = 0; base < h.n_buckets; base += blockDim.x) {
    const int b = base + threadIdx.x;
    const uint32_t v = b < h.n_buckets ? off[b + 1] : 0u;
    const uint32_t pv = (v + (uint32_t)h.bucket_pad - 1u) / (uint32_t)h.bucket_pad * (uint32_t)h.bucket_pad;
    const uint32_t incl = block_incl_scan(pv, s_warp) + carry;
    if (b < h.n_buckets) {
      off[b + 1] = incl;
      cur[b] = incl - pv;
      for (uint32_t k = incl - pv + v; k < incl; ++k) {
        slots[k] = kEmpty;
        for (int x = 0; x < h.fwp; ++x) bfine[(size_t)k * h.fwp + x] = 0ull;
      }
    }
    if (threadIdx.x == blockDim.x - 1) s_carry = incl;
    __syncthreads();
    carry = s_carry;
    __syncthreads();
  }
  if (threadIdx.x < kSentinel) {
    const uint32_t k = im.ns - kSentinel + threadIdx.x;
    slots[k] = kEmpty;
    for (int x = 0; x < h.fwp; ++x) bfine[(size_t)k * h.fwp + x] = 0ull;
  }
}

// One CTA per (image, table), counting sort in shared memory: histogram with
// shared atomics, the padded bucket scan (same layout as tables_scan_kernel:
// buckets padded to kBucketPad with pad entries, the sentinel chunk at the
// end), then the scatter with shared cursors.  Used for 2^m <= 4096 buckets;
// the three global-atomic kernels above remain for larger m.
constexpr int kTablesFusedMaxBuckets = 4096;
__global__ void __launch_bounds__(1024) tables_fused_kernel(HashDev h, const ImgDev* __restrict__ imgs) {
  extern __shared__ uint32_t s_cnt[];  // [n_buckets]: counts, then cursors
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_carry;
  const ImgDev im = imgs[blockIdx.x];
  const int t = blockIdx.y, L = h.tables, nb = h.n_buckets;
  uint32_t* off = im.offsets + (size_t)t * (nb + 1);
  uint32_t* slots = im.slots + (size_t)t * im.ns;
  uint64_t* bfine = im.bfine + (size_t)t * im.ns * h.fwp;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) s_cnt[b] = 0u;
  __syncthreads();
  // bucket ids are loaded kTblBatch per thread ahead of their shared
  // atomics (independent loads in flight instead of load -> atomic chains)
  constexpr int kTblBatch = 8;
  const uint32_t* ccol = im.coarse + t;
  for (uint32_t i0 = 0; i0 < im.n; i0 += kTblBatch * blockDim.x) {
    uint32_t bk[kTblBatch];
#pragma unroll
    for (int j = 0; j < kTblBatch; ++j) {
      const uint32_t i = i0 + j * blockDim.x + threadIdx.x;
      bk[j] = i < im.n ? __ldg(ccol + (size_t)i * L) : kEmpty;
    }
#pragma unroll
    for (int j = 0; j < kTblBatch; ++j)
      if (bk[j] != kEmpty) atomicAdd(s_cnt + bk[j], 1u);
  }
  __syncthreads();
  uint32_t carry = 0;
  if (threadIdx.x == 0) off[0] = 0u;
  for (int b0 = 0; b0 < nb; b0 += blockDim.x) {
    const int b = b0 + threadIdx.x;
    const uint32_t v = b < nb ? s_cnt[b] : 0u;
    const uint32_t pv = (v + (uint32_t)h.bucket_pad - 1u) / (uint32_t)h.bucket_pad * (uint32_t)h.bucket_pad;
    const uint32_t incl = block_incl_scan(pv, s_warp) + carry;
    if (b < nb) {
      off[b + 1] = incl;
      s_cnt[b] = incl - pv;  // cursor
      for (uint32_t k = incl - pv + v; k < incl; ++k) {
        slots[k] = kEmpty;
        for (int x = 0; x < h.fwp; ++x) bfine[(size_t)k * h.fwp + x] = 0ull;
      }
    }
    if (threadIdx.x == blockDim.x - 1) s_carry = incl;
    __syncthreads();
    carry = s_carry;
    __syncthreads();
  }
  if (threadIdx.x < kSentinel) {
    const uint32_t k = im.ns - kSentinel + threadIdx.x;
    slots[k] = kEmpty;
    for (int x = 0; x < h.fwp; ++x) bfine[(size_t)k * h.fwp + x] = 0ull;
  }
  for (uint32_t i0 = 0; i0 < im.n; i0 += kTblBatch * blockDim.x) {
    uint32_t bk[kTblBatch];
#pragma unroll
    for (int j = 0; j < kTblBatch; ++j) {
      const uint32_t i = i0 + j * blockDim.x + threadIdx.x;
      bk[j] = i < im.n ? __ldg(ccol + (size_t)i * L) : kEmpty;
    }
#pragma unroll
    for (int j = 0; j < kTblBatch; ++j) {
      if (bk[j] == kEmpty) continue;
      const uint32_t i = i0 + j * blockDim.x + threadIdx.x;
      const uint32_t pos = atomicAdd(s_cnt + bk[j], 1u);
      slots[pos] = i;
      if (h.fwp == 2) {
        reinterpret_cast<ulonglong2*>(bfine)[pos] = __ldg(reinterpret_cast<const ulonglong2*>(im.fine) + i);
      } else {
        for (int x = 0; x < h.fwp; ++x) bfine[(size_t)pos * h.fwp + x] = im.fine[(size_t)i * h.fwp + x];
      }
    }
  }
}

__global__ void tables_scatter_kernel(HashDev h, const ImgDev* __restrict__ imgs,
                                      const uint32_t* __restrict__ tile_img,
                                      const uint32_t* __restrict__ tile_start) {
  const ImgDev im = imgs[tile_img[blockIdx.x]];
  const uint32_t i = tile_start[blockIdx.x] + threadIdx.x;
  if (i >= im.n) return;
  for (int t = 0; t < h.tables; ++t) {
    const uint32_t b = im.coarse[(size_t)i * h.tables + t];
    const uint32_t pos = atomicAdd(im.cursor + (size_t)t * h.n_buckets + b, 1u);
    const size_t si = (size_t)t * im.ns + pos;
    im.slots[si] = i;
    // the fine code again in slot order: the matcher's candidate walk then
    // reads consecutive entries (coalesced) instead of gathering by index
    for (int x = 0; x < h.fwp; ++x) im.bfine[si * h.fwp + x] = im.fine[(size_t)i * h.fwp + x];
  }
}

// ---------------------------------------------------------------------------
// K4: the cascade.  CTA = (image pair, query range); one WARP per query.
//   1. the query's bucket union over the L tables (hashmatch.cpp:154-169):
//      table t contributes the bucket range [lo_t, lo_t + sz_t) of the train
//      image's bucket-ordered slot / fine-code arrays (written by the tables
//      scatter).  Buckets are padded to whole 8-entry chunks and the warp's
//      four 8-lane groups take four chunks per round, so a lane's entry is
//      chunk_base + (lane & 7): coalesced 128-byte code loads, no per-lane
//      table search or bounds test.  Chunk descriptors are built one per
//      lane (32 per page) and fetched per round with one shuffle; loads run
//      two rounds ahead;
//   2. per candidate: 128-bit Hamming via POPC and the unique key
//      (hamming << idx_bits | train_idx; the shift folded into IMADs).  Each
//      lane keeps its kLaneKeys (4) smallest keys (branch-free sorted
//      insert); the warp then pulls the K smallest out of the lanes' lists
//      with the single-instruction warp min (REDUX), lanes 0..7 taking the
//      pulls by a select on their lane bits.  Equal keys are the same train
//      index reached from several tables and are taken once -- the
//      reference's last_seen dedup + stable counting sort by (hamming, idx)
//      (:160-200).  A lane that dropped a key below the K-th pull kept 4
//      smaller keys, all of which the pulls take: a full lane that ends the
//      pulls empty sends the query to the exact path (sorted list over lanes
//      0..KM-1, REDUX-driven insertion; ~0.17% of queries);
//   3. re-rank (:196-208): lanes 4c..4c+3 hold candidate c; FP32 squared
//      distances (packed FFMA2) with a certified relative error <= 1e-5
//      decide the (dist, idx) argmin and the ratio test; uncertified queries
//      rerun the reference's sequential FP64 euclidean (:35-42)
//      lane-per-candidate.
// ---------------------------------------------------------------------------
constexpr int kMaxTables = 32;
// keys each lane keeps during the walk (K4 fast path); a query whose top 8
// crowd more than this into one lane reruns on the exact path (3 measured no
// faster: the walk is not bound by the sorted insert)
#ifndef BMG_LANE_KEYS
#define BMG_LANE_KEYS 4
#endif
constexpr int kLaneKeys = BMG_LANE_KEYS;
// rounds the candidate walk's loads run ahead of their use
#ifndef BMG_WALK_DEPTH
#define BMG_WALK_DEPTH 2
#endif
constexpr int kWalkDepth = BMG_WALK_DEPTH;

// FWP code words of one bucket-ordered entry (16-byte loads where possible)
template <int FWP>
__device__ __forceinline__ void load_code(const uint64_t* __restrict__ p, uint64_t (&c)[FWP]) {
  if constexpr (FWP % 2 == 0) {
#pragma unroll
    for (int x = 0; x < FWP / 2; ++x) {
      const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(p) + x);
      c[2 * x] = v.x;
      c[2 * x + 1] = v.y;
    }
  } else {
    c[0] = __ldg(p);
  }
}

template <int FWP>
__device__ __forceinline__ uint32_t hamming(const uint64_t (&q)[FWP], const uint64_t (&t)[FWP]) {
  uint32_t h = 0;
#pragma unroll
  for (int x = 0; x < FWP; ++x) h += __popcll(q[x] ^ t[x]);
  return h;
}

// Walks the union; round(key) is called by every lane once per round
// (warp-uniform trip count).  lo / sz: lane t < L holds table t's bucket range
// (a whole number of 8-entry chunks); other lanes hold zeros.
// key = hamming << ib | train_idx; pad entries carry idx kEmpty, so their key
// is kEmpty.  Chunk descriptors live in registers, one chunk per lane, and
// are fetched per round with one shuffle; loads run two rounds ahead.
template <int FWP, typename F>
__device__ __forceinline__ void walk_union(const ImgDev& T, int L, uint32_t lo, uint32_t sz, int ib,
                                           const uint64_t (&qc)[FWP], F&& round) {
  const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
  const uint32_t nch = sz >> 3;
  uint32_t cend = nch;  // inclusive scan of the chunk counts over tables
#pragma unroll
  for (int o = 1; o < kMaxTables; o <<= 1) {
    if (o < L) {  // warp-uniform
      const uint32_t y = __shfl_up_sync(kFull, cend, o);
      cend += lane >= o ? y : 0u;
    }
  }
  const uint32_t n_chunks = __shfl_sync(kFull, cend, L - 1);
  const uint32_t cstart = cend - nch;
  const uint32_t cend_s = lane < L ? cend : kEmpty;  // past the tables: never <= k
  const uint32_t sbase = (uint32_t)lane * T.ns + lo;
  const uint32_t sentinel = T.ns - kSentinel;  // all-pad chunk of table 0
  const uint32_t kmul = 1u << ib;
  for (uint32_t pg = 0; pg < n_chunks; pg += 32) {
    // lane j describes chunk pg + j: table = #tables ending at or before it
    // (binary search over the nondecreasing chunk ends, one shuffle a step)
    const uint32_t k = pg + lane;
    int t = 0;
    if (L > 8) {
      t += __shfl_sync(kFull, cend_s, 15) <= k ? 16 : 0;
      t += __shfl_sync(kFull, cend_s, t + 7) <= k ? 8 : 0;
    }
    t += __shfl_sync(kFull, cend_s, t + 3) <= k ? 4 : 0;
    t += __shfl_sync(kFull, cend_s, t + 1) <= k ? 2 : 0;
    t += __shfl_sync(kFull, cend_s, t) <= k ? 1 : 0;
    const uint32_t ts = __shfl_sync(kFull, cstart, t);
    const uint32_t tb = __shfl_sync(kFull, sbase, t);
    // chunks past the union read the sentinel: every load is in bounds and
    // every entry of a full chunk is used, so the loop has no bounds tests
    const uint32_t my_base = k < n_chunks ? tb + (k - ts) * 8u : sentinel;
    const uint32_t nr = (min(32u, n_chunks - pg) + 3u) >> 2;
    // source lane 4r + grp wraps past 31 only for rounds >= 8 >= nr, whose
    // loads are discarded
    auto fetch = [&](int kk, uint32_t& jo, uint64_t (&co)[FWP]) {
      const uint32_t si = __shfl_sync(kFull, my_base, kk) + (uint32_t)sub;
      jo = __ldg(T.slots + si);
      load_code<FWP>(T.bfine + (size_t)si * FWP, co);
    };
    // loads run kWalkDepth rounds ahead
    uint32_t jr[kWalkDepth];
    uint64_t cr[kWalkDepth][FWP];
#pragma unroll
    for (int d = 0; d < kWalkDepth; ++d) fetch(4 * d + grp, jr[d], cr[d]);
    for (uint32_t r = 0; r < nr; ++r) {
      uint32_t jn;
      uint64_t cn[FWP];
      fetch(4 * (int)(r + kWalkDepth) + grp, jn, cn);
      {
        uint32_t acc = 0;
#pragma unroll
        for (int x = 0; x < FWP; ++x) {
          const uint64_t d = qc[x] ^ cr[0][x];
          acc = __popc((uint32_t)d) * kmul + acc;
          acc = __popc((uint32_t)(d >> 32)) * kmul + acc;
        }
        round(acc | jr[0]);
      }
#pragma unroll
      for (int d = 0; d + 1 < kWalkDepth; ++d) {
        jr[d] = jr[d + 1];
#pragma unroll
        for (int x = 0; x < FWP; ++x) cr[d][x] = cr[d + 1][x];
      }
      jr[kWalkDepth - 1] = jn;
#pragma unroll
      for (int x = 0; x < FWP; ++x) cr[kWalkDepth - 1][x] = cn[x];
    }
  }
}

// Euclidean re-rank + ratio test of query q (hashmatch.cpp:196-208), warp-
// wide: lane r < kept holds the query's r-th key (hamming << ib | train idx,
// ascending).  Returns the matched train index or -1.
//   lanes hold dims 4l..4l+3 of the query and of every kept candidate; FP32
//   squared distances (packed FP32x2 ops) with a certified relative error
//   decide the (dist, idx) argmin and the ratio test; uncertified queries
//   rerun the reference's sequential FP64 euclidean (:35-42) lane-per-candidate.
template <int KM>
__device__ __forceinline__ int32_t rerank_query(const MatchLaunch& a, const ImgDev& Q, const ImgDev& T,
                                                uint32_t q, uint32_t lst, int kept, uint32_t idx_mask) {
  const int lane = threadIdx.x & 31;
  const float4* __restrict__ Qd = reinterpret_cast<const float4*>(Q.desc);
  const float4* __restrict__ Td = reinterpret_cast<const float4*>(T.desc);
  const double ratio = a.ratio;
  const float r2f = (float)(ratio * ratio);
  int32_t result = -1;
  if (kept == 1) {
    result = (int32_t)(__shfl_sync(kFull, lst, 0) & idx_mask);
  } else if (kept > 1) {
    const bool mine = lane < kept;
    const uint32_t my_idx = lst & idx_mask;
    float s_min, s_2;
    uint32_t i_min;
    if constexpr (KM == 8) {
      const int ck = lane >> 2, part = lane & 3;
      const uint32_t jk = __shfl_sync(kFull, my_idx, ck);
      const float2 neg1 = make_float2(-1.f, -1.f);
      // lane l holds dims 4l..4l+3 of the query and of every kept
      // candidate (one coalesced 512-byte row per candidate); a
      // transpose-reduce over lane bits 4, 3, 2 then two xor steps leave
      // candidate c's sum in lanes 4c..4c+3.  Depth <= 3 + 5 per sum:
      // relative error ~1e-6.
      const float4 qv = __ldg(Qd + (size_t)q * 32 + lane);
      float pt[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        pt[c] = 0.f;
        const uint32_t jc = __shfl_sync(kFull, my_idx, c);
        if (c < kept) {
          const float4 tv = __ldg(Td + (size_t)jc * 32 + lane);
          const float2 d0 = __ffma2_rn(make_float2(tv.x, tv.y), neg1, make_float2(qv.x, qv.y));
          const float2 d1 = __ffma2_rn(make_float2(tv.z, tv.w), neg1, make_float2(qv.z, qv.w));
          const float2 p2 = __ffma2_rn(d1, d1, __fmul2_rn(d0, d0));
          pt[c] = p2.x + p2.y;
        }
      }
#pragma unroll
      for (int st = 0; st < 3; ++st) {
        const int half = 4 >> st, msk = 16 >> st;
        const bool up = (lane & msk) != 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i < half) {
            const float send = up ? pt[i] : pt[i + half];
            const float keep = up ? pt[i + half] : pt[i];
            pt[i] = keep + __shfl_xor_sync(kFull, send, msk);
          }
        }
      }
      float s = pt[0];
      s += __shfl_xor_sync(kFull, s, 2);
      s += __shfl_xor_sync(kFull, s, 1);
      // squared distances are >= 0 (or NaN, caught by `finite`): their
      // bit patterns order like the values, so REDUX finds the (s, idx)
      // argmin and the runner-up
      const bool lead = part == 0 && ck < kept;
      const uint32_t sb = lead ? __float_as_uint(s) : kEmpty;
      const uint32_t mb = __reduce_min_sync(kFull, sb);
      i_min = __reduce_min_sync(kFull, (lead && sb == mb) ? jk : kEmpty);
      s_min = __uint_as_float(mb);
      s_2 = __uint_as_float(__reduce_min_sync(kFull, (lead && jk != i_min) ? sb : kEmpty));
    } else {
      const float4 qv = __ldg(Qd + (size_t)q * 32 + lane);
      float part[KM];
#pragma unroll
      for (int k = 0; k < KM; ++k) {
        const uint32_t jk = __shfl_sync(kFull, lst, k) & idx_mask;
        part[k] = 0.f;
        if (k < kept) {
          const float4 tv = __ldg(Td + (size_t)jk * 32 + lane);
          const float dx = qv.x - tv.x, dy = qv.y - tv.y, dz = qv.z - tv.z, dw = qv.w - tv.w;
          part[k] = fmaf(dw, dw, fmaf(dz, dz, fmaf(dy, dy, dx * dx)));
        }
      }
      // transpose-reduce: after log2(KM) halving steps the lane whose bits
      // (4, 3, .., 5-log2 KM) spell k holds candidate k's partial sum
      constexpr int kLog = KM == 8 ? 3 : (KM == 16 ? 4 : 5);
#pragma unroll
      for (int st = 0; st < kLog; ++st) {
        const int half = (KM >> st) >> 1, m = 16 >> st;
        const bool up = (lane & m) != 0;
#pragma unroll
        for (int i = 0; i < KM / 2; ++i) {
          if (i < half) {
            const float send = up ? part[i] : part[i + half];
            const float keep = up ? part[i + half] : part[i];
            part[i] = keep + __shfl_xor_sync(kFull, send, m);
          }
        }
      }
      float red = part[0];
#pragma unroll
      for (int m = 16 >> kLog; m > 0; m >>= 1) red += __shfl_xor_sync(kFull, red, m);
      int src_lane = 0;
#pragma unroll
      for (int b = 0; b < kLog; ++b)
        if (lane & (1 << b)) src_lane |= 1 << (4 - (kLog - 1 - b));
      const float s_own = __shfl_sync(kFull, red, src_lane);  // lane k: candidate k
      // argmin of (s, idx) and runner-up value over lanes < kept
      float bs = mine ? s_own : __int_as_float(0x7f800000);
      uint32_t bi = mine ? my_idx : 0xffffffffu;
#pragma unroll
      for (int o = KM / 2; o > 0; o >>= 1) {
        const float os = __shfl_xor_sync(kFull, bs, o);
        const uint32_t oi = __shfl_xor_sync(kFull, bi, o);
        if (os < bs || (os == bs && oi < bi)) {
          bs = os;
          bi = oi;
        }
      }
      s_min = __shfl_sync(kFull, bs, 0);
      i_min = __shfl_sync(kFull, bi, 0);
      float s2 = (mine && my_idx != i_min) ? s_own : __int_as_float(0x7f800000);
#pragma unroll
      for (int o = KM / 2; o > 0; o >>= 1) s2 = fminf(s2, __shfl_xor_sync(kFull, s2, o));
      s_2 = __shfl_sync(kFull, s2, 0);
    }
    // certified in FP32: the distances carry relative error < 1e-6, each
    // product below 2^-24 and r2f its own 2^-24, all far inside the 2e-5
    // margins (ties d1 == r^2 d2 land in the FP64 band, which rejects them)
    // Accept also needs the argmin itself certified (s_min clearly below
    // s_2): with ratio > 1 a near tie passes the ratio margin, and the FP32
    // argmin could then differ from the reference's FP64 (dist, idx) first.
    // ratio <= 0 or NaN: d1 < d2 * ratio never holds (hashmatch.cpp:47-49),
    // so only lone candidates are kept.
    const float c_hi = 1.0f + 2.0e-5f, c_lo = 1.0f - 2.0e-5f;
    const bool finite = s_min >= 1.0e-30f && s_2 < 3.0e38f;
    const bool rpos = ratio > 0.0;
    const bool fast = (a.test_flags & kTestForceFp64Rerank) == 0;
    const bool accept = fast && rpos && finite && s_min * c_hi < r2f * s_2 && s_min * c_hi < s_2;
    const bool reject = fast && (!rpos || (finite && s_min * c_lo >= (r2f * s_2) * c_hi));
    if (accept) {
      result = (int32_t)i_min;
    } else if (!reject) {
      // FP64 reference path (hashmatch.cpp:35-42, :196-208)
      double e = __longlong_as_double(0x7ff0000000000000ll);
      if (mine) {
        const float* qd = Q.desc + (size_t)q * kDim;
        const float* td = T.desc + (size_t)my_idx * kDim;
        double s = 0.0;
#pragma unroll 8
        for (int c = 0; c < kDim; ++c) {
          const double d = __dsub_rn((double)__ldg(qd + c), (double)__ldg(td + c));
          s = __dadd_rn(s, __dmul_rn(d, d));
        }
        e = __dsqrt_rn(s);
      }
      double be = e;
      uint32_t bj = mine ? my_idx : 0xffffffffu;
#pragma unroll
      for (int o = KM / 2; o > 0; o >>= 1) {
        const double oe = __shfl_xor_sync(kFull, be, o);
        const uint32_t oj = __shfl_xor_sync(kFull, bj, o);
        if (oe < be || (oe == be && oj < bj)) {
          be = oe;
          bj = oj;
        }
      }
      const double e_first = __shfl_sync(kFull, be, 0);
      const uint32_t i_first = __shfl_sync(kFull, bj, 0);
      double e2 = (mine && my_idx != i_first) ? e : __longlong_as_double(0x7ff0000000000000ll);
#pragma unroll
      for (int o = KM / 2; o > 0; o >>= 1) e2 = fmin(e2, __shfl_xor_sync(kFull, e2, o));
      const double e_second = __shfl_sync(kFull, e2, 0);
      if (e_first < __dmul_rn(e_second, ratio)) result = (int32_t)i_first;
      if (lane == 0 && a.exact_queries) atomicAdd(a.exact_queries, 1ull);
    }
  }
  return result;
}

#ifndef BMG_MATCH_MINB
#define BMG_MATCH_MINB 1  // resident match CTAs per SM the register budget is sized for
#endif
template <int FWP, int KM, int NT, int KC>
__global__ void __launch_bounds__(NT, (KM == 8 ? BMG_MATCH_MINB : 1)) match_kernel(MatchLaunch a) {
  const PairWork w = a.work[blockIdx.x];
  const ImgDev T = a.imgs[w.t_img];
  const ImgDev Q = a.imgs[w.q_img];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kWarps = NT / 32;

  const int L = a.tables, K = KC ? KC : a.k, ib = a.idx_bits;
  const uint32_t idx_mask = (1u << ib) - 1u;
  const int nb1 = a.n_buckets + 1;
  uint32_t n_matched = 0;

  auto emit = [&](uint32_t q, int32_t result) {
    if (lane == 0) {
      a.dense[a.dense_off[w.pair] + q] = result;
      n_matched += result >= 0 ? 1u : 0u;
    }
  };
  auto finish = [&](uint32_t q, uint32_t lst, int kept) {
    emit(q, rerank_query<KM>(a, Q, T, q, lst, kept, idx_mask));
  };

  // the next query's bucket ids are loaded two queries ahead and its bucket
  // ranges one query ahead (lanes >= L and past the range keep 0 / empty)
  auto load_b = [&](uint32_t q) -> uint32_t {
    return lane < L && q < w.q_end ? __ldg(Q.coarse + (size_t)q * L + lane) : kEmpty;
  };
  auto load_range = [&](uint32_t b, uint32_t& lo, uint32_t& hi) {
    lo = hi = 0;
    if (b != kEmpty) {
      const uint32_t* off = T.offsets + (size_t)lane * nb1 + b;
      lo = __ldg(off);
      hi = __ldg(off + 1);
    }
  };
  uint32_t lo_next, hi_next;
  load_range(load_b(w.q_begin + warp), lo_next, hi_next);
  uint32_t b_next = load_b(w.q_begin + warp + kWarps);
  for (uint32_t q = w.q_begin + warp; q < w.q_end; q += kWarps) {
    const uint32_t lo = lo_next, sz = hi_next - lo_next;
    load_range(b_next, lo_next, hi_next);
    b_next = load_b(q + 2 * kWarps);
    uint64_t qc[FWP];
#pragma unroll
    for (int x = 0; x < FWP; ++x) qc[x] = __ldg(Q.fine + (size_t)q * FWP + x);

    uint32_t lst = kEmpty;
    bool exact = KM != 8;
    if constexpr (KM == 8) {
      // Each lane keeps its kLaneKeys smallest keys sorted in kl[].
      uint32_t kl[kLaneKeys];
#pragma unroll
      for (int i = 0; i < kLaneKeys; ++i) kl[i] = kEmpty;
      walk_union<FWP>(T, L, lo, sz, ib, qc, [&](uint32_t key) {
#pragma unroll
        for (int i = kLaneKeys - 1; i > 0; --i) kl[i] = max(kl[i - 1], min(kl[i], key));
        kl[0] = min(kl[0], key);
      });
      // a lane that dropped a key x kept 4 keys <= x; if x is below the last
      // pull, all 4 are pulled too, so the lane ends empty: a full lane that
      // ends empty reruns the query exactly (a superset of the harmful drops)
      const bool full = kl[kLaneKeys - 1] != kEmpty;
      uint32_t m = kEmpty;
      // Copies of one key that landed in one lane sit next to each other:
      // squeeze them out so a lane's list is a prefix of its distinct keys.
      // Copies in different lanes are popped together below.
      bool dup = false;
#pragma unroll
      for (int i = 0; i + 1 < kLaneKeys; ++i) dup |= (kl[i] == kl[i + 1]) & (kl[i + 1] != kEmpty);
      if (__any_sync(kFull, dup)) {
#pragma unroll
        for (int rep = 0; rep + 1 < kLaneKeys; ++rep) {
#pragma unroll
          for (int i = 0; i + 1 < kLaneKeys; ++i) {
            if (kl[i] == kl[i + 1]) {
#pragma unroll
              for (int x = i + 1; x + 1 < kLaneKeys; ++x) kl[x] = kl[x + 1];
              kl[kLaneKeys - 1] = kEmpty;
            }
          }
        }
      }
      // Pull r is the smallest key not pulled yet, unless some lane dropped a
      // key below the last pull (it may be missing from the lists; a dropped
      // copy of a listed key also counts): then the query reruns on the
      // exact path below.
      // the pulls are warp-uniform: lane r < 8 takes pull r through a
      // 3-level select on its lane bits (7 SEL) instead of a compare and
      // select per pull
      uint32_t mv[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        mv[r] = kEmpty;
        if (r < K) {
          m = __reduce_min_sync(kFull, kl[0]);
          mv[r] = m;
          const bool pop = kl[0] == m;
#pragma unroll
          for (int i = 0; i + 1 < kLaneKeys; ++i) kl[i] = pop ? kl[i + 1] : kl[i];
          kl[kLaneKeys - 1] = pop ? kEmpty : kl[kLaneKeys - 1];
        }
      }
      {
        const bool b0 = (lane & 1) != 0, b1 = (lane & 2) != 0, b2 = (lane & 4) != 0;
        const uint32_t x0 = b0 ? mv[1] : mv[0], x1 = b0 ? mv[3] : mv[2];
        const uint32_t x2 = b0 ? mv[5] : mv[4], x3 = b0 ? mv[7] : mv[6];
        const uint32_t y0 = b1 ? x1 : x0, y1 = b1 ? x3 : x2;
        lst = lane < 8 ? (b2 ? y1 : y0) : kEmpty;
      }
      exact = __any_sync(kFull, full && kl[0] == kEmpty) || (a.test_flags & kTestForceExactWalk) != 0;
    }
    if (exact) {
      // ---- exact path: keys below the current K-th key are pulled out in
      // ascending order with REDUX and inserted into the sorted list held by
      // lanes 0..KM-1.  Every lane holding the pulled key clears it, and a
      // key already listed is skipped, so a train index reached from several
      // tables is taken once.
      lst = kEmpty;
      uint32_t thr = kEmpty;
      walk_union<FWP>(T, L, lo, sz, ib, qc, [&](uint32_t key) {
        key = key < thr ? key : kEmpty;
        for (;;) {
          const uint32_t m = __reduce_min_sync(kFull, key);
          if (m >= thr) break;
          if (key == m) key = kEmpty;
          if (!__any_sync(kFull, lane < KM && lst == m)) {
            const uint32_t prev = __shfl_up_sync(kFull, lst, 1);
            const uint32_t nv = lst < m ? lst : ((lane == 0 || prev < m) ? m : prev);
            lst = lane < KM ? nv : kEmpty;
            thr = __shfl_sync(kFull, lst, K - 1);
          }
        }
      });
      if (lane == 0 && a.exact_queries) atomicAdd(a.exact_queries + 1, 1ull);
    }

    // ---- re-rank + ratio test
    const int kept = __popc(__ballot_sync(kFull, lane < K && lst != kEmpty));
    finish(q, lst, kept);
  }
  if (lane == 0 && n_matched) atomicAdd(a.pair_count + w.pair, n_matched);
}

// ---------------------------------------------------------------------------
// K6: per-launch exclusive scan of match counts (appending after the running
// total of earlier rows) and ascending-query compaction of the dense arrays.
// ---------------------------------------------------------------------------
// ranges[2i], ranges[2i+1] = [begin, end) of pair i's matches in the result
// log; a launch's pairs are packed from `base` (the row's own log region).
__global__ void __launch_bounds__(1024) scan_counts_kernel(const uint32_t* __restrict__ counts, int n,
                                                           uint64_t* __restrict__ ranges, uint64_t base) {
  __shared__ uint32_t s_warp[32];
  __shared__ unsigned long long s_carry;
  if (threadIdx.x == 0) s_carry = base;
  __syncthreads();
  for (int b0 = 0; b0 < n; b0 += blockDim.x) {
    const int i = b0 + threadIdx.x;
    const uint32_t v = i < n ? counts[i] : 0u;
    const unsigned long long carry = s_carry;
    const uint32_t incl = block_incl_scan(v, s_warp);
    if (i < n) {
      ranges[2 * i] = carry + incl - v;
      ranges[2 * i + 1] = carry + incl;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_carry = carry + incl;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) compact_kernel(const int32_t* __restrict__ dense,
                                                       const uint64_t* __restrict__ dense_off,
                                                       const uint32_t* __restrict__ nq,
                                                       const uint64_t* __restrict__ out_off,
                                                       int32_t* __restrict__ out) {
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_base;
  const int p = blockIdx.x;
  const int32_t* d = dense + dense_off[p];
  const uint32_t n = nq[p];
  uint64_t base = out_off[2 * p];  // [begin, end) ranges from scan_counts
  for (uint32_t q0 = 0; q0 < n; q0 += blockDim.x) {
    const uint32_t q = q0 + threadIdx.x;
    const int32_t v = q < n ? d[q] : -1;
    const uint32_t f = v >= 0 ? 1u : 0u;
    const uint32_t incl = block_incl_scan(f, s_warp);
    if (f) reinterpret_cast<int2*>(out)[base + incl - 1] = make_int2((int32_t)q, v);
    if (threadIdx.x == blockDim.x - 1) s_base = incl;
    __syncthreads();
    base += s_base;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Row metadata (pointer tables, tile and work lists) is read from mapped
// pinned host memory and zero fills are done by this kernel on the row's own
// stream: cudaMemcpyAsync / cudaMemsetAsync would queue on the copy engines
// behind the bulk descriptor uploads and stall rows that could already run.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) meta_kernel(MetaBatch b) {
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
  for (int i = 0; i < b.n; ++i) {
    const MetaOp o = b.op[i];
    const size_t n16 = o.bytes >> 4;
    uint4* d = static_cast<uint4*>(o.dst);
    const uint4* src = static_cast<const uint4*>(o.src);
    for (size_t k = tid; k < n16; k += nth) d[k] = src ? src[k] : make_uint4(0u, 0u, 0u, 0u);
    for (size_t k = (n16 << 4) + tid; k < o.bytes; k += nth)
      static_cast<unsigned char*>(o.dst)[k] = src ? reinterpret_cast<const unsigned char*>(o.src)[k] : 0;
  }
}

}  // namespace

void launch_meta(const MetaBatch& b, cudaStream_t s) {
  size_t units = 0;
  for (int i = 0; i < b.n; ++i) units = std::max<size_t>(units, (b.op[i].bytes + 15) >> 4);
  const int grid = (int)std::min<size_t>(148, std::max<size_t>(1, (units + 255) / 256));
  if (b.n) meta_kernel<<<grid, 256, 0, s>>>(b);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
int launch_row_mean(const ImgDev* imgs, int n_imgs, const uint32_t* tile_img,
                    const uint32_t* tile_start, int n_tiles, unsigned long long total, void* scratch,
                    MeanState* st, float* mean_out, double* acc_out, bool chain_only, bool sums_resident,
                    cudaStream_t s) {
  int launches = 0;
  const uint32_t* gate = nullptr;
  if (!chain_only && n_tiles > 0) {
    if (!sums_resident) {
      mean_sums_kernel<<<n_tiles, kSumsThreads, 0, s>>>(imgs, tile_img, tile_start);
      ++launches;
    }
    mean_resolve_kernel<<<kDim, kResolveThreads, 0, s>>>(imgs, tile_img, tile_start, static_cast<i128*>(scratch),
                                                         n_tiles, total, st, mean_out, acc_out);
    ++launches;
    gate = &st->need_chain;
  }
  mean_chain_kernel<<<kDim / 32, 32, 0, s>>>(imgs, n_imgs, gate, mean_out, acc_out);
  return launches + 1;
}

static int proj_pstride(const HashDev& h) { return (std::min(kPlaneChunk, h.n_planes) + 11) / 12 * 12; }

static size_t proj_smem_bytes(int pstride) {
  return sizeof(float) * (2 * kCodesTile * kTileStride + kDim * pstride) + 2 * sizeof(uint64_t);
}

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(project_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)proj_smem_bytes(kPlaneChunk));
  }
  return n;
}

static size_t proj_tc_smem_bytes(const HashDev& h) {
  return 1024 + 3 * (size_t)kTcDigitBytes + 3 * (size_t)h.tc_npad * 128 + sizeof(float) * kTcRows * kDim +
         sizeof(int) * (kTcRows + h.tc_npad + 2) + 3 * sizeof(uint64_t) + 16 + sizeof(TileStatsSmem<kTcParts>) + 16;
}


static bool project_simt_forced() {
  static const bool v = [] {
    const char* e = getenv("BMG_PROJECT_SIMT");  // A/B switch: the FP32 SIMT K2
    return e && e[0] == '1';
  }();
  return v;
}

bool project_writes_tile_stats(const HashDev& h) { return h.tc_b != nullptr && !project_simt_forced(); }

static void launch_project_job(const HashDev& h, const ProjJob& job, cudaStream_t s) {
  if (job.n_tiles <= 0) return;
  if (h.tc_b && !project_simt_forced()) {
    const size_t smem = proj_tc_smem_bytes(h);
    static int configured = -1;
    if (configured != (int)smem) {
      cudaFuncSetAttribute(project_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      configured = (int)smem;
    }
    project_tc_kernel<<<std::min(job.n_tiles, sm_count()), kTcThreads, smem, s>>>(h, job);
    return;
  }
  const int pstride = proj_pstride(h);
  dim3 grid(std::min(job.n_tiles, sm_count()), (h.n_planes + kPlaneChunk - 1) / kPlaneChunk);
  project_kernel<<<grid, 512, proj_smem_bytes(pstride), s>>>(h, job, pstride);
}

void launch_project(const HashDev& h, const ImgDev& one, cudaStream_t s) {
  // one image right behind its upload (tile per CTA for an 8k image)
  ProjJob j{};
  j.n_tiles = (int)((one.n + kCodesTile - 1) / kCodesTile);
  j.one = one;
  launch_project_job(h, j, s);
}

void launch_project_tiles(const HashDev& h, const ImgDev* imgs_dev, const uint32_t* tile_img,
                          const uint32_t* tile_start, int n_tiles, cudaStream_t s) {
  ProjJob j{};
  j.imgs = imgs_dev;
  j.tile_img = tile_img;
  j.tile_start = tile_start;
  j.n_tiles = n_tiles;
  launch_project_job(h, j, s);
}

void launch_codes(const HashDev& h, const ImgDev* imgs_dev, const uint32_t* tile_img,
                  const uint32_t* tile_start, int n_tiles, const float* mean, float* mproj, Fixup* fix,
                  uint32_t* fix_count, uint32_t fix_cap, cudaStream_t s) {
  const int mw = (h.n_planes + 31) / 32 + 2;
  const size_t smem = sizeof(uint32_t) * kCodesTile * mw + sizeof(float) * (h.n_planes + 1);
  // overflow flags live right after the fixup counter (see bmg_api.cpp)
  uint32_t* overflow = fix_count + 1;
  if (n_tiles <= 0) return;
  mproj_kernel<<<(h.n_planes + 255) / 256, 256, 0, s>>>(h, mean, mproj);
  if (h.proj_stride <= 192) {
    const size_t tsmem = sizeof(float) * 2 * kCodesTile * h.proj_stride + sizeof(uint32_t) * (kCodesTile * mw + 2) +
                         16 + sizeof(float) * (2 * kCodesTile + 2 * h.n_planes + 4) + 32;
    static size_t configured = 0;
    if (configured != tsmem) {
      cudaFuncSetAttribute(codes_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
      configured = tsmem;
    }
    codes_tma_kernel<<<std::min(n_tiles, sm_count()), kCodesTmaThreads, tsmem, s>>>(
        h, imgs_dev, tile_img, tile_start, n_tiles, mproj, fix, fix_count, fix_cap, overflow);
    return;
  }
  codes_kernel<<<n_tiles, kCodesThreads, smem, s>>>(h, imgs_dev, tile_img, tile_start, mproj, fix, fix_count,
                                                    fix_cap, overflow);
}

void launch_codes_fixup(const HashDev& h, const ImgDev* imgs_dev, int n_imgs, const float* mean,
                        const Fixup* fix, const uint32_t* fix_count, uint32_t fix_cap,
                        unsigned long long* fixed_bits, cudaStream_t s) {
  codes_fixup_kernel<<<4 * 148, kFixupThreads, 0, s>>>(h, imgs_dev, mean, fix, fix_count, fix_cap, fixed_bits);
  codes_overflow_kernel<<<148, 256, 0, s>>>(h, imgs_dev, n_imgs, mean, fix_count + 1);
}

int launch_tables(const HashDev& h, const ImgDev* imgs_dev, const uint32_t* tile_img,
                  const uint32_t* tile_start, int n_tiles, int n_imgs, cudaStream_t s) {
  if (h.n_buckets <= kTablesFusedMaxBuckets) {
    tables_fused_kernel<<<dim3(n_imgs, h.tables), 1024, sizeof(uint32_t) * h.n_buckets, s>>>(h, imgs_dev);
    return 1;
  }
  tables_hist_kernel<<<n_tiles, kCodesTile, 0, s>>>(h, imgs_dev, tile_img, tile_start);
  tables_scan_kernel<<<dim3(n_imgs, h.tables), 1024, 0, s>>>(h, imgs_dev);
  tables_scatter_kernel<<<n_tiles, kCodesTile, 0, s>>>(h, imgs_dev, tile_img, tile_start);
  return 3;
}

template <int FWP, int KM, int NT, int KC>
static void launch_match_t(const MatchLaunch& a, int n_work, cudaStream_t s) {
  match_kernel<FWP, KM, NT, KC><<<n_work, NT, 0, s>>>(a);
}

template <int FWP>
static void launch_match_fw(const MatchLaunch& a, int n_work, cudaStream_t s) {
  if (a.k == 8) {
    launch_match_t<FWP, 8, kMatchThreads, 8>(a, n_work, s);  // MatchParams default
  } else if (a.k < 8) {
    launch_match_t<FWP, 8, kMatchThreads, 0>(a, n_work, s);
  } else {
    launch_match_t<FWP, 32, 512, 0>(a, n_work, s);
  }
}

int device_sm_count() { return sm_count(); }

int match_queries_per_cta(int fwp, int k) {
  (void)fwp;
  (void)k;
  return kMatchQueries;
}

void launch_match(const MatchLaunch& a, int fwp, int n_work, cudaStream_t s) {
  switch (fwp) {
    case 1: launch_match_fw<1>(a, n_work, s); break;
    case 2: launch_match_fw<2>(a, n_work, s); break;
    case 4: launch_match_fw<4>(a, n_work, s); break;
    case 8: launch_match_fw<8>(a, n_work, s); break;
    case 16: launch_match_fw<16>(a, n_work, s); break;
    default: break;  // bmg_create rejects fine_bits > 1024 (fwp > 16)
  }
}

void launch_scan_counts(const uint32_t* counts, int n, uint64_t* ranges_out, uint64_t base, cudaStream_t s) {
  scan_counts_kernel<<<1, 1024, 0, s>>>(counts, n, ranges_out, base);
}

void launch_compact(const int32_t* dense, const uint64_t* dense_off, const uint32_t* nq,
                    const uint64_t* out_off, int n_pairs, int32_t* out, cudaStream_t s) {
  if (n_pairs > 0) compact_kernel<<<n_pairs, 1024, 0, s>>>(dense, dense_off, nq, out_off, out);
}

}  // namespace bmg
