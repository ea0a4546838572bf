// vlad.cu -- VLAD image encoding for retrieval:
// encode_vlad (/root/reference/proj/src/retrieval.cpp:160-205,
// include/bandmatch/retrieval.hpp:36-47) for a batch of images, bit-exact.
//
//   V1 vlad_assign_kernel  nearest centroid per descriptor (:170-183): FP32
//                          squared distances of a 128-descriptor x 64-centroid
//                          tile (packed FP32x2 ops) as a certified filter; a
//                          descriptor whose best and runner-up are not
//                          separated by the error bound goes to V1b
//   V1b vlad_fix_kernel    the reference's FP64 loop for those descriptors:
//                          s = sum_c ((double)d - c)^2 sequentially, strict <
//                          over k ascending (first minimum wins)
//   V2 vlad_accum_kernel   residual sums acc[k][c] += (double)d[c] - c_k[c]
//                          (:184-187) in descriptor order: one thread per
//                          (k, c) chain, members of cluster k compacted per
//                          128-descriptor chunk with ballots
//   V3 vlad_final_kernel   signed square root, the sequential FP64 norm over
//                          k*128 values, 1/sqrt, float cast (:189-203)
//
// Exactness: FP32 only decides the argmin when a rigorous bound proves the
// FP64 one equal.  Each FP32 difference of two floats is rounded once, each
// FMA accumulation once: |s32 - s| <= 130 u s (u = 2^-24) = 7.8e-6 s, plus at
// most 128 * 2^-149 from underflow; the reference's own FP64 sum is within
// 128 * 2^-53 s.  Accept iff best * (1 + 1e-5) < second * (1 - 1e-5) and
// second >= 1e-30 (or there is no second centroid / it overflowed), with
// every value finite; anything else (ties, NaN, inf, tiny distances) is
// recomputed in FP64.  Accumulation and normalisation are the reference's
// FP64 operations in its order (__dadd_rn / __dsub_rn / __dmul_rn /
// __dsqrt_rn / __ddiv_rn: no contraction, like the reference's x86-64 build).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "bmg_internal.h"

namespace bmg {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kVTile = kVladTile;  // descriptors per tile
constexpr int kVCents = 64;       // centroids per smem tile
constexpr int kVThreads = 256;    // 32 descriptor groups (4 rows each) x 8 centroid groups (8 each)
constexpr int kVRowStride = kDim + 4;  // 528-byte rows: conflict-free LDS.128 across 4 rows

struct VSmem {
  float d[kVTile][kVRowStride];  // descriptor tile, row-major (one bulk copy per row)
  float nc[kDim][kVCents];       // negated centroid tile, transposed
  uint64_t bar;                  // tile-arrival mbarrier
};

__device__ __forceinline__ uint32_t v_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Persistent CTAs (grid <= 2 per SM): each loops over 128-descriptor tiles;
// a tile's rows arrive by cp.async.bulk (one 512-byte copy per row, issued
// by warp 0 onto one mbarrier) while the previous tile's
// results are folded and written.  Thread (dg, cg): rows dg + 32q (q < 4)
// against centroids 8cg..8cg+7 of the centroid tile.
__global__ void __launch_bounds__(kVThreads, 2) vlad_assign_kernel(VladBatch b, int n_tiles) {
  extern __shared__ float4 v_smem_raw[];
  VSmem& sm = *reinterpret_cast<VSmem*>(v_smem_raw);
  const int t = threadIdx.x;
  const int cg = t & 7, dg = t >> 3;
  auto issue = [&](int tile) {  // warp 0: lane l copies rows l, l + 32, ...
    const uint32_t img = b.tile_img[tile], i0 = b.tile_start[tile];
    const VladImg im = b.imgs[img];
    const uint32_t rows = min((uint32_t)kVTile, im.n - i0);
    if (t == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(v_smem(&sm.bar)),
                   "r"(rows * 512u)
                   : "memory");
    __syncwarp();
    for (uint32_t r = t; r < rows; r += 32)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
              v_smem(&sm.d[r][0])),
          "l"(im.desc + (size_t)(i0 + r) * kDim), "r"(v_smem(&sm.bar))
          : "memory");
  };
  auto wait_tile = [&](uint32_t par) {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(v_smem(&sm.bar)), "r"(par)
          : "memory");
  };
  auto load_cents = [&](int k0, int kc) {
    for (int e = t; e < kVCents * kDim; e += kVThreads) {
      const int k = e & (kVCents - 1), c = e / kVCents;  // conflict-free stores
      sm.nc[c][k] = k < kc ? -__ldg(b.centroids + (size_t)(k0 + k) * kDim + c) : 0.f;
    }
  };
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(v_smem(&sm.bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if ((int)blockIdx.x < n_tiles && t < 32) issue(blockIdx.x);
  const bool one_cent_tile = b.k_words <= kVCents;
  if (one_cent_tile) load_cents(0, b.k_words);
  uint32_t par = 0;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, par ^= 1u) {
    const uint32_t img = b.tile_img[tile], i0 = b.tile_start[tile];
    const VladImg im = b.imgs[img];
    const uint32_t rows = min((uint32_t)kVTile, im.n - i0);
    // rows past the image's end hold stale data: they are never written out
    wait_tile(par);
    __syncthreads();  // also: centroid tile stores visible
    float best[4], second[4];
    uint32_t bidx[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      best[q] = second[q] = __int_as_float(0x7f800000);
      bidx[q] = 0u;
    }
    bool nan_seen[4] = {false, false, false, false};
    for (int k0 = 0; k0 < b.k_words; k0 += kVCents) {
      const int kc = min(kVCents, b.k_words - k0);
      if (!one_cent_tile) {
        __syncthreads();
        load_cents(k0, kc);
        __syncthreads();
      }
      float2 acc[4][4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int p = 0; p < 4; ++p) acc[q][p] = make_float2(0.f, 0.f);
      for (int c = 0; c < kDim; c += 4) {
        float4 dv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) dv[q] = *reinterpret_cast<const float4*>(&sm.d[dg + 32 * q][c]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float4 c0 = *reinterpret_cast<const float4*>(&sm.nc[c + e][8 * cg]);
          const float4 c1 = *reinterpret_cast<const float4*>(&sm.nc[c + e][8 * cg + 4]);
          const float2 nc2[4] = {make_float2(c0.x, c0.y), make_float2(c0.z, c0.w), make_float2(c1.x, c1.y),
                                 make_float2(c1.z, c1.w)};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float dq = e == 0 ? dv[q].x : e == 1 ? dv[q].y : e == 2 ? dv[q].z : dv[q].w;
            const float2 d2 = make_float2(dq, dq);
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              const float2 df = __fadd2_rn(d2, nc2[p]);
              acc[q][p] = __ffma2_rn(df, df, acc[q][p]);
            }
          }
        }
      }
      // fold this centroid tile into the running (best, index, second)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int p = 0; p < 4; ++p) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int kk = 8 * cg + 2 * p + h;
            if (kk < kc) {
              const float sv = h ? acc[q][p].y : acc[q][p].x;
              nan_seen[q] |= sv != sv;
              const uint32_t k = (uint32_t)(k0 + kk);
              if (sv < best[q]) {
                second[q] = best[q];
                best[q] = sv;
                bidx[q] = k;
              } else {
                second[q] = fminf(second[q], sv);
              }
            }
          }
        }
      }
    }
    // every thread is done reading the tile: the next one may land
    __syncthreads();
    const int next = tile + gridDim.x;
    if (next < n_tiles && t < 32) issue(next);
    // reduce over the 8 centroid groups (lanes differing in bits 0..2)
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float ob = __shfl_xor_sync(kFull, best[q], o), os = __shfl_xor_sync(kFull, second[q], o);
        const uint32_t oi = __shfl_xor_sync(kFull, bidx[q], o);
        if (ob < best[q] || (ob == best[q] && oi < bidx[q])) {
          second[q] = fminf(best[q], os);
          best[q] = ob;
          bidx[q] = oi;
        } else {
          second[q] = fminf(second[q], fminf(ob, os));
        }
      }
    }
    // a NaN distance of a row in any of its 8 lanes sends it to the FP64
    // loop (fminf would hide it)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) nan_seen[q] |= __shfl_xor_sync(kFull, (int)nan_seen[q], o) != 0;
    if (cg == 0) {
      const float c_hi = 1.0f + 1.0e-5f, c_lo = 1.0f - 1.0e-5f;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t row = (uint32_t)(dg + 32 * q);
        if (row >= rows) continue;
        const float bs = best[q], s2 = second[q];
        const bool finite = bs <= 3.0e38f;
        bool sep = s2 == __int_as_float(0x7f800000) || (s2 >= 1.0e-30f && bs * c_hi < s2 * c_lo);
        if (b.cent64) {
          // float-rounded double centroids: |s32 - s| <= 132 u s + 2.1 u ||c|| sqrt(s)
          // + 2 u^2 ||c||^2 (u = 2^-24), taken with generous constants
          const float cn = b.cnorm_max;
          auto bound = [&](float x) { return 1.0e-5f * x + 2.5e-7f * cn * sqrtf(x) + 1.0e-13f * cn * cn; };
          sep = s2 == __int_as_float(0x7f800000) || (s2 >= 1.0e-30f && bs + bound(bs) < s2 - bound(s2));
        }
        const size_t gi = im.assign_off + i0 + row;
        if (!nan_seen[q] && finite && sep) {
          b.assign[gi] = (int32_t)bidx[q];
        } else {
          b.assign[gi] = -1;
          const uint32_t slot = atomicAdd(b.fix_count, 1u);
          if (slot < b.fix_cap) b.fix[slot] = make_uint2(img, i0 + row);
        }
      }
    }
  }
}

// sq_dist (retrieval.cpp:45-52): sequential FP64 sum of ((double)d - c)^2
__device__ __forceinline__ double sq_dist64(const float* __restrict__ d, const double* __restrict__ c) {
  const float4* dp = reinterpret_cast<const float4*>(d);
  const double2* cp = reinterpret_cast<const double2*>(c);
  double s = 0.0;
#pragma unroll 8
  for (int c4 = 0; c4 < kDim / 4; ++c4) {
    const float4 dv = __ldg(dp + c4);
    const double2 c0 = __ldg(cp + 2 * c4), c1 = __ldg(cp + 2 * c4 + 1);
    const float dd[4] = {dv.x, dv.y, dv.z, dv.w};
    const double cc[4] = {c0.x, c0.y, c1.x, c1.y};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const double diff = __dsub_rn((double)dd[e], cc[e]);
      s = __dadd_rn(s, __dmul_rn(diff, diff));
    }
  }
  return s;
}

// The reference's loop (:170-183) for the uncertified descriptors; one warp
// per descriptor, lanes over centroids, each distance a sequential FP64 sum.
__global__ void __launch_bounds__(256) vlad_fix_kernel(VladBatch b) {
  const uint32_t n_fix = min(*b.fix_count, b.fix_cap);
  const int lane = threadIdx.x & 31;
  for (uint32_t f = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; f < n_fix;
       f += (gridDim.x * blockDim.x) >> 5) {
    const uint2 e = b.fix[f];
    const VladImg im = b.imgs[e.x];
    const float* d = im.desc + (size_t)e.y * kDim;
    double bv = __longlong_as_double(0x7ff0000000000000ll);  // +inf: s < inf required
    int bk = 0x7fffffff;
    bool nan0 = false;  // k-means: centroid 0's distance is NaN
    for (int k = lane; k < b.k_words; k += 32) {
      double s = 0.0;
      if (b.cent64) {
        s = sq_dist64(d, b.cent64 + (size_t)k * kDim);
      } else {
        const float4* cp = reinterpret_cast<const float4*>(b.centroids + (size_t)k * kDim);
        const float4* dp = reinterpret_cast<const float4*>(d);
#pragma unroll 8
        for (int c4 = 0; c4 < kDim / 4; ++c4) {
          const float4 dv = __ldg(dp + c4), cv = __ldg(cp + c4);
          const float dd[4] = {dv.x, dv.y, dv.z, dv.w}, cc[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const double diff = __dsub_rn((double)dd[e], (double)cc[e]);
            s = __dadd_rn(s, __dmul_rn(diff, diff));
          }
        }
      }
      if (k == 0) nan0 = s != s;
      if (s < bv) {  // lanes visit their k ascending: first minimum per lane
        bv = s;
        bk = k;
      }
    }
    // train_codebook starts from centroid 0's distance (retrieval.cpp:101-108):
    // a NaN there is never replaced
    nan0 = __shfl_sync(kFull, (int)nan0, 0) != 0 && b.cent64;
    // first index of the minimum over lanes; none below +inf -> 0
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(kFull, bv, o);
      const int ok = __shfl_xor_sync(kFull, bk, o);
      if (ov < bv || (ov == bv && ok < bk)) {
        bv = ov;
        bk = ok;
      }
    }
    if (lane == 0) b.assign[im.assign_off + e.y] = (bk == 0x7fffffff || nan0) ? 0 : bk;
  }
}

// k-means: every point's FP64 distance to its centroid, the reference's
// best_d2 (retrieval.cpp:99-117: sq_dist with double centroids).
__global__ void __launch_bounds__(256) kmeans_d2_kernel(VladBatch b, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const VladImg im = b.imgs[0];
  const int32_t k = b.assign[i];
  b.point_d2[i] = sq_dist64(im.desc + (size_t)i * kDim, b.cent64 + (size_t)k * kDim);
}

// Stable counting sort of an image's descriptors by nearest centroid (the
// accumulation order of :184-187 within a cluster is descriptor order).
// CTA per image, 32 warps; warp w owns a contiguous segment and walks it 32
// descriptors at a time (peers by __match_any_sync).
constexpr int kSortThreads = 1024;
__global__ void __launch_bounds__(kSortThreads) vlad_sort_kernel(VladBatch b) {
  extern __shared__ uint32_t s_cnt[];  // [32 warps][k_words]
  const uint32_t img = blockIdx.x;
  const VladImg im = b.imgs[img];
  const int K = b.k_words, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t seg = (im.n + 31u) / 32u, s0 = min(im.n, (uint32_t)warp * seg), s1 = min(im.n, s0 + seg);
  const int32_t* as = b.assign + im.assign_off;
  uint32_t* cnt = s_cnt + (size_t)warp * K;
  for (int k = lane; k < K; k += 32) cnt[k] = 0u;
  __syncwarp();
  for (uint32_t i0 = s0; i0 < s1; i0 += 32) {
    const bool v = i0 + lane < s1;
    const int32_t k = v ? as[i0 + lane] : -1;
    const uint32_t peers = __match_any_sync(kFull, k);
    if (v && (peers & ((1u << lane) - 1u)) == 0u) cnt[k] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // exclusive offsets in (cluster, warp) order; cluster starts to global
  __shared__ uint32_t s_tot[32];
  __shared__ uint32_t s_carry;
  if (threadIdx.x == 0) s_carry = 0u;
  __syncthreads();
  uint32_t* offs = b.member_off + (size_t)img * (K + 1);
  for (int k0 = 0; k0 < K; k0 += kSortThreads) {
    const int k = k0 + (int)threadIdx.x;
    uint32_t tot = 0;
    if (k < K)
      for (int w = 0; w < 32; ++w) {
        const uint32_t c = s_cnt[(size_t)w * K + k];
        s_cnt[(size_t)w * K + k] = tot;  // within-cluster prefix over warps
        tot += c;
      }
    // block-wide exclusive scan of the cluster totals
    uint32_t x = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      x += lane >= o ? y : 0u;
    }
    if (lane == 31) s_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t z = s_tot[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, z, o);
        z += lane >= o ? y : 0u;
      }
      s_tot[lane] = z;  // inclusive over warps
    }
    __syncthreads();
    const uint32_t base = s_carry + (warp ? s_tot[warp - 1] : 0u) + x - tot;
    if (k < K) {
      offs[k] = base;
      for (int w = 0; w < 32; ++w) s_cnt[(size_t)w * K + k] += base;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_carry += s_tot[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) offs[K] = im.n;
  __syncthreads();
  uint32_t* mem = b.members + im.assign_off;
  for (uint32_t i0 = s0; i0 < s1; i0 += 32) {
    const bool v = i0 + lane < s1;
    const int32_t k = v ? as[i0 + lane] : -1;
    const uint32_t peers = __match_any_sync(kFull, k);
    uint32_t pos = 0;
    if (v) pos = cnt[k] + __popc(peers & ((1u << lane) - 1u));
    __syncwarp();
    if (v) {
      mem[pos] = i0 + lane;
      if ((peers & ((1u << lane) - 1u)) == 0u) cnt[k] += __popc(peers);
    }
    __syncwarp();
  }
}

// acc[k][c] = sequential FP64 sum over cluster k's members in descriptor
// order (:184-187).  CTA = (image, centroid k), thread = channel c; member
// indices are staged in shared memory 512 at a time and the member rows
// gathered 16 ahead of the dependent __dadd_rn chain.
constexpr int kAccUnroll = 16;
__global__ void __launch_bounds__(kDim) vlad_accum_kernel(VladBatch b) {
  __shared__ uint32_t s_idx[4 * kDim];
  const uint32_t img = blockIdx.x, k = blockIdx.y;
  const VladImg im = b.imgs[img];
  const int c = threadIdx.x;
  const uint32_t* offs = b.member_off + (size_t)img * (b.k_words + 1);
  const uint32_t e0 = offs[k], e1 = offs[k + 1];
  const uint32_t* mem = b.members + im.assign_off;
  const float* dcol = im.desc + c;
  const double ck = (double)__ldg(b.centroids + (size_t)k * kDim + c);
  double acc = 0.0;
  for (uint32_t base = e0; base < e1; base += 4 * kDim) {
    const uint32_t m = min((uint32_t)(4 * kDim), e1 - base);
    __syncthreads();
    for (uint32_t i = c; i < m; i += kDim) s_idx[i] = __ldg(mem + base + i);
    __syncthreads();
    uint32_t e = 0;
    for (; e + kAccUnroll <= m; e += kAccUnroll) {
      float dv[kAccUnroll];
#pragma unroll
      for (int u = 0; u < kAccUnroll; ++u) dv[u] = __ldg(dcol + (size_t)s_idx[e + u] * kDim);
#pragma unroll
      for (int u = 0; u < kAccUnroll; ++u) acc = __dadd_rn(acc, __dsub_rn((double)dv[u], ck));
    }
    for (; e < m; ++e) acc = __dadd_rn(acc, __dsub_rn((double)__ldg(dcol + (size_t)s_idx[e] * kDim), ck));
  }
  b.acc[(size_t)img * b.k_words * kDim + (size_t)k * kDim + c] = acc;
}

// signed square root, sequential norm, scale (:189-203).  CTA per image.
// The norm is one dependent FP64 chain in index order: the CTA squares a
// chunk of values into shared memory, then one thread adds them up from
// there (the chain is __dadd_rn-latency bound, not load bound).
constexpr int kFinalThreads = 256;
constexpr int kNormChunk = 4096;  // doubles of squares staged per step (32 KiB)
__global__ void __launch_bounds__(kFinalThreads) vlad_final_kernel(VladBatch b) {
  __shared__ double s_sq[kNormChunk];
  __shared__ double s_norm;
  const uint32_t img = blockIdx.x;
  const VladImg im = b.imgs[img];
  const size_t dim = (size_t)b.k_words * kDim;
  double* acc = b.acc + (size_t)img * dim;
  float* out = b.values + (size_t)img * dim;
  if (im.n == 0) {
    for (size_t e = threadIdx.x; e < dim; e += blockDim.x) out[e] = 0.f;
    if (threadIdx.x == 0) b.degenerate[img] = 1;
    return;
  }
  double n2 = 0.0;  // thread 0's chain
  for (size_t c0 = 0; c0 < dim; c0 += kNormChunk) {
    const size_t m = min((size_t)kNormChunk, dim - c0);
    for (size_t e = threadIdx.x; e < m; e += blockDim.x) {
      const double v0 = acc[c0 + e];
      const double v = v0 >= 0.0 ? __dsqrt_rn(v0) : -__dsqrt_rn(-v0);
      acc[c0 + e] = v;
      s_sq[e] = __dmul_rn(v, v);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      size_t e = 0;
      for (; e + 16 <= m; e += 16) {
        double q[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) q[u] = s_sq[e + u];
#pragma unroll
        for (int u = 0; u < 16; ++u) n2 = __dadd_rn(n2, q[u]);
      }
      for (; e < m; ++e) n2 = __dadd_rn(n2, s_sq[e]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    s_norm = n2;
    b.degenerate[img] = (uint8_t)(n2 <= 0.0);
  }
  __syncthreads();
  const double nn = s_norm;
  if (nn <= 0.0) {
    for (size_t e = threadIdx.x; e < dim; e += blockDim.x) out[e] = 0.f;
    return;
  }
  const double inv = __ddiv_rn(1.0, __dsqrt_rn(nn));
  for (size_t e = threadIdx.x; e < dim; e += blockDim.x) out[e] = __double2float_rn(__dmul_rn(acc[e], inv));
}

}  // namespace

size_t vlad_assign_smem_bytes() { return sizeof(VSmem); }

void launch_vlad(const VladBatch& b, int n_imgs, int n_tiles, cudaStream_t s) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(vlad_assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(VSmem));
    cudaFuncSetAttribute(vlad_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(32 * sizeof(uint32_t) * kVladMaxWords));
  }
  if (n_tiles > 0) {
    vlad_assign_kernel<<<std::min(n_tiles, 2 * sms), kVThreads, sizeof(VSmem), s>>>(b, n_tiles);
    vlad_fix_kernel<<<sms, 256, 0, s>>>(b);
  }
  if (n_imgs > 0) {
    vlad_sort_kernel<<<n_imgs, kSortThreads, 32 * sizeof(uint32_t) * b.k_words, s>>>(b);
    vlad_accum_kernel<<<dim3(n_imgs, b.k_words), kDim, 0, s>>>(b);
    vlad_final_kernel<<<n_imgs, kFinalThreads, 0, s>>>(b);
  }
}

void launch_kmeans_assign(const VladBatch& b, int n_tiles, cudaStream_t s) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(vlad_assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(VSmem));
  }
  if (n_tiles <= 0) return;
  vlad_assign_kernel<<<std::min(n_tiles, 2 * sms), kVThreads, sizeof(VSmem), s>>>(b, n_tiles);
  vlad_fix_kernel<<<sms, 256, 0, s>>>(b);
  const uint32_t n = (uint32_t)b.fix_cap;  // the pool's size
  kmeans_d2_kernel<<<(n + 255) / 256, 256, 0, s>>>(b, n);
}

void launch_kmeans_sums(const VladBatch& b, cudaStream_t s) {
  cudaFuncSetAttribute(vlad_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(32 * sizeof(uint32_t) * kVladMaxWords));
  vlad_sort_kernel<<<1, kSortThreads, 32 * sizeof(uint32_t) * b.k_words, s>>>(b);
  vlad_accum_kernel<<<dim3(1, b.k_words), kDim, 0, s>>>(b);
}

}  // namespace bmg
