// track.cu — f1 cast-fused tracking (Alg. 1; hook P:386).
//
// The paper's own integration point: the diff is taken inside the optimizer-step epilogue that casts the
// fp32 master weights into the bf16 model weights (CastAndCopy, Alg. 1 l.5), and the changed indices
// accumulate across steps into the cumulative set I_T (Alg. 1 l.7) until the next sync. No persistent
// snapshot is kept and the sync no longer streams 2S bytes: it reads the 1-bit-per-element set and
// gathers V = W[I] (Alg. 2 l.5).
//
//  * k_cast_track   one tile (32768 elements = 1024 bitmap words) per CTA iteration; thread owns whole
//                   32-element words (so the bitmap update is a plain read-modify-write): 8 x 16 B fp32
//                   loads + 4 x 16 B bf16 loads, round_BF16 (RNE, NaN -> 0x7FC0, DESIGN C18), bitwise
//                   compare (C1); the new bf16 values are written per 32-byte sector only where a sector
//                   changed (full-sector stores: no L2 fill), the bitmap word only where a bit is new.
//  * k_track_count  per tile: popcount of its bitmap words.
//  * k_track_scan   per group of 1024 tiles: exclusive scan in place + group total; then one CTA scans the
//                   group totals; per-tensor counts from the tile offsets.
//  * k_track_write  per tile: word-order block scan, I = tile base + set-bit positions (ascending), V = W[I],
//                   the words cleared (next interval, Alg. 1 l.1).
#include "common.cuh"
#include "kernels.h"

namespace ss {

constexpr int kTT = 256;                         // threads per CTA
constexpr u32 kWordsPerTile = (u32)(kTile / 32); // 1024
constexpr u32 kGroup = 1024;                     // tiles per scan group

__device__ __forceinline__ u16 bf16_rne(u32 f) {
  if (((f >> 23) & 0xFFu) == 0xFFu && (f & 0x7FFFFFu) != 0) return 0x7FC0;
  return (u16)((f + 0x7FFFu + ((f >> 16) & 1u)) >> 16);
}

__device__ __forceinline__ u32 tile_words(u64 numel, u64 tile_base) {
  const u64 rem = numel - tile_base;
  const u64 ne = rem < kTile ? rem : kTile;
  return (u32)((ne + 31) / 32);
}

// Warp-cooperative: a warp takes 1024 consecutive elements per iteration; lane l handles elements
// 128k + 4l (k = 0..7): 16-byte fp32 loads and 8-byte bf16 loads, every load instruction covering 512 / 256
// contiguous bytes. Change bits: a 4-bit nibble per lane and k; the 8 lanes of a 32-element word OR their
// nibbles together (3 shuffles), lane 8j writes word j. Sectors (16 elements = 4 lanes) are stored whole when
// any of their elements changed.
__global__ void __launch_bounds__(kTT, 4) k_cast_track(TrackArgs a, const float* const* master, u16* const* W) {
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (u64 tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
    const u32 t = a.tile_tensor[tile];
    const u64 n = a.numel[t];
    const u64 base = (tile - a.tile_prefix[t]) * kTile;
    const u64 ne = (n - base) < kTile ? (n - base) : kTile;
    const float* M = master[t] + base;
    u16* Wt = W[t] + base;
    u32* bm = a.bitmap + a.bm_off[t] + base / 32;
    const bool vec = ((((uintptr_t)M) & 15u) | (((uintptr_t)Wt) & 7u)) == 0;   // else the scalar path
    for (u32 c = warp; c * 1024 < ne; c += kTT / 32) {
      const u32 e0 = c * 1024;
      uint4 m[8];
      uint2 o[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const u32 e = e0 + 128 * k + 4 * lane;
        if (vec && e + 4 <= ne) {
          m[k] = *reinterpret_cast<const uint4*>(M + e);
          o[k] = *reinterpret_cast<const uint2*>(Wt + e);
        } else {
          u32 mf[4] = {0, 0, 0, 0}, ow[4] = {0, 0, 0, 0};
#pragma unroll
          for (u32 q = 0; q < 4; ++q)
            if (e + q < ne) {
              mf[q] = __float_as_uint(M[e + q]);
              ow[q] = Wt[e + q];
            }
          m[k] = make_uint4(mf[0], mf[1], mf[2], mf[3]);
          o[k] = make_uint2(ow[0] | (ow[1] << 16), ow[2] | (ow[3] << 16));
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const u32 e = e0 + 128 * k + 4 * lane;
        const u32 valid = e >= ne ? 0u : (e + 4 <= ne ? 0xFu : ((1u << (ne - e)) - 1u));
        const u32 r0 = (u32)bf16_rne(m[k].x) | ((u32)bf16_rne(m[k].y) << 16);
        const u32 r1 = (u32)bf16_rne(m[k].z) | ((u32)bf16_rne(m[k].w) << 16);
        const u32 x0 = r0 ^ o[k].x, x1 = r1 ^ o[k].y;
        const u32 nib = (((x0 & 0xFFFFu) ? 1u : 0u) | ((x0 >> 16) ? 2u : 0u) | ((x1 & 0xFFFFu) ? 4u : 0u) |
                         ((x1 >> 16) ? 8u : 0u)) & valid;
        // sector of 16 elements = lanes 4s..4s+3: store it whole if any of them changed
        u32 sec = nib;
        sec |= __shfl_xor_sync(0xffffffffu, sec, 1);
        sec |= __shfl_xor_sync(0xffffffffu, sec, 2);
        if (sec) {
          if (vec && e + 4 <= ne) {
            *reinterpret_cast<uint2*>(Wt + e) = make_uint2(r0, r1);
          } else {
            const u16 rv[4] = {(u16)r0, (u16)(r0 >> 16), (u16)r1, (u16)(r1 >> 16)};
#pragma unroll
            for (u32 q = 0; q < 4; ++q)
              if (nib & (1u << q)) Wt[e + q] = rv[q];
          }
        }
        // word of 32 elements = lanes 8j..8j+7 (4 bits each)
        u32 word = nib << (4 * (lane & 7));
        word |= __shfl_xor_sync(0xffffffffu, word, 1);
        word |= __shfl_xor_sync(0xffffffffu, word, 2);
        word |= __shfl_xor_sync(0xffffffffu, word, 4);
        if ((lane & 7) == 0 && word) {
          u32* wp = bm + (e0 + 128 * k) / 32 + (lane >> 3);
          const u32 old = *wp;
          if ((old | word) != old) *wp = old | word;
        }
      }
    }
  }
}

__device__ __forceinline__ u32 block_sum32(u32 v, u32* s) {
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) s[warp] = v;
  __syncthreads();
  u32 t = lane < (blockDim.x >> 5) ? s[lane] : 0u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  __syncthreads();
  return t;
}

// exclusive block scan (kTT threads) of a u64, returns the block total
__device__ __forceinline__ u64 block_excl64(u64 v, u64* excl, u64* s) {
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u64 inc = warp_incl_scan64(v);
  if (lane == 31) s[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const u64 w = lane < (blockDim.x >> 5) ? s[lane] : 0;
    const u64 wi = warp_incl_scan64(w);
    s[lane] = wi - w;
    if (lane == 31) s[32] = wi;
  }
  __syncthreads();
  *excl = s[warp] + inc - v;
  const u64 tot = s[32];
  __syncthreads();
  return tot;
}

__global__ void __launch_bounds__(kTT) k_track_count(TrackArgs a) {
  __shared__ u32 s[32];
  for (u64 tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
    const u32 t = a.tile_tensor[tile];
    const u64 base = (tile - a.tile_prefix[t]) * kTile;
    const u32 nw = tile_words(a.numel[t], base);
    const u32* bm = a.bitmap + a.bm_off[t] + base / 32;
    const u32 w0 = 4 * threadIdx.x;
    u32 c = 0;
    if (w0 + 4 <= nw && (((uintptr_t)(bm + w0)) & 15u) == 0) {
      const uint4 v = *reinterpret_cast<const uint4*>(bm + w0);
      c = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
    } else {
      for (u32 w = w0; w < w0 + 4 && w < nw; ++w) c += __popc(bm[w]);
    }
    c = block_sum32(c, s);
    if (threadIdx.x == 0) a.tile_off[tile] = c;
  }
}

// per group of kGroup tiles: exclusive scan of the tile counts in place, group total into group_sum
__global__ void __launch_bounds__(kTT) k_track_scan_groups(TrackArgs a) {
  __shared__ u64 s[33];
  const u64 g0 = (u64)blockIdx.x * kGroup;
  u64 carry = 0;
  for (u32 r = 0; r < kGroup; r += kTT) {
    const u64 tile = g0 + r + threadIdx.x;
    const u64 v = tile < a.n_tiles ? a.tile_off[tile] : 0;
    u64 ex;
    const u64 tot = block_excl64(v, &ex, s);
    if (tile < a.n_tiles) a.tile_off[tile] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) a.group_sum[blockIdx.x] = carry;
}

// one CTA: exclusive scan of the group totals; totals / capacity
__global__ void __launch_bounds__(kTT) k_track_scan_top(TrackArgs a, u64 n_groups) {
  __shared__ u64 s[33];
  u64 carry = 0;
  for (u64 r = 0; r < n_groups; r += kTT) {
    const u64 g = r + threadIdx.x;
    const u64 v = g < n_groups ? a.group_sum[g] : 0;
    u64 ex;
    const u64 tot = block_excl64(v, &ex, s);
    if (g < n_groups) a.group_sum[g] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    a.group_sum[n_groups] = carry;
    a.totals[kTotNnz] = carry;
    if (carry > a.cap) latch(a.status, SYNC_ERR_CAPACITY);
  }
}

__device__ __forceinline__ u64 tile_offset(const TrackArgs& a, u64 tile) {
  if (tile >= a.n_tiles) return a.group_sum[(a.n_tiles + kGroup - 1) / kGroup];
  return a.group_sum[tile / kGroup] + a.tile_off[tile];
}

// per-tensor counts (and record offsets) from the tile offsets
__global__ void k_track_counts(TrackArgs a) {
  for (u32 t = blockIdx.x * blockDim.x + threadIdx.x; t < a.n_tensors; t += gridDim.x * blockDim.x)
    a.counts[t] = tile_offset(a, a.tile_prefix[t + 1]) - tile_offset(a, a.tile_prefix[t]);
}

// Thread i owns words 4i..4i+3 of the tile (one 16-byte load): one block scan per tile gives each thread its
// first output position, and its set bits are written in ascending element order.
__global__ void __launch_bounds__(kTT) k_track_write(TrackArgs a, u16* const* W, int clear) {
  __shared__ u64 s[33];
  const bool fits = tile_offset(a, a.n_tiles) <= a.cap;   // on overflow the set is kept for a retry
  for (u64 tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
    const u32 t = a.tile_tensor[tile];
    const u64 base = (tile - a.tile_prefix[t]) * kTile;
    const u32 nw = tile_words(a.numel[t], base);
    u32* bm = a.bitmap + a.bm_off[t] + base / 32;
    const u16* Wt = W[t];
    const u32 w0 = 4 * threadIdx.x;
    u32 wv[4] = {0, 0, 0, 0};
    const bool v16 = w0 + 4 <= nw && (((uintptr_t)(bm + w0)) & 15u) == 0;
    if (v16) {
      const uint4 v = *reinterpret_cast<const uint4*>(bm + w0);
      wv[0] = v.x, wv[1] = v.y, wv[2] = v.z, wv[3] = v.w;
    } else {
      for (u32 j = 0; j < 4; ++j)
        if (w0 + j < nw) wv[j] = bm[w0 + j];
    }
    const u32 c = __popc(wv[0]) + __popc(wv[1]) + __popc(wv[2]) + __popc(wv[3]);
    u64 ex;
    const u64 tot = block_excl64((u64)c, &ex, s);
    if (tot == 0) continue;
    u64 pos = tile_offset(a, tile) + ex;
    if (c && clear && fits) {
      if (v16) *reinterpret_cast<uint4*>(bm + w0) = make_uint4(0, 0, 0, 0);
      else
        for (u32 j = 0; j < 4; ++j)
          if (w0 + j < nw) bm[w0 + j] = 0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      u32 bits = wv[j];
      while (bits) {
        const u32 b = __ffs(bits) - 1;
        bits &= bits - 1;
        const u32 idx = (u32)(base + 32ull * (w0 + j) + b);
        if (pos < a.cap) {
          a.I[pos] = idx;
          a.V[pos] = Wt[idx];
        }
        ++pos;
      }
    }
  }
}

void launch_cast_track(const TrackArgs& a, const float* const* master, u16* const* W, int grid, cudaStream_t s) {
  if (!a.n_tiles) return;
  k_cast_track<<<grid, kTT, 0, s>>>(a, master, W);
  count_launch();
}

void launch_extract_tracked(const TrackArgs& a, u16* const* W, int clear, int grid, cudaStream_t s) {
  if (!a.n_tiles) {
    if (a.n_tensors) {
      k_track_counts<<<1, 256, 0, s>>>(a);
      count_launch();
    }
    return;
  }
  const u64 n_groups = (a.n_tiles + kGroup - 1) / kGroup;
  k_track_count<<<grid, kTT, 0, s>>>(a);
  k_track_scan_groups<<<(unsigned)n_groups, kTT, 0, s>>>(a);
  k_track_scan_top<<<1, kTT, 0, s>>>(a, n_groups);
  k_track_counts<<<(a.n_tensors + 255) / 256, 256, 0, s>>>(a);
  k_track_write<<<grid, kTT, 0, s>>>(a, W, clear);
  for (int i = 0; i < 5; ++i) count_launch();
}

}  // namespace ss
