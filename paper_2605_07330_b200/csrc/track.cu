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
#include "tma.cuh"

namespace ss {

constexpr int kTT = 256;                         // threads per CTA
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

// TMA-fed persistent kernel (the K1 pattern): a producer warp streams each tile's fp32 masters and bf16
// weights in 4096-element stages (16 KB + 8 KB) into shared memory with cp.async.bulk + mbarrier
// complete_tx (L2 evict-first); 16 consumer warps take 256 elements of a stage each: lane l handles elements
// 128k + 4l (k = 0, 1) from shared memory, rounds to bf16, ORs the 4-bit change nibbles of the 8 lanes of a
// 32-element word (3 shuffles; lane 8j writes word j) and stores the 32-byte sectors (4 lanes) that changed.
constexpr int kCStages = 4;
constexpr u32 kCSub = 4096;                               // elements per stage
constexpr u32 kCStageBytes = kCSub * 6;                   // 16 KB fp32 + 8 KB bf16
constexpr int kCConsumers = 512;
constexpr int kCBlock = kCConsumers + 32;

struct CastInfo {
  const float* M;   // nullptr = no more work
  u16* W;
  u32* bm;
  u32 n_valid;
  u32 bulk;         // elements delivered by the bulk copies (multiple of 8)
};

__device__ __forceinline__ void cast_quad(const uint4& m, const uint2& o, u32 valid, u16* wdst, bool full,
                                          u32* word_dst, u32 lane) {
  const u32 r0 = (u32)bf16_rne(m.x) | ((u32)bf16_rne(m.y) << 16);
  const u32 r1 = (u32)bf16_rne(m.z) | ((u32)bf16_rne(m.w) << 16);
  const u32 x0 = r0 ^ o.x, x1 = r1 ^ o.y;
  const u32 nib = (((x0 & 0xFFFFu) ? 1u : 0u) | ((x0 >> 16) ? 2u : 0u) | ((x1 & 0xFFFFu) ? 4u : 0u) |
                   ((x1 >> 16) ? 8u : 0u)) & valid;
  u32 sec = nib;   // sector of 16 elements = lanes 4s..4s+3: stored whole if any of them changed
  sec |= __shfl_xor_sync(0xffffffffu, sec, 1);
  sec |= __shfl_xor_sync(0xffffffffu, sec, 2);
  if (sec) {
    if (full) {
      *reinterpret_cast<uint2*>(wdst) = make_uint2(r0, r1);
    } else {
      if (nib & 1u) wdst[0] = (u16)r0;
      if (nib & 2u) wdst[1] = (u16)(r0 >> 16);
      if (nib & 4u) wdst[2] = (u16)r1;
      if (nib & 8u) wdst[3] = (u16)(r1 >> 16);
    }
  }
  u32 word = nib << (4 * (lane & 7));   // word of 32 elements = lanes 8j..8j+7
  word |= __shfl_xor_sync(0xffffffffu, word, 1);
  word |= __shfl_xor_sync(0xffffffffu, word, 2);
  word |= __shfl_xor_sync(0xffffffffu, word, 4);
  // fire-and-forget OR (RED): no read round trip stalls the warp (a word has one writer per launch, the
  // atomic only avoids the load of a plain read-modify-write)
  if ((lane & 7) == 0 && word) atomicOr(word_dst, word);
}

__global__ void __launch_bounds__(kCBlock, 2) k_cast_track(TrackArgs a, const float* const* master,
                                                           u16* const* W) {
  extern __shared__ __align__(128) u8 smem[];
  u64* full = reinterpret_cast<u64*>(smem + kCStages * kCStageBytes);
  u64* empty = full + kCStages;
  CastInfo* info = reinterpret_cast<CastInfo*>(empty + kCStages);
  const u32 tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < kCStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kCConsumers / 32) {
    // ---------------------------------------------------------------- producer warp
    const u64 pol = policy_evict_first();
    u32 it = 0;
    for (u64 tile = blockIdx.x;; tile += gridDim.x) {
      const bool done = tile >= a.n_tiles;
      u32 t = 0;
      u64 base = 0, ne = 0;
      if (!done) {
        t = a.tile_tensor[tile];
        const u64 n = a.numel[t];
        base = (tile - a.tile_prefix[t]) * kTile;
        ne = (n - base) < kTile ? (n - base) : kTile;
      }
      const u32 n_sub = done ? 1u : (u32)((ne + kCSub - 1) / kCSub);
      const float* M0 = done ? nullptr : master[t] + base;
      u16* W0 = done ? nullptr : W[t] + base;
      u32* bm0 = done ? nullptr : a.bitmap + a.bm_off[t] + base / 32;
      const bool aligned = ((((uintptr_t)M0) | ((uintptr_t)W0)) & 15u) == 0;
      for (u32 sub = 0; sub < n_sub; ++sub, ++it) {
        const u32 s = it % kCStages;
        if (it >= (u32)kCStages) mbar_wait(&empty[s], ((it / kCStages) - 1) & 1);
        if (lane == 0) {
          CastInfo ci;
          if (done) {
            ci.M = nullptr;
            info[s] = ci;
            mbar_arrive(&full[s]);
          } else {
            const u64 e0 = (u64)sub * kCSub;
            const u32 nv = (u32)((ne - e0) < kCSub ? (ne - e0) : kCSub);
            ci.M = M0 + e0;
            ci.W = W0 + e0;
            ci.bm = bm0 + e0 / 32;
            ci.n_valid = nv;
            ci.bulk = aligned ? (nv & ~7u) : 0u;
            info[s] = ci;
            u8* dst = smem + (size_t)s * kCStageBytes;
            if (ci.bulk) {
              mbar_arrive_tx(&full[s], 6u * ci.bulk);
              bulk_g2s(dst, ci.M, 4u * ci.bulk, &full[s], pol);
              bulk_g2s(dst + 4 * kCSub, ci.W, 2u * ci.bulk, &full[s], pol);
            } else {
              mbar_arrive(&full[s]);
            }
          }
        }
        __syncwarp();
      }
      if (done) break;
    }
    return;
  }

  // ------------------------------------------------------------------ consumer warps
  for (u32 it = 0;; ++it) {
    const u32 s = it % kCStages;
    mbar_wait(&full[s], (it / kCStages) & 1);
    const CastInfo ci = info[s];
    if (ci.M == nullptr) break;
    const float* sm = reinterpret_cast<const float*>(smem + (size_t)s * kCStageBytes);
    const u16* sw = reinterpret_cast<const u16*>(smem + (size_t)s * kCStageBytes + 4 * kCSub);
    constexpr u32 kPerWarp = kCSub / (kCConsumers / 32);   // elements of a stage per consumer warp
#pragma unroll
    for (int k = 0; k < (int)(kPerWarp / 128); ++k) {
      const u32 e = kPerWarp * warp + 128 * k + 4 * lane;
      uint4 m = make_uint4(0, 0, 0, 0);
      uint2 o = make_uint2(0, 0);
      u32 valid = 0;
      bool fullq = false;
      if (e + 4 <= ci.bulk) {
        m = *reinterpret_cast<const uint4*>(sm + e);
        o = *reinterpret_cast<const uint2*>(sw + e);
        valid = 0xFu;
        fullq = true;
      } else if (e < ci.n_valid) {   // tail / unaligned: straight from global
        u32 mf[4] = {0, 0, 0, 0}, ow[4] = {0, 0, 0, 0};
#pragma unroll
        for (u32 q = 0; q < 4; ++q)
          if (e + q < ci.n_valid) {
            mf[q] = __float_as_uint(ci.M[e + q]);
            ow[q] = ci.W[e + q];
            valid |= 1u << q;
          }
        m = make_uint4(mf[0], mf[1], mf[2], mf[3]);
        o = make_uint2(ow[0] | (ow[1] << 16), ow[2] | (ow[3] << 16));
        fullq = false;
      }
      cast_quad(m, o, valid, ci.W + e, fullq, ci.bm + (kPerWarp * warp + 128 * k) / 32 + (lane >> 3), lane);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

static size_t cast_smem() { return (size_t)kCStages * kCStageBytes + 2 * kCStages * 8 + kCStages * sizeof(CastInfo); }

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
// first output position. A tile with at most kTW set bits (rho <= 25%) lists its tile-local indices in shared
// memory (each thread its own set bits, ascending, at its scan position), then all threads gather
// V = W[tile base + local] for consecutive list entries with kTG loads in flight per thread and store I / V
// coalesced — the gather is a random 32-byte-sector read, so it needs many loads in flight (a thread walking
// its own bits issued one dependent load at a time). Denser tiles take that per-thread walk.
constexpr u32 kTW = 8192;   // list capacity per tile (u16 local indices: 16 KB of shared memory)
constexpr int kTG = 4;      // gathers in flight per thread
template <bool k8>   // k8: 8-bit elements (FP8): V = the byte, zero-extended
__global__ void __launch_bounds__(kTT) k_track_write(TrackArgs a, u16* const* W, int clear) {
  __shared__ u64 s[33];
  __shared__ u16 s_idx[kTW];
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
    const u64 tot = block_excl64((u64)c, &ex, s);   // ends with a barrier: s_idx is free again
    if (tot == 0) continue;
    const u64 pos0 = tile_offset(a, tile);
    if (c && clear && fits) {
      if (v16) *reinterpret_cast<uint4*>(bm + w0) = make_uint4(0, 0, 0, 0);
      else
        for (u32 j = 0; j < 4; ++j)
          if (w0 + j < nw) bm[w0 + j] = 0;
    }
    if (tot <= kTW) {
      u32 q = (u32)ex;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        u32 bits = wv[j];
        while (bits) {
          const u32 b = __ffs(bits) - 1;
          bits &= bits - 1;
          s_idx[q++] = (u16)(32u * (w0 + j) + b);
        }
      }
      __syncthreads();
      const u32 n = (u32)tot;
      for (u32 e0 = 0; e0 < n; e0 += kTT * kTG) {
        u32 li[kTG];
        u16 v[kTG];
#pragma unroll
        for (int u = 0; u < kTG; ++u) {
          const u32 e = e0 + u * kTT + threadIdx.x;
          li[u] = e < n ? (u32)s_idx[e] : 0u;
          v[u] = e < n ? (k8 ? (u16)reinterpret_cast<const uint8_t*>(Wt)[base + li[u]] : Wt[base + li[u]]) : (u16)0;
        }
#pragma unroll
        for (int u = 0; u < kTG; ++u) {
          const u32 e = e0 + u * kTT + threadIdx.x;
          if (e < n && pos0 + e < a.cap) {
            a.I[pos0 + e] = (u32)(base + li[u]);
            a.V[pos0 + e] = v[u];
          }
        }
      }
      continue;   // the next tile's block scan starts with a barrier before s_idx is rewritten
    }
    u64 pos = pos0 + ex;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      u32 bits = wv[j];
      while (bits) {
        const u32 b = __ffs(bits) - 1;
        bits &= bits - 1;
        const u32 idx = (u32)(base + 32ull * (w0 + j) + b);
        if (pos < a.cap) {
          a.I[pos] = idx;
          a.V[pos] = k8 ? (u16)reinterpret_cast<const uint8_t*>(Wt)[idx] : Wt[idx];
        }
        ++pos;
      }
    }
  }
}

void launch_cast_track(const TrackArgs& a, const float* const* master, u16* const* W, int grid, cudaStream_t s) {
  if (!a.n_tiles) return;
  static int cap[kMaxDevices] = {};   // per device: the attribute is a per-device setting
  const size_t sm = cast_smem();
  const int dev = current_device();
  if (!cap[dev]) {
    cudaFuncSetAttribute(k_cast_track, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int n_sm = 148, per = 1;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cast_track, kCBlock, sm);
    cap[dev] = n_sm * (per > 0 ? per : 1);
  }
  const u64 lim = (u64)(grid < cap[dev] ? grid : cap[dev]);   // grid: the caller's (clamped) CTA budget
  const u64 g = a.n_tiles < lim ? a.n_tiles : lim;   // persistent, no cross-CTA waits
  k_cast_track<<<(unsigned)g, kCBlock, sm, s>>>(a, master, W);
  count_launch();
}

// FP8 extraction (f2, 8-bit elements): per tile, the change bitmap of old vs new (bitwise, C1) — thread
// owns 32-element words: two 16-byte loads of each array — then the tracked compaction below gathers
// V = new[I] (bytes).
__global__ void __launch_bounds__(kTT) k_diff8(TrackArgs a, const uint8_t* const* olds, const uint8_t* const* news) {
  for (u64 tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
    const u32 t = a.tile_tensor[tile];
    const u64 n = a.numel[t];
    const u64 base = (tile - a.tile_prefix[t]) * kTile;
    const u32 nw = tile_words(n, base);
    const uint8_t* O = olds[t] + base;
    const uint8_t* N = news[t] + base;
    u32* bm = a.bitmap + a.bm_off[t] + base / 32;
    const bool vec = ((((uintptr_t)O) | ((uintptr_t)N)) & 15u) == 0;
    for (u32 w = threadIdx.x; w < nw; w += kTT) {
      const u64 e0 = (u64)w * 32;
      u32 mask = 0;
      if (vec && base + e0 + 32 <= n) {
        const uint4* o4 = reinterpret_cast<const uint4*>(O + e0);
        const uint4* n4 = reinterpret_cast<const uint4*>(N + e0);
        const uint4 oa = o4[0], ob = o4[1], na = n4[0], nb = n4[1];
        const u32 x[8] = {oa.x ^ na.x, oa.y ^ na.y, oa.z ^ na.z, oa.w ^ na.w,
                          ob.x ^ nb.x, ob.y ^ nb.y, ob.z ^ nb.z, ob.w ^ nb.w};
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
          for (int b = 0; b < 4; ++b)
            mask |= (((x[j] >> (8 * b)) & 0xFFu) ? 1u : 0u) << (4 * j + b);
      } else {
        for (u32 k = 0; k < 32 && base + e0 + k < n; ++k) mask |= (O[e0 + k] != N[e0 + k] ? 1u : 0u) << k;
      }
      bm[w] = mask;
    }
  }
}

void launch_extract8(const TrackArgs& a, const uint8_t* const* olds, const uint8_t* const* news, int grid,
                     cudaStream_t s) {
  if (a.n_tiles) {
    k_diff8<<<grid, kTT, 0, s>>>(a, olds, news);
    count_launch();
  }
  launch_extract_tracked(a, (u16* const*)news, 0, grid, s, true);   // read-only: V = new[I]
}

void launch_extract_tracked(const TrackArgs& a, u16* const* W, int clear, int grid, cudaStream_t s, bool k8) {
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
  if (k8) k_track_write<true><<<grid, kTT, 0, s>>>(a, W, clear);
  else k_track_write<false><<<grid, kTT, 0, s>>>(a, W, clear);
  for (int i = 0; i < 5; ++i) count_launch();
}

}  // namespace ss
