// chunk.cuh — CTA-per-chunk staging shared by K2 (chunk_stats) and K3 (encode).
//
// A chunk is up to 16384 values of one record. 256 threads stage
// its hi bytes (V >> 8) in shared memory while building the byte histogram
// (per-warp sub-histograms with shared-memory atomics, then merged) and the chunk's maximum first
// difference ("prepending a zero": Δ_0 = I_0); warp 0 then normalises
// the model and runs the serial 32-lane rANS pass from shared
// memory.
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace ss {

constexpr int kCThreads = 128;  // small CTAs: more concurrent serial rANS warps per SM

struct ChunkSmem {
  u8 hi[kChunk];                  // staged hi bytes
  u32 sub_hist[kCThreads / 32][256];
  WarpModel m;                    // merged histogram + model (warp 0)
  u32 t;                          // tensor of the chunk
  u32 gmax[kCThreads / 32];
};

struct ChunkPos {
  u32 t;
  u64 nnz, k, p0;
  u32 nk;
  const u32* Ir;                  // record's I
  const u16* Vc;                  // chunk's V
};

// Renormalisation words of chunk g (first value at global position vpos) live at
// word_scratch[vpos / 2 + g ...]: a chunk keeping its rANS block has fewer than
// n_k / 2 words, so consecutive chunks never overlap.
__device__ __forceinline__ u64 chunk_words_base(u64 vpos, u64 g) { return vpos / 2 + g; }

// Locate chunk g (warp 0 searches the chunk offsets) — all threads get the same.
__device__ __forceinline__ ChunkPos locate_chunk(const Plan& p, const u64* counts, u64 g, u32& s_t,
                                                 const u32* I, const u16* V) {
  const u32 warp = threadIdx.x >> 5;
  if (warp == 0) {
    const u64* co = p.chunk_off;
    const u32 t = warp_upper_search(p.n_tensors, g, [&](u32 i) { return co[i]; });
    if ((threadIdx.x & 31) == 0) s_t = t;
  }
  __syncthreads();
  ChunkPos c;
  c.t = s_t;
  c.nnz = counts[c.t];
  c.k = g - p.chunk_off[c.t];
  c.p0 = c.k * kChunk;
  c.nk = (u32)((c.nnz - c.p0) < kChunk ? (c.nnz - c.p0) : kChunk);
  c.Ir = I + p.rec_off[c.t];
  c.Vc = V + p.rec_off[c.t] + c.p0;
  return c;
}

// Stage hi bytes + histogram (+ optional max gap). Ends with __syncthreads();
// on return sm.m.hist holds the merged histogram and (if want_gap) the max gap
// is returned to every thread.
__device__ __forceinline__ u32 stage_chunk(ChunkSmem& sm, const u32* Ir, const u16* Vc, u64 p0, u32 nk,
                                           bool want_gap) {
  const u32 tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  u32* h = sm.sub_hist[warp];
  for (u32 s = lane; s < 256; s += 32) h[s] = 0;
  __syncwarp();
  u32 gmax = 0;
  constexpr int kU = 8;
  for (u32 b0 = 0; b0 < nk; b0 += kCThreads * kU) {  // CTA-uniform trip count (shuffles below)
    const u32 q0 = b0 + tid;
    u16 v[kU];
    u32 cur[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const u32 q = q0 + u * kCThreads;
      const bool act = q < nk;
      v[u] = act ? Vc[q] : (u16)0;
      if (want_gap) cur[u] = act ? Ir[p0 + q] : 0u;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const u32 q = q0 + u * kCThreads;
      const bool act = q < nk;
      if (act) {
        const u32 s = v[u] >> 8;
        sm.hi[q] = (u8)s;
        atomicAdd(&h[s], 1u);
      }
      if (want_gap) {
        // previous index: the neighbour lane's, except lane 0 which loads it
        u32 prev = __shfl_up_sync(0xffffffffu, cur[u], 1);
        if (lane == 0) prev = (act && (p0 + q)) ? Ir[p0 + q - 1] : 0u;
        if (act) {
          const u32 d = cur[u] - ((p0 + q) ? prev : 0u);
          gmax = d > gmax ? d : gmax;
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const u32 x = __shfl_xor_sync(0xffffffffu, gmax, o);
    gmax = x > gmax ? x : gmax;
  }
  if (lane == 0) sm.gmax[warp] = gmax;
  __syncthreads();
  // merge the sub-histograms (256 bins, one per thread) and the gap maxima
  for (u32 bin = tid; bin < 256; bin += kCThreads) {
    u32 sum = 0;
#pragma unroll
    for (int w = 0; w < kCThreads / 32; ++w) sum += sm.sub_hist[w][bin];
    sm.m.hist[bin] = sum;
  }
  u32 g = 0;
#pragma unroll
  for (int w = 0; w < kCThreads / 32; ++w) g = sm.gmax[w] > g ? sm.gmax[w] : g;
  __syncthreads();
  return g;
}

}  // namespace ss
