// chunk.cuh — chunk helpers shared by K2 (chunk_stats) and K3 (encode).
//
// A chunk is up to 16384 values of one record: its position in
// the plan and the location of its rANS words in the scratch.
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace ss {

constexpr int kCThreads = 128;  // k_encode CTA size (one CTA per chunk)

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

__device__ __forceinline__ ChunkPos chunk_at(const Plan& p, const u64* counts, u64 g, u32 t, const u32* I,
                                             const u16* V) {
  ChunkPos c;
  c.t = t;
  c.nnz = counts[t];
  c.k = g - p.chunk_off[t];
  c.p0 = c.k * kChunk;
  c.nk = (u32)((c.nnz - c.p0) < kChunk ? (c.nnz - c.p0) : kChunk);
  c.Ir = I + p.rec_off[t];
  c.Vc = V + p.rec_off[t] + c.p0;
  return c;
}

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

}  // namespace ss
