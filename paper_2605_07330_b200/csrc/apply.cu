// apply.cu — K5/K6 plain scatter (rows a8 + a9; Alg. 3 l.6; snapshot
// commit after the transfer, P:300 / DESIGN C13).
//
// W[I[k]] <- V[k]. Scattered 2-byte stores: the cost is the partial-sector
// read-modify-write of every touched 32-byte sector (ncu: one 32 B DRAM read +
// one 32 B write per touched sector), not the I/V stream. Stores are fire-and-
// forget, so throughput is set by how many (I, V) loads each thread keeps in
// flight: every thread loads kU pairs before issuing its kU stores. (A full-
// sector read-merge-write variant measured 1.3-2.5x slower on B200: the L2's
// partial-write fill path is the better one.)
// The batched commit walks the raw (I, V) of sync_extract_batched chunk by
// chunk (one CTA per 16384 values; tensor found by a warp search over the
// chunk offsets of the plan).
#include "common.cuh"
#include "kernels.h"

namespace ss {

constexpr int kU = 8;  // (I, V) pairs in flight per thread

__global__ void __launch_bounds__(256) k_apply(u16* W, const u32* I, const u16* V, u64 count, u64 numel,
                                              u32* status) {
  const u64 stride = (u64)gridDim.x * blockDim.x * kU;
  bool bad = false;
  for (u64 k0 = (u64)blockIdx.x * blockDim.x * kU + threadIdx.x; k0 < count; k0 += stride) {
    u32 idx[kU];
    u16 val[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const u64 k = k0 + (u64)u * blockDim.x;
      idx[u] = k < count ? I[k] : 0xFFFFFFFFu;
      val[u] = k < count ? V[k] : (u16)0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const u64 k = k0 + (u64)u * blockDim.x;
      if (k < count) {
        if (idx[u] < numel) W[idx[u]] = val[u];
        else bad = true;
      }
    }
  }
  if (bad) latch(status, SYNC_ERR_INDEX_RANGE);
}

template <typename E>   // element type: u16 (BF16 / FP16) or u8 (FP8)
__global__ void __launch_bounds__(256) k_commit_batched(Plan p, u16* const* snaps, const u32* I, const u16* V) {
  // CTA per chunk; warp w takes the contiguous changes [w*2048, (w+1)*2048) of the
  // chunk (contiguous per-warp ranges measured 3-16% faster than CTA-strided ones
  // on B200: tools/scatter_bench.cu).
  __shared__ u32 s_t;
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr u32 kPerWarp = kChunk / 8;
  const u64 n_chunks = p.totals[kTotChunks];
  const u64* co = p.chunk_off;
  for (u64 g = blockIdx.x; g < n_chunks; g += gridDim.x) {
    if (warp == 0) {
      u32 t = warp_upper_search(p.n_tensors, g, [&](u32 i) { return co[i]; });
      if (lane == 0) s_t = t;
    }
    __syncthreads();
    const u32 t = s_t;
    const u64 nnz = p.rec_off[t + 1] - p.rec_off[t];
    const u64 p0 = (g - co[t]) * kChunk;
    const u32 nk = (u32)((nnz - p0) < kChunk ? (nnz - p0) : kChunk);
    const u32* Ir = I + p.rec_off[t] + p0;
    const u16* Vr = V + p.rec_off[t] + p0;
    E* S = reinterpret_cast<E*>(snaps[t]);
    const u64 lim = p.numel[t];
    bool bad = false;
    const u32 wb = warp * kPerWarp, we = wb + kPerWarp < nk ? wb + kPerWarp : nk;
    for (u32 q0 = wb + lane; q0 < we; q0 += 32 * kU) {
      u32 idx[kU];
      u16 val[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const u32 q = q0 + u * 32;
        idx[u] = q < we ? Ir[q] : 0xFFFFFFFFu;
        val[u] = q < we ? Vr[q] : (u16)0;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const u32 q = q0 + u * 32;
        if (q < we) {
          if (idx[u] < lim) S[idx[u]] = (E)val[u];
          else bad = true;
        }
      }
    }
    if (bad) latch(p.status, SYNC_ERR_INDEX_RANGE);
    __syncthreads();
  }
}

void launch_apply(u16* W, const u32* I, const u16* V, u64 count, u64 numel, u32* status, cudaStream_t s) {
  if (count == 0) return;
  u64 blocks = (count + 256 * kU - 1) / (256 * kU);
  int grid = (int)(blocks < 148ull * 8 ? blocks : 148ull * 8);
  k_apply<<<grid, 256, 0, s>>>(W, I, V, count, numel, status);
  count_launch();
}

void launch_commit_batched(const Plan& p, u16* const* snaps, const u32* I, const u16* V, int grid, cudaStream_t s) {
  if (p.dtype == SYNC_DTYPE_FP8) k_commit_batched<uint8_t><<<grid * 2, 256, 0, s>>>(p, snaps, I, V);
  else k_commit_batched<u16><<<grid * 2, 256, 0, s>>>(p, snaps, I, V);
  count_launch();
}

}  // namespace ss

