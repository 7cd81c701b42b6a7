// plan.cu — K2: record plan for the §3.3 encodings (rows a2 + sizing of a3/a4).
//
// From the per-tensor counts of K1:
//  * k_plan_scan   (1 CTA)   value offsets, chunk offsets, totals (manifest order)
//  * k_chunk_stats (grid)    per chunk: max index gap (-> DELTA16/ABS32, P:360,
//                            DESIGN C4), hi-byte histogram, normalised rANS model
//                            and the rANS encode pass -> exact hi block size and
//                            RAW/RANS decision (never-expand); words, states
//                            and model kept in scratch for k_encode
//  * k_plan_sizes  (1 CTA)   chunk hi-offset prefix, record sizes,
//                            record byte offsets, statistics
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "chunk.cuh"

namespace ss {

constexpr int kScanThreads = 1024;

// Block-wide exclusive scan of a u64 (1024 threads); returns the block total.
__device__ __forceinline__ u64 block_excl_scan64(u64 v, u64* excl, u64* s_w) {
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u64 inc = warp_incl_scan64(v);
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    u64 w = s_w[lane];
    u64 wi = warp_incl_scan64(w);
    s_w[lane] = wi - w;
    if (lane == 31) s_w[32] = wi;
  }
  __syncthreads();
  *excl = s_w[warp] + inc - v;
  u64 total = s_w[32];
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(kScanThreads) k_plan_scan(Plan p, const u64* counts) {
  __shared__ u64 s_w[33];
  __shared__ u64 s_w2[33];
  u64 carry_nnz = 0, carry_ch = 0, carry_rec = 0;
  const u32 T = p.n_tensors;
  for (u32 b = 0; b < T; b += kScanThreads) {
    u32 t = b + threadIdx.x;
    u64 c = t < T ? counts[t] : 0;
    u64 ch = (c + kChunk - 1) / kChunk;
    u64 packed = (ch << 32) | (c ? 1u : 0u);   // chunks (< 2^32 total) | record flag
    u64 e1, e2;
    u64 tot1 = block_excl_scan64(c, &e1, s_w);
    u64 tot2 = block_excl_scan64(packed, &e2, s_w2);
    if (t < T) {
      p.rec_off[t] = carry_nnz + e1;
      p.chunk_off[t] = carry_ch + (e2 >> 32);
      p.maxgap[t] = 0;
    }
    carry_nnz += tot1;
    carry_ch += tot2 >> 32;
    carry_rec += tot2 & 0xFFFFFFFFull;
  }
  if (threadIdx.x == 0) {
    p.rec_off[T] = carry_nnz;
    p.chunk_off[T] = carry_ch;
    bool over = carry_nnz > p.cap || carry_ch > p.max_chunks;
    if (over) latch(p.status, SYNC_ERR_CAPACITY);
    for (int k = 0; k < 16; ++k) p.totals[k] = 0;
    p.totals[kTotNnz] = carry_nnz;
    p.totals[kTotChunks] = over ? 0 : carry_ch;
    p.totals[kTotRecords] = carry_rec;
    p.totals[kTotOverflow] = over ? 1 : 0;
  }
}

__device__ unsigned long long g_cprof[8];  // debug cycle counters (SS_CPROF=1)

// One warp per chunk: the warp builds its chunk's histogram + max first difference (8
// loads in flight per lane, per-warp shared histogram), normalises the model, then runs
// the rANS encode pass reading V from L2 with the next 8 steps prefetched into registers
// (words to the chunk's scratch in emission order; final states + model to chunk_rhdr).
// No hi plane in shared memory: ~32 independent rANS chains per SM (a CTA-per-chunk
// variant with the hi plane staged in shared memory measured 1.2-1.7x slower).
constexpr int kWPF = 8;
__global__ void __launch_bounds__(256) k_chunk_stats(Plan p, const u32* I, const u16* V, const u64* counts) {
  __shared__ WarpModel s_m[8];
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpModel& m = s_m[warp];
  const u64 n_chunks = p.totals[kTotChunks];
  const u64 nwarps = (u64)gridDim.x * 8;
  const bool comp = p.codec == SYNC_CODEC_COMPRESSED;
  for (u64 g = (u64)blockIdx.x * 8 + warp; g < n_chunks; g += nwarps) {
    const long long t0 = clock64();
    const u64* co = p.chunk_off;
    const u32 t = warp_upper_search(p.n_tensors, g, [&](u32 i) { return co[i]; });
    const u64 nnz = counts[t];
    const u64 p0 = (g - co[t]) * kChunk;
    const u32 nk = (u32)((nnz - p0) < kChunk ? (nnz - p0) : kChunk);
    const u32* Ir = I + p.rec_off[t];
    const u16* Vc = V + p.rec_off[t] + p0;
    const long long t1 = clock64();
    // ---- histogram + max first difference
    for (u32 sym = lane; sym < 256; sym += 32) m.hist[sym] = 0;
    __syncwarp();
    u32 gmax = 0;
    for (u32 b0 = 0; b0 < nk; b0 += 32 * kWPF) {
      u32 hv[kWPF], cur[kWPF];
#pragma unroll
      for (int u = 0; u < kWPF; ++u) {
        const u32 q = b0 + u * 32 + lane;
        hv[u] = q < nk ? (u32)(Vc[q] >> 8) : 0x100u;
        cur[u] = q < nk ? Ir[p0 + q] : 0u;
      }
#pragma unroll
      for (int u = 0; u < kWPF; ++u) {
        const u32 q = b0 + u * 32 + lane;
        if (hv[u] < 256) atomicAdd(&m.hist[hv[u]], 1u);
        u32 prev = __shfl_up_sync(0xffffffffu, cur[u], 1);
        if (lane == 0) prev = (p0 + q) ? Ir[p0 + q - 1] : 0u;
        if (q < nk) {
          const u32 d = cur[u] - prev;
          gmax = d > gmax ? d : gmax;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const u32 x = __shfl_xor_sync(0xffffffffu, gmax, o);
      gmax = x > gmax ? x : gmax;
    }
    if (lane == 0 && gmax) atomicMax(&p.maxgap[t], gmax);
    __syncwarp();
    const long long t2 = clock64();
    if (!comp) continue;
    const u32 nsym = warp_normalize(m, nk);
    const long long t3 = clock64();
    // ---- counted rANS pass (words -> scratch in emission order; states/model -> chunk_rhdr)
    u32 x = kLow, nwords = 0;
    const u32 G = (nk + 31) / 32;
    const u32 lt = (1u << lane) - 1u;
    const u32 wcap = nk / 2;
    u16* ws = p.word_scratch + chunk_words_base(p.rec_off[t] + p0, g);
    u32 nxt[kWPF];
    auto load_block = [&](int top, u32* dst) {  // steps top, top-1, ..., top-7
#pragma unroll
      for (int u = 0; u < kWPF; ++u) {
        const int gg = top - u;
        const u32 q = (u32)gg * 32 + lane;
        dst[u] = (gg >= 0 && q < nk) ? (u32)(Vc[q] >> 8) : 0x100u;
      }
    };
    load_block((int)G - 1, nxt);
    for (int top = (int)G - 1; top >= 0; top -= kWPF) {
      u32 cur[kWPF];
#pragma unroll
      for (int u = 0; u < kWPF; ++u) cur[u] = nxt[u];
      if (top - kWPF >= 0) load_block(top - kWPF, nxt);
#pragma unroll
      for (int u = 0; u < kWPF; ++u) {
        if (top - u < 0) break;
        const u32 sym = cur[u];
        const bool act = sym < 256;
        const u32 fcs = act ? m.fc[sym] : 0u, rcp = act ? m.rcp[sym] : 0u;
        const u32 f = fcs & 0xFFFFu;
        const bool emit = act && (x >> 20) >= f;
        const u32 em = __ballot_sync(0xffffffffu, emit);
        if (emit) {
          const u32 e = nwords + __popc(em & lt);
          if (e < wcap) ws[e] = (u16)(x & 0xFFFFu);
          x >>= 16;
        }
        nwords += __popc(em);
        if (act) {
          u32 r;
          const u32 qq = div_by(x, f, rcp, &r);
          x = qq * kM + r + (fcs >> 16);
        }
      }
    }
    u32* rh = p.chunk_rhdr + g * kRhdrWords;
    rh[lane] = x;
    if (lane == 0) {
      rh[32] = nwords;
      rh[33] = nsym;
    }
    {
      u32 present = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) present += m.freq[lane * 8 + j] ? 1u : 0u;
      u32 rank = warp_incl_scan(present) - present;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const u32 sym = lane * 8 + j;
        const u32 f = m.freq[sym];
        if (f) rh[34 + rank++] = sym | (f << 16);
      }
    }
    u32 hb = 136u + 4u * nsym + 2u * nwords;
    u32 mode = 1;
    if (hb >= nk) {
      hb = nk;
      mode = 0;
    }
    if (lane == 0) {
      p.chunk_hi[g] = hb;
      p.chunk_mode[g] = mode;
      if (p.prof) {
        const long long t4 = clock64();
        atomicAdd(&g_cprof[0], (unsigned long long)(t1 - t0));
        atomicAdd(&g_cprof[1], (unsigned long long)(t2 - t1));
        atomicAdd(&g_cprof[2], (unsigned long long)(t3 - t2));
        atomicAdd(&g_cprof[3], (unsigned long long)(t4 - t3));
        atomicAdd(&g_cprof[4], 1ull);
      }
    }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(kScanThreads) k_plan_sizes(Plan p, const u64* counts) {
  __shared__ u64 s_w[33];
  __shared__ u64 s_w2[33];
  const u32 T = p.n_tensors;
  const bool comp = p.codec == SYNC_CODEC_COMPRESSED;
  const u64 n_chunks = p.totals[kTotChunks];
  const bool over = p.totals[kTotOverflow] != 0;
  // 1. exclusive prefix of padded hi block sizes over all chunks (+ RANS chunk count)
  u64 carry = 0, rans = 0;
  if (comp) {
    for (u64 b = 0; b < n_chunks; b += kScanThreads) {
      u64 g = b + threadIdx.x;
      u64 v = g < n_chunks ? pad_to(p.chunk_hi[g], 4) : 0;
      u64 r = g < n_chunks ? p.chunk_mode[g] : 0;
      u64 e, e2;
      u64 tot = block_excl_scan64(v, &e, s_w);
      u64 tr = block_excl_scan64(r, &e2, s_w2);
      if (g < n_chunks) p.chunk_hioff[g] = carry + e;
      carry += tot;
      rans += tr;
    }
    if (threadIdx.x == 0) p.chunk_hioff[n_chunks] = carry;
    __syncthreads();
  }
  // 2. record sizes and offsets
  u64 carry_enc = 0, n16 = 0, n32 = 0, ib_tot = 0, vb_tot = 0;
  for (u32 b = 0; b < T; b += kScanThreads) {
    u32 t = b + threadIdx.x;
    u64 c = (t < T && !over) ? counts[t] : 0;
    u64 bytes = 0, ib = 0;
    u32 mode = 1;
    if (c) {
      if (comp) {
        mode = p.maxgap[t] <= 32767u ? 0u : 1u;
        ib = pad_to((mode ? 4 : 2) * c, 4);
        u64 ch0 = p.chunk_off[t], ch1 = p.chunk_off[t + 1];
        u64 hi = p.chunk_hioff[ch1] - p.chunk_hioff[ch0];
        bytes = pad_to(16 + ib + pad_to(c, 4) + 16 * (ch1 - ch0) + hi, 16);
      } else {
        ib = 4 * c;
        bytes = pad_to(16 + 6 * c, 16);
      }
    }
    if (t < T) {
      p.rec_mode[t] = mode;
      p.rec_bytes[t] = bytes;
    }
    u64 e;
    u64 tot = block_excl_scan64(bytes, &e, s_w);
    if (t < T) p.enc_off[t] = carry_enc + e;
    carry_enc += tot;
    u64 flags = c ? (mode ? (1ull << 32) : 1ull) : 0ull;
    u64 e2;
    u64 tf = block_excl_scan64(flags, &e2, s_w2);
    n16 += tf & 0xFFFFFFFFull;
    n32 += tf >> 32;
    u64 e3;
    ib_tot += block_excl_scan64(ib, &e3, s_w);
    u64 e4;
    vb_tot += block_excl_scan64(c ? bytes - 16 - ib : 0, &e4, s_w2);
  }
  if (threadIdx.x == 0) {
    p.enc_off[T] = carry_enc;
    if (carry_enc > p.enc_cap) {
      latch(p.status, SYNC_ERR_CAPACITY);
      p.totals[kTotOverflow] = 1;
      p.totals[kTotChunks] = 0;   // nothing gets encoded
    }
    p.totals[kTotEnc] = carry_enc;
    p.totals[kTotDelta16] = comp ? n16 : 0;
    p.totals[kTotAbs32] = comp ? n32 : n16 + n32;
    p.totals[kTotRansChunks] = rans;
    p.totals[kTotIndexBytes] = ib_tot;
    p.totals[kTotValueBytes] = vb_tot;
  }
}

void launch_plan_scan(const Plan& p, const u64* counts, cudaStream_t s) {
  k_plan_scan<<<1, kScanThreads, 0, s>>>(p, counts);
  count_launch();
}

void launch_chunk_stats(const Plan& p, const u32* I, const u16* V, const u64* counts, int grid, cudaStream_t s) {
  static int want = -1;
  if (want < 0) want = getenv("SS_CPROF") ? 1 : 0;
  Plan q = p;
  q.prof = want;
  if (want) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbolAsync(g_cprof, z, sizeof(z), 0, cudaMemcpyHostToDevice, s);
  }
  k_chunk_stats<<<grid, 256, 0, s>>>(q, I, V, counts);
  if (want) {
    unsigned long long h[8];
    cudaMemcpyFromSymbolAsync(h, g_cprof, sizeof(h), 0, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const double n = h[4] ? (double)h[4] : 1.0;
    fprintf(stderr, "[cprof] chunks %llu per-chunk cycles: locate %.0f stage %.0f normalize %.0f rans %.0f\n", h[4],
            h[0] / n, h[1] / n, h[2] / n, h[3] / n);
  }
  count_launch();
}

void launch_plan_sizes(const Plan& p, const u64* counts, cudaStream_t s) {
  k_plan_sizes<<<1, kScanThreads, 0, s>>>(p, counts);
  count_launch();
}

}  // namespace ss
