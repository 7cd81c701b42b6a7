// plan.cu — K2: record plan for the §3.3 encodings (rows a2 + sizing of a3/a4).
//
// From the per-tensor counts of K1:
//  * k_plan_scan   (1 CTA)   value offsets, chunk offsets, totals (manifest order)
//  * k_chunk_stats (grid)    per chunk: max index gap (-> DELTA16/ABS32, P:360,
//                            DESIGN C4), hi-byte histogram, normalised rANS model
//                            and an encode pass that only counts renormalisation
//                            words -> exact hi block size and RAW/RANS decision
//                            (never-expand)
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

// One CTA per chunk: staged hi bytes + histogram + max gap (all threads), then
// the model and a counted rANS pass from shared memory (warp 0).
__device__ unsigned long long g_cprof[8];  // debug cycle counters (SS_CPROF=1)

__global__ void __launch_bounds__(kCThreads) k_chunk_stats(Plan p, const u32* I, const u16* V, const u64* counts) {
  __shared__ ChunkSmem sm;
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u64 n_chunks = p.totals[kTotChunks];
  for (u64 g = blockIdx.x; g < n_chunks; g += gridDim.x) {
    __syncthreads();  // shared memory of the previous chunk is free
    const long long t0 = clock64();
    const ChunkPos c = locate_chunk(p, counts, g, sm.t, I, V);
    const bool comp = p.codec == SYNC_CODEC_COMPRESSED;
    const long long t1 = clock64();
    const u32 gmax = stage_chunk(sm, c.Ir, c.Vc, c.p0, c.nk, true);
    const long long t2 = clock64();
    if (threadIdx.x == 0 && gmax) atomicMax(&p.maxgap[c.t], gmax);
    if (!comp || warp != 0) continue;
    const u32 nsym = warp_normalize(sm.m, c.nk);
    const long long t3 = clock64();
    // counted encode pass: steps G-1..0, renorm if x >= f * 2^20
    // encode pass: steps G-1..0, renorm if x >= f * 2^20. The words go to the
    // chunk's scratch in emission order and the final states + model to chunk_rhdr, so the
    // encode kernel only copies them into the record.
    u32 x = kLow, nwords = 0;
    const u32 G = (c.nk + 31) / 32;
    const u32 lt = (1u << lane) - 1u;
    const u32 wcap = c.nk / 2;
    u16* ws = p.word_scratch + chunk_words_base(p.rec_off[c.t] + c.p0, g);
    // symbol + model of the next step are loaded one step ahead (independent of x)
    auto fetch = [&](int gg, u32& s_, u32& fc_, u32& rc_) {
      const u32 q = (u32)gg * 32 + lane;
      s_ = (gg >= 0 && q < c.nk) ? (u32)sm.hi[q] : 0x100u;
      fc_ = s_ < 256 ? sm.m.fc[s_] : 0u;
      rc_ = s_ < 256 ? sm.m.rcp[s_] : 0u;
    };
    u32 ns, nfc, nrc;
    fetch((int)G - 1, ns, nfc, nrc);
    for (int gg = (int)G - 1; gg >= 0; --gg) {
      const u32 s = ns, fcs = nfc, rcp = nrc;
      fetch(gg - 1, ns, nfc, nrc);
      const bool act = s < 256;
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
    u32* rh = p.chunk_rhdr + (u64)g * kRhdrWords;
    rh[lane] = x;
    if (lane == 0) {
      rh[32] = nwords;
      rh[33] = nsym;
    }
    {
      u32 present = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) present += sm.m.freq[lane * 8 + j] ? 1u : 0u;
      u32 rank = warp_incl_scan(present) - present;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const u32 s = lane * 8 + j;
        const u32 f = sm.m.freq[s];
        if (f) rh[34 + rank++] = s | (f << 16);
      }
    }
    u32 hb = 136u + 4u * nsym + 2u * nwords;
    u32 mode = 1;
    if (hb >= c.nk) {
      hb = c.nk;
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
  k_chunk_stats<<<grid, kCThreads, 0, s>>>(q, I, V, counts);
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
