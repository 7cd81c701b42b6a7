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

constexpr int kPerScan = 8;   // tensors per thread per round (one block scan pair per 8192 tensors)
__global__ void __launch_bounds__(kScanThreads) k_plan_scan(Plan p, const u64* counts) {
  __shared__ u64 s_w[33];
  __shared__ u64 s_w2[33];
  u64 carry_nnz = 0, carry_ch = 0, carry_rec = 0;
  const u32 T = p.n_tensors;
  constexpr u32 kRound = kScanThreads * kPerScan;
  for (u32 b = 0; b < T; b += kRound) {
    const u32 t0 = b + threadIdx.x * kPerScan;
    u64 c[kPerScan];
    u64 s1 = 0, s2 = 0;
#pragma unroll
    for (int k = 0; k < kPerScan; ++k) {
      const u32 t = t0 + k;
      c[k] = t < T ? counts[t] : 0;
      s1 += c[k];
      s2 += (((c[k] + kChunk - 1) / kChunk) << 32) | (c[k] ? 1u : 0u);   // chunks (< 2^32 total) | record flag
    }
    u64 e1, e2;
    const u64 tot1 = block_excl_scan64(s1, &e1, s_w);
    const u64 tot2 = block_excl_scan64(s2, &e2, s_w2);
    u64 r1 = carry_nnz + e1, r2 = carry_ch + (e2 >> 32);
#pragma unroll
    for (int k = 0; k < kPerScan; ++k) {
      const u32 t = t0 + k;
      if (t < T) {
        p.rec_off[t] = r1;
        p.chunk_off[t] = r2;
        p.maxgap[t] = 0;
      }
      r1 += c[k];
      r2 += (c[k] + kChunk - 1) / kChunk;
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
    p.work[0] = 0;   // chunk counters of k_chunk_stats / k_encode
    p.work[1] = 0;
    p.totals[kTotNnz] = carry_nnz;
    p.totals[kTotChunks] = over ? 0 : carry_ch;
    p.totals[kTotRecords] = carry_rec;
    p.totals[kTotOverflow] = over ? 1 : 0;
  }
}

__device__ unsigned long long g_cprof[8];  // debug cycle counters (SS_CPROF=1)

// One warp per chunk: the warp builds its chunk's histogram + max first difference, normalises the model,
// then runs the rANS encode pass reading V from L2 with the next 8 steps prefetched into registers (words to
// the chunk's scratch in emission order; final states + model to chunk_rhdr). No hi plane in shared memory:
// ~32 independent rANS chains per SM (a CTA-per-chunk variant with the hi plane staged in shared memory
// measured 1.2-1.7x slower). Persistent grid (the resident CTAs); each warp claims its next chunk from a
// counter, so no CTA waits for its slowest warp and there is no tail of partial waves.
// Histogram / gap pass: lane l owns the 8 consecutive values of an 8-aligned group (one 16-byte load of V,
// two of I); the gap into the group comes from lane l-1's last index (one shuffle), the warp's carry from
// the previous round.
constexpr int kWPF = 8;
__global__ void __launch_bounds__(256, 4) k_chunk_stats(Plan p, const u32* I, const u16* V, const u64* counts) {
  __shared__ WarpModel s_m[8];
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpModel& m = s_m[warp];
  const u64 n_chunks = p.totals[kTotChunks];
  const bool comp = p.codec == SYNC_CODEC_COMPRESSED;
  // the coded value plane: the hi byte of a 16-bit element, the whole byte of an FP8 one (V's low half)
  const u32 sh = p.dtype == SYNC_DTYPE_FP8 ? 0u : 8u;
  for (;;) {
    u64 g = 0;
    if (lane == 0) g = atomicAdd(reinterpret_cast<unsigned long long*>(p.work), 1ull);
    g = __shfl_sync(0xffffffffu, g, 0);
    if (g >= n_chunks) break;
    const long long t0 = clock64();
    const u64* co = p.chunk_off;
    const u32 t = warp_upper_search(p.n_tensors, g, [&](u32 i) { return co[i]; });
    const u64 nnz = counts[t];
    const u64 p0 = (g - co[t]) * kChunk;
    const u32 nk = (u32)((nnz - p0) < kChunk ? (nnz - p0) : kChunk);
    const u64 gs = p.rec_off[t] + p0, ge = gs + nk;   // the chunk's values in I / V
    const u16* Vc = V + gs;
    const long long t1 = clock64();
    for (u32 sym = lane; sym < 256; sym += 32) m.hist[sym] = 0;
    __syncwarp();
    // I of the element before the chunk (Δ_0 = I_0 when the chunk starts its record)
    u32 carry0 = (lane == 0 && p0) ? I[gs - 1] : 0u;
    carry0 = __shfl_sync(0xffffffffu, carry0, 0);
    u32 carry = carry0;
    u32 gmax = 0, nesc = 0;
    for (u64 e0 = gs & ~7ull; e0 < ge; e0 += 256) {
      const u64 e = e0 + 8ull * lane;
      u32 iv[8], hv[8];
      if (e < ge && e + 8 <= p.cap) {   // a whole 8-group inside the I / V arrays (values outside the chunk
                                        // are loaded and masked below)
        const uint4 va = *reinterpret_cast<const uint4*>(V + e);
        const uint4 ia = *reinterpret_cast<const uint4*>(I + e);
        const uint4 ib = *reinterpret_cast<const uint4*>(I + e + 4);
        const u32 vw[4] = {va.x, va.y, va.z, va.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          hv[2 * k] = (vw[k] >> sh) & 0xFFu;
          hv[2 * k + 1] = (vw[k] >> (16 + sh)) & 0xFFu;
        }
        iv[0] = ia.x; iv[1] = ia.y; iv[2] = ia.z; iv[3] = ia.w;
        iv[4] = ib.x; iv[5] = ib.y; iv[6] = ib.z; iv[7] = ib.w;
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const bool in = e + k >= gs && e + k < ge;
          iv[k] = in ? I[e + k] : 0u;
          hv[k] = in ? ((u32)V[e + k] >> sh) & 0xFFu : 0u;
        }
      }
      u32 prev = __shfl_up_sync(0xffffffffu, iv[7], 1);
      if (lane == 0) prev = carry;
      carry = __shfl_sync(0xffffffffu, iv[7], 31);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const u64 q = e + k;
        if (q >= gs && q < ge) {
          atomicAdd(&m.hist[hv[k]], 1u);
          const u32 d = iv[k] - (q == gs ? carry0 : (k ? iv[k - 1] : prev));
          gmax = d > gmax ? d : gmax;
          nesc += d > 32767u ? 1u : 0u;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const u32 x = __shfl_xor_sync(0xffffffffu, gmax, o);
      gmax = x > gmax ? x : gmax;
    }
    if (lane == 0 && gmax) atomicMax(&p.maxgap[t], gmax);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nesc += __shfl_xor_sync(0xffffffffu, nesc, o);
    if (lane == 0) p.chunk_esc[g] = nesc;   // f4: gaps that need an escape word
    __syncwarp();
    const long long t2 = clock64();
    if (!comp) continue;
    const u32 nsym = warp_normalize(m, nk);
    const long long t3 = clock64();
    // ---- counted rANS pass (words -> scratch in emission order; states/model -> chunk_rhdr).
    //      Branch-free steps: positions past the chunk end use the no-op symbol 256; the state update is
    //      x' = x + q * (M - f) + cum with q = floor(x / f) (= floor(x/f) * M + x mod f + cum).
    u32 x = kLow, nwords = 0;
    const u32 G = (nk + 31) / 32;
    const u32 lt = (1u << lane) - 1u;
    const u32 wcap = nk / 2;
    u16* ws = p.word_scratch + chunk_words_base(gs, g);
    const u8* Vb = reinterpret_cast<const u8*>(Vc) + (sh ? 1 : 0);   // byte 2q + vb: the coded byte of V[q]
    asm volatile("" : "+l"(ws));   // keep the 64-bit base in registers (no per-step rematerialisation)
    const uint2* const fr = m.fr;
    u32 nxt[kWPF];
    auto load_block = [&](int top, u32* dst) {  // steps top, top-1, ..., top-7
      if (top >= kWPF - 1 && (u32)(top + 1) * 32 <= nk) {   // all 8 steps full
        const u8* vp = Vb + 2 * ((u32)top * 32 + lane);
#pragma unroll
        for (int u = 0; u < kWPF; ++u) dst[u] = vp[-64 * u];
        return;
      }
#pragma unroll
      for (int u = 0; u < kWPF; ++u) {
        const int gg = top - u;
        const u32 q = (u32)gg * 32 + lane;
        dst[u] = (gg >= 0 && q < nk) ? (u32)Vb[2 * q] : 0x100u;
      }
    };
    load_block((int)G - 1, nxt);
    for (int top = (int)G - 1; top >= 0; top -= kWPF) {
      u32 cs[kWPF];
#pragma unroll
      for (int u = 0; u < kWPF; ++u) cs[u] = nxt[u];
      if (top - kWPF >= 0) load_block(top - kWPF, nxt);
#pragma unroll
      for (int u = 0; u < kWPF; ++u) {
        const uint2 e2 = fr[cs[u]];
        const u32 f = e2.x & 0xFFFFu;
        const bool emit = (x >> 20) >= f;
        const u32 em = __ballot_sync(0xffffffffu, emit);
        const u32 e = nwords + __popc(em & lt);
        if (emit && e < wcap) ws[e] = (u16)(x & 0xFFFFu);
        x = emit ? (x >> 16) : x;
        nwords += __popc(em);
        u32 q = __umulhi(x, e2.y);
        q += (x - q * f) >= f ? 1u : 0u;
        x = x + q * ((u32)kM - f) + (e2.x >> 16);
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

// Block-wide sum of a u64 (1024 threads); every thread gets the total.
__device__ __forceinline__ u64 block_sum64(u64 v, u64* s_w) {
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) s_w[warp] = v;
  __syncthreads();
  u64 t = s_w[lane];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  __syncthreads();
  return t;
}

// Single CTA; every thread owns kPer consecutive items per round, so a round covers 8192 chunks or tensors
// with one block scan (30B: 3 rounds over the chunks, 3 over the tensors).
constexpr int kPer = 8;
__global__ void __launch_bounds__(kScanThreads) k_plan_sizes(Plan p, const u64* counts) {
  __shared__ u64 s_w[33];
  __shared__ u64 s_w2[33];
  const u32 T = p.n_tensors;
  const bool comp = p.codec == SYNC_CODEC_COMPRESSED;
  const bool e8 = p.dtype == SYNC_DTYPE_FP8;
  const u64 n_chunks = p.totals[kTotChunks];
  const bool over = p.totals[kTotOverflow] != 0;
  constexpr u64 kRound = (u64)kScanThreads * kPer;
  // 1. exclusive prefix of padded hi block sizes over all chunks (+ RANS chunk count)
  u64 carry = 0, rans_local = 0, ecarry = 0;
  if (comp) {
    for (u64 b = 0; b < n_chunks; b += kRound) {
      const u64 g0 = b + (u64)threadIdx.x * kPer;
      u64 v[kPer], es[kPer];
      u64 sum = 0, esum = 0;
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const u64 g = g0 + k;
        v[k] = g < n_chunks ? pad_to(p.chunk_hi[g], 4) : 0;
        es[k] = (p.escape && g < n_chunks) ? p.chunk_esc[g] : 0;
        rans_local += g < n_chunks ? p.chunk_mode[g] : 0;
        sum += v[k];
        esum += es[k];
      }
      u64 e, ee;
      const u64 tot = block_excl_scan64(sum, &e, s_w);
      const u64 etot = block_excl_scan64(esum, &ee, s_w2);
      u64 run = carry + e, erun = ecarry + ee;
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const u64 g = g0 + k;
        if (g < n_chunks) {
          p.chunk_hioff[g] = run;
          p.chunk_escoff[g] = erun;
        }
        run += v[k];
        erun += es[k];
      }
      carry += tot;
      ecarry += etot;
    }
    if (threadIdx.x == 0) {
      p.chunk_hioff[n_chunks] = carry;
      p.chunk_escoff[n_chunks] = ecarry;
    }
    __syncthreads();
  }
  const u64 rans = block_sum64(rans_local, s_w2);
  // 2. record sizes and offsets; the record table (compacted: tensors with a change, in manifest order) with
  //    the byte and on-wire chunk prefixes the device bucket planner walks (bucket.cu)
  u64 carry_enc = 0, n16 = 0, n32 = 0, ib_tot = 0, vb_tot = 0, nfull = 0, n16e = 0, carry_r = 0, carry_c = 0;
  for (u32 b = 0; b < T; b += (u32)kRound) {
    const u32 t0 = b + threadIdx.x * kPer;
    u64 bytes[kPer], wch[kPer];
    u64 sum = 0, rsum = 0, csum = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const u32 t = t0 + k;
      const u64 c = (t < T && !over) ? counts[t] : 0;
      u64 by = 0, ib = 0;
      u32 mode = 1;
      if (c) {
        if (comp) {
          const u64 ch0 = p.chunk_off[t], ch1 = p.chunk_off[t + 1];
          mode = p.maxgap[t] <= 32767u ? 0u : 1u;
          u64 table = 0;
          if (mode && p.escape) {   // f4: escapes < nnz -> DELTA16E beats ABS32
            const u64 ne = p.chunk_escoff[ch1] - p.chunk_escoff[ch0];
            if (ne < c) {
              mode = kModeDelta16E;
              table = 4 * (ch1 - ch0 + 1);
              ib = pad_to(2 * (c + ne), 4);
            }
          }
          if (mode != kModeDelta16E) ib = pad_to((mode ? 4 : 2) * c, 4);
          const u64 hi = p.chunk_hioff[ch1] - p.chunk_hioff[ch0];
          by = pad_to(16 + table + ib + (e8 ? 0 : pad_to(c, 4)) + 16 * (ch1 - ch0) + hi, 16);   // FP8: no lo plane
        } else {
          ib = 4 * c;
          by = pad_to(16 + (e8 ? 5 : 6) * c, 16);
        }
        const u64 full = pad_to(16 + (e8 ? 1 : 2) * p.numel[t], 16);   // f3 routing (DESIGN C19)
        if (p.route && full < by) {
          mode = kModeFull;
          by = full;
          ib = 0;
          nfull++;
        } else if (mode == kModeDelta16E) {
          n16e++;
        } else if (mode) {
          n32++;
        } else {
          n16++;
        }
        ib_tot += ib;
        vb_tot += by - 16 - ib;
      }
      if (t < T) {
        p.rec_mode[t] = mode;
        p.rec_bytes[t] = by;
      }
      bytes[k] = by;
      // chunks of a record on the wire = ceil(nnz field / C); a FULL record's nnz field is numel
      wch[k] = !by ? 0 : mode == kModeFull ? (p.numel[t] + kChunk - 1) / kChunk : p.chunk_off[t + 1] - p.chunk_off[t];
      sum += by;
      rsum += by ? 1 : 0;
      csum += wch[k];
    }
    u64 e, re, ce;
    const u64 tot = block_excl_scan64(sum, &e, s_w);
    const u64 rtot = block_excl_scan64(rsum, &re, s_w2);
    const u64 ctot = block_excl_scan64(csum, &ce, s_w);
    u64 run = carry_enc + e, rrun = carry_r + re, crun = carry_c + ce;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const u32 t = t0 + k;
      if (t < T) p.enc_off[t] = run;
      if (bytes[k]) {
        p.rec_list[rrun] = t;
        p.srec[rrun] = run;
        p.crec[rrun] = crun;
        rrun++;
      }
      run += bytes[k];
      crun += wch[k];
    }
    carry_enc += tot;
    carry_r += rtot;
    carry_c += ctot;
  }
  if (threadIdx.x == 0) {
    p.srec[carry_r] = carry_enc;
    p.crec[carry_r] = carry_c;
  }
  n16 = block_sum64(n16, s_w);
  n32 = block_sum64(n32, s_w2);
  ib_tot = block_sum64(ib_tot, s_w);
  vb_tot = block_sum64(vb_tot, s_w2);
  nfull = block_sum64(nfull, s_w);
  n16e = block_sum64(n16e, s_w2);
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
    p.totals[kTotFull] = nfull;
    p.totals[kTotDelta16E] = n16e;
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
  static int cap[kMaxDevices] = {};   // persistent: the resident CTAs (the warps claim chunks)
  const int dev = current_device();
  if (!cap[dev]) {
    int n_sm = 148, per = 1;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_chunk_stats, 256, 0);
    cap[dev] = n_sm * (per > 0 ? per : 1);
  }
  k_chunk_stats<<<grid < cap[dev] ? grid : cap[dev], 256, 0, s>>>(q, I, V, counts);
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
