// plan.cu — K2: record plan for the §3.3 encodings (rows a2 + sizing of a3/a4).
//
// From the per-tensor counts of K1:
//  * k_plan_scan   (grid)    value offsets, chunk offsets, totals (manifest order)
//  * k_chunk_stats (grid)    per chunk: max index gap (-> DELTA16/ABS32, P:360,
//                            DESIGN C4), hi-byte histogram, normalised rANS model
//                            and the rANS encode pass -> exact hi block size and
//                            RAW/RANS decision (never-expand); words, states
//                            and model kept in scratch for k_encode
//  * k_plan_chunks (grid)    chunk hi-offset / escape prefixes
//  * k_plan_records (grid)   record sizes and modes, record byte offsets, the compacted
//                            record table for the bucket planner, statistics
// The scans are grid-wide (scan.cuh: one item per thread, CTA totals published with the scan's epoch):
// single-CTA versions took 40 + 117 us of latency per sync on the 30B manifest.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "chunk.cuh"
#include "scan.cuh"

// k_chunk_stats CTAs per SM (dev override -DSS_CS_MINB): 4 at 64 registers; same-box A/B round 2: 3 (78
// registers) +5%, 5 or 6 (spilling) +4% / +30%
#ifndef SS_CS_MINB
#define SS_CS_MINB 4
#endif

namespace ss {

#define G_STATE(p, off) (reinterpret_cast<GScanState*>((p).gscan) + (off))
#define G_OFF_CHUNKS(p) ((p).gscan_T)
#define G_OFF_RECORDS(p) ((p).gscan_T + (p).gscan_C)

// one tensor per thread: (nnz, chunks, record flag) -> rec_off, chunk_off; the last CTA writes the totals
__global__ void __launch_bounds__(kGScan) k_plan_scan(Plan p, const u64* counts) {
  __shared__ u64 s_w[3 * 33];
  __shared__ u32 s_j;
  const u32 T = p.n_tensors;
  const u32 G = T ? (T + kGScan - 1) / kGScan : 1;
  __shared__ u64 s_e;
  const u32 j = gscan_rank(p.tickets + 0, G, &s_j);
  const u64 epoch = gscan_epoch(p.epochs + 0, &s_e);
  const u32 t = j * kGScan + threadIdx.x;
  const u64 c = t < T ? counts[t] : 0;
  const u64 v[3] = {c, (c + kChunk - 1) / kChunk, c ? 1ull : 0ull};
  u64 ex[3], tot[3], pre[3];
  block_scan3(v, ex, tot, s_w);
  gscan_publish_and_prefix(G_STATE(p, 0), j, epoch, tot, pre, s_w);
  if (j + 1 == G) gscan_advance(p.epochs + 0, epoch);
  if (t < T) {
    p.rec_off[t] = pre[0] + ex[0];
    p.chunk_off[t] = pre[1] + ex[1];
    p.maxgap[t] = 0;
  }
  if (j + 1 == G && threadIdx.x == 0) {
    const u64 nnz = pre[0] + tot[0], ch = pre[1] + tot[1], rec = pre[2] + tot[2];
    p.rec_off[T] = nnz;
    p.chunk_off[T] = ch;
    const bool over = nnz > p.cap || ch > p.max_chunks;
    if (over) latch(p.status, SYNC_ERR_CAPACITY);
    for (int k = 0; k < 16; ++k) p.totals[k] = 0;
    p.work[0] = 0;   // chunk counters of k_chunk_stats / k_encode
    p.work[1] = 0;
    p.totals[kTotNnz] = nnz;
    p.totals[kTotChunks] = over ? 0 : ch;
    p.totals[kTotRecords] = rec;
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
#ifndef SS_WPF
#define SS_WPF 8
#endif
constexpr int kWPF = SS_WPF;   // rANS steps per prefetched block of coded bytes (dev override -DSS_WPF)
template <bool kEsc>   // f4: also count the gaps > 32767 per chunk (escape words)
__global__ void __launch_bounds__(256, SS_CS_MINB) k_chunk_stats(Plan p, const u32* I, const u16* V, const u64* counts) {
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
    if (lane == 0) p.chunk_t[g] = t;   // for k_encode
    const u64 nnz = counts[t];
    const u64 p0 = (g - co[t]) * kChunk;
    const u32 nk = (u32)((nnz - p0) < kChunk ? (nnz - p0) : kChunk);
    const u64 gs = p.rec_off[t] + p0, ge = gs + nk;   // the chunk's values in I / V
    const long long t1 = clock64();
    for (u32 sym = lane; sym < 256; sym += 32) m.hist[sym] = 0;
    __syncwarp();
    // I of the element before the chunk (Δ_0 = I_0 when the chunk starts its record)
    u32 carry0 = (lane == 0 && p0) ? I[gs - 1] : 0u;
    carry0 = __shfl_sync(0xffffffffu, carry0, 0);
    u32 carry = carry0;
    u32 gmax = 0, nesc = 0;
    // one round = 256 values (8 per lane); the next round's 16-byte loads are issued before this round is
    // consumed. Groups wholly inside the chunk (all but its first and last) take the unmasked path.
    auto load = [&](u64 e, uint4& va, uint4& ia, uint4& ib) {
      if (e < ge && e + 8 <= p.cap) {   // a whole 8-group inside the I / V arrays
        va = *reinterpret_cast<const uint4*>(V + e);
        ia = *reinterpret_cast<const uint4*>(I + e);
        ib = *reinterpret_cast<const uint4*>(I + e + 4);
      } else {                           // the arrays' tail: element loads (masked below)
        u32 h[8], x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const bool in = e + k < ge;
          x[k] = in ? I[e + k] : 0u;
          h[k] = in ? (u32)V[e + k] : 0u;
        }
        va = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
        ia = make_uint4(x[0], x[1], x[2], x[3]);
        ib = make_uint4(x[4], x[5], x[6], x[7]);
      }
    };
    uint4 nva, nia, nib;
    const u64 eb = gs & ~7ull;
    load(eb + 8ull * lane, nva, nia, nib);
    for (u64 e0 = eb; e0 < ge; e0 += 256) {
      const u64 e = e0 + 8ull * lane;
      const uint4 va = nva, ia = nia, ib = nib;
      if (e0 + 256 < ge) load(e + 256, nva, nia, nib);
      const u32 vw[4] = {va.x, va.y, va.z, va.w};
      u32 hv[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        hv[2 * k] = (vw[k] >> sh) & 0xFFu;
        hv[2 * k + 1] = (vw[k] >> (16 + sh)) & 0xFFu;
      }
      const u32 iv[8] = {ia.x, ia.y, ia.z, ia.w, ib.x, ib.y, ib.z, ib.w};
      u32 prev = __shfl_up_sync(0xffffffffu, iv[7], 1);
      if (lane == 0) prev = carry;
      carry = __shfl_sync(0xffffffffu, iv[7], 31);
      if (e >= gs && e + 8 <= ge) {
        // whole group inside the chunk; if it starts the chunk it is lane 0's of the first round, whose
        // prev is carry0
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          atomicAdd(&m.hist[hv[k]], 1u);
          const u32 d = iv[k] - (k ? iv[k - 1] : prev);
          gmax = d > gmax ? d : gmax;
          if (kEsc) nesc += d > 32767u ? 1u : 0u;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const u64 q = e + k;
          if (q >= gs && q < ge) {
            atomicAdd(&m.hist[hv[k]], 1u);
            const u32 d = iv[k] - (q == gs ? carry0 : (k ? iv[k - 1] : prev));
            gmax = d > gmax ? d : gmax;
            if (kEsc) nesc += d > 32767u ? 1u : 0u;
          }
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
    if (kEsc && lane == 0) p.chunk_esc[g] = nesc;   // f4: gaps that need an escape word
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
    const u8* Vb = reinterpret_cast<const u8*>(V + gs) + (sh ? 1 : 0);   // byte 2q + vb: the coded byte of V[q]
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

// one chunk per thread: exclusive prefixes of the padded hi block sizes and of the escape counts; RANS chunks
__global__ void __launch_bounds__(kGScan) k_plan_chunks(Plan p, u32 G) {
  __shared__ u64 s_w[3 * 33];
  __shared__ u32 s_j;
  __shared__ u64 s_e;
  const u32 j = gscan_rank(p.tickets + 1, G, &s_j);
  const u64 epoch = gscan_epoch(p.epochs + 1, &s_e);
  const u64 n_chunks = p.totals[kTotChunks];
  const u64 g = (u64)j * kGScan + threadIdx.x;
  const bool in = g < n_chunks;
  const u64 v[3] = {in ? pad_to(p.chunk_hi[g], 4) : 0, (in && p.escape) ? p.chunk_esc[g] : 0,
                    in ? p.chunk_mode[g] : 0};
  u64 ex[3], tot[3], pre[3];
  block_scan3(v, ex, tot, s_w);
  gscan_publish_and_prefix(G_STATE(p, G_OFF_CHUNKS(p)), j, epoch, tot, pre, s_w);
  if (j + 1 == G) gscan_advance(p.epochs + 1, epoch);
  if (in) {
    p.chunk_hioff[g] = pre[0] + ex[0];
    p.chunk_escoff[g] = pre[1] + ex[1];
  }
  if (j + 1 == G && threadIdx.x == 0) {
    p.chunk_hioff[n_chunks] = pre[0] + tot[0];
    p.chunk_escoff[n_chunks] = pre[1] + tot[1];
    p.totals[kTotRansChunks] = pre[2] + tot[2];
  }
}

// one tensor per thread: record mode and size (C4, C19, §3.6), the byte offset of each record
// in the contiguous stream (enc_off), and the record table (compacted: tensors with a change, manifest order)
// with its byte and on-wire chunk prefixes for the bucket planner (bucket.cu); statistics by atomics
__global__ void __launch_bounds__(kGScan) k_plan_records(Plan p, const u64* counts) {
  __shared__ u64 s_w[3 * 33];
  __shared__ u64 s_st[6];
  __shared__ u32 s_j;
  const u32 T = p.n_tensors;
  const u32 G = T ? (T + kGScan - 1) / kGScan : 1;
  const bool comp = p.codec == SYNC_CODEC_COMPRESSED;
  const bool e8 = p.dtype == SYNC_DTYPE_FP8;
  const bool over = p.totals[kTotOverflow] != 0;
  __shared__ u64 s_e;
  const u32 j = gscan_rank(p.tickets + 2, G, &s_j);
  const u64 epoch = gscan_epoch(p.epochs + 2, &s_e);
  if (threadIdx.x < 6) s_st[threadIdx.x] = 0;
  const u32 t = j * kGScan + threadIdx.x;
  const u64 c = (t < T && !over) ? counts[t] : 0;
  u64 by = 0, ib = 0, wch = 0;
  u32 mode = 1;
  if (c) {
    const u64 ch0 = p.chunk_off[t], ch1 = p.chunk_off[t + 1];
    const u64 numel = p.numel[t];
    if (comp) {
      const u32 mg = p.maxgap[t];
      const u64 hi = p.chunk_hioff[ch1] - p.chunk_hioff[ch0];
      mode = mg <= 32767u ? 0u : 1u;
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
      by = pad_to(16 + table + ib + (e8 ? 0 : pad_to(c, 4)) + 16 * (ch1 - ch0) + hi, 16);   // FP8: no lo plane
    } else {
      ib = 4 * c;
      by = pad_to(16 + (e8 ? 5 : 6) * c, 16);
    }
    const u64 full = pad_to(16 + (e8 ? 1 : 2) * numel, 16);   // f3 routing (DESIGN C19)
    if (p.route && full < by) {
      mode = kModeFull;
      by = full;
      ib = 0;
    }
    // chunks of a record on the wire = ceil(nnz field / C); a FULL record's nnz field is numel
    wch = mode == kModeFull ? (numel + kChunk - 1) / kChunk : ch1 - ch0;
  }
  if (t < T) {
    p.rec_mode[t] = mode;
    p.rec_bytes[t] = by;
  }
  __syncthreads();   // s_st zeroed
  {                  // statistics: record kinds, index / value bytes (warp sums, then one shared atomic per warp)
    const int kind = !by ? -1 : mode == kModeFull ? 3 : mode == kModeDelta16E ? 2 : mode ? 1 : 0;
    u64 st[6] = {kind == 0, kind == 1, kind == 2, kind == 3, by ? ib : 0, by ? by - 16 - ib : 0};
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      st[k] = warp_sum64(st[k]);
      if ((threadIdx.x & 31) == 0 && st[k]) atomicAdd(reinterpret_cast<unsigned long long*>(&s_st[k]), st[k]);
    }
  }
  const u64 v[3] = {by, by ? 1ull : 0ull, wch};
  u64 ex[3], tot[3], pre[3];
  block_scan3(v, ex, tot, s_w);
  gscan_publish_and_prefix(G_STATE(p, G_OFF_RECORDS(p)), j, epoch, tot, pre, s_w);
  if (j + 1 == G) gscan_advance(p.epochs + 2, epoch);
  const u64 off = pre[0] + ex[0];
  if (t < T) p.enc_off[t] = off;
  if (by) {
    const u64 r = pre[1] + ex[1];
    p.rec_list[r] = t;
    p.srec[r] = off;
    p.crec[r] = pre[2] + ex[2];
  }
  if (threadIdx.x == 0) {
    // codec RAW: every record counts as ABS32 (u32 indices)
    const u64 n16 = s_st[0], n32 = s_st[1], n16e = s_st[2], nfull = s_st[3];
    if (n16 && comp) atomicAdd(reinterpret_cast<unsigned long long*>(&p.totals[kTotDelta16]), n16);
    if (n32 + (comp ? 0 : n16)) atomicAdd(reinterpret_cast<unsigned long long*>(&p.totals[kTotAbs32]), n32 + (comp ? 0 : n16));
    if (n16e) atomicAdd(reinterpret_cast<unsigned long long*>(&p.totals[kTotDelta16E]), n16e);
    if (nfull) atomicAdd(reinterpret_cast<unsigned long long*>(&p.totals[kTotFull]), nfull);
    if (s_st[4]) atomicAdd(reinterpret_cast<unsigned long long*>(&p.totals[kTotIndexBytes]), (unsigned long long)s_st[4]);
    if (s_st[5]) atomicAdd(reinterpret_cast<unsigned long long*>(&p.totals[kTotValueBytes]), (unsigned long long)s_st[5]);
    if (j + 1 == G) {
      const u64 enc = pre[0] + tot[0], R = pre[1] + tot[1];
      p.enc_off[T] = enc;
      p.srec[R] = enc;
      p.crec[R] = pre[2] + tot[2];
      p.totals[kTotEnc] = enc;
      if (enc > p.enc_cap) {
        latch(p.status, SYNC_ERR_CAPACITY);
        p.totals[kTotOverflow] = 1;
        p.totals[kTotChunks] = 0;   // nothing gets encoded
      }
    }
  }
}

void launch_plan_scan(const Plan& p, const u64* counts, cudaStream_t s) {
  const u32 T = p.n_tensors ? p.n_tensors : 1;
  k_plan_scan<<<(T + kGScan - 1) / kGScan, kGScan, 0, s>>>(p, counts);
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
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_chunk_stats<false>, 256, 0);
    cap[dev] = n_sm * (per > 0 ? per : 1);
  }
  const int g = grid < cap[dev] ? grid : cap[dev];
  if (p.escape) k_chunk_stats<true><<<g, 256, 0, s>>>(q, I, V, counts);
  else k_chunk_stats<false><<<g, 256, 0, s>>>(q, I, V, counts);
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
  if (p.codec == SYNC_CODEC_COMPRESSED) {
    k_plan_chunks<<<p.gscan_C, kGScan, 0, s>>>(p, p.gscan_C);
    count_launch();
  }
  const u32 T = p.n_tensors ? p.n_tensors : 1;
  k_plan_records<<<(T + kGScan - 1) / kGScan, kGScan, 0, s>>>(p, counts);
  count_launch();
}

}  // namespace ss
