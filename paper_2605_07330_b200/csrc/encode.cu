// encode.cu — K3: record encoding (rows a3 + a4), DESIGN §3.1 / §3.2.
//
// One CTA per chunk (16384 values). COMPRESSED: the chunk's slice of the
// index stream (DELTA16 first differences with a prepended zero, or ABS32
// absolutes), its slice of the raw lo plane, its directory entry and
// its hi block — a static order-0 rANS over 32 interleaved lanes (lane j owns
// positions p = 32g + j, so a warp step encodes 32 symbols and the serial word
// order of DESIGN §3.3 is recovered with one ballot per step). RAW: u32 I and
// u16 V slices (the paper's measured raw path). Chunk 0 of a
// record writes the header; the last chunk writes the section paddings.
#include "common.cuh"
#include "kernels.h"
#include "chunk.cuh"

// k_encode is bound by load latency (ncu: long-scoreboard stalls, DRAM at ~55% of peak with 24 warps per SM):
// the vectorised rounds below with 2 rounds in flight per thread at 8 CTAs (32 warps) per SM beat 4 rounds at
// 6 CTAs by 5% (rho = 1%) / 4-7% (rho = 10%) and the one-value-per-thread loop alone by 5% / 7% (same-box A/B,
// round 2; 10 or 12 CTAs spill). Dev overrides for A/B builds: -DSS_ENC_KV, -DSS_ENC_MINB.
#ifndef SS_ENC_KV
#define SS_ENC_KV 2
#endif
#ifndef SS_ENC_MINB
#define SS_ENC_MINB 8
#endif

namespace ss {

__device__ __forceinline__ void zero_bytes(u8* p, u64 n) {
  for (u64 q = threadIdx.x; q < n; q += blockDim.x) p[q] = 0;
}

// Vectorised index stream + lo plane (compressed codec, DELTA16 / ABS32): lane l of warp w owns the 4 values
// q = 512 r + 128 w + 4 l .. + 3 of round r — one 16-byte load of I and one 8-byte load of V per 4 values (twice
// the bytes in flight per register of the one-value-per-thread loop), one 8-byte DELTA16 / 16-byte ABS32 store
// and one 4-byte lo store. The chunk's first value sits at global position cs, D = cs mod 4 (uniform): lanes load
// the aligned quads at cs - D + ... and shift by D with the next lane's quad (a shuffle; lane 31 loads the quad
// after its own). Processes the whole rounds (512 values) of [0, nk); returns how many values it did.
template <int D>
__device__ __forceinline__ u32 encode_vec(const u32* I, const u16* V, u64 cs, u32 nk, u64 cap, bool first_rec,
                                          u32 mode, bool e8, u16* D16, u32* A32, u8* L) {
  constexpr int kV = SS_ENC_KV;   // rounds in flight per thread
  const u32 tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  u32 nr = nk / 512;
  while (nr && cs + (u64)nr * 512 + 4 > cap) --nr;   // keep every quad load inside the arrays
  const u64 ab = cs - D;                              // 4-aligned
  for (u32 r0 = 0; r0 < nr; r0 += kV) {
    uint4 qi[kV], ni[kV];
    uint2 qv[kV], nv[kV];
    u32 pred[kV];
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const u32 qb = (r0 + u) * 512 + 128 * warp;     // the warp's first value of this round
      qi[u] = make_uint4(0, 0, 0, 0);
      qv[u] = make_uint2(0, 0);
      ni[u] = make_uint4(0, 0, 0, 0);
      nv[u] = make_uint2(0, 0);
      pred[u] = 0;
      if (r0 + u < nr) {
        const u64 a = ab + qb + 4 * lane;
        qi[u] = *reinterpret_cast<const uint4*>(I + a);
        qv[u] = *reinterpret_cast<const uint2*>(V + a);
        if (D && lane == 31) {
          ni[u] = *reinterpret_cast<const uint4*>(I + a + 4);
          nv[u] = *reinterpret_cast<const uint2*>(V + a + 4);
        }
        if (lane == 0 && (mode == 0) && !(first_rec && qb == 0)) pred[u] = I[cs + qb - 1];
      }
    }
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      if (r0 + u >= nr) break;
      const u32 q = (r0 + u) * 512 + 128 * warp + 4 * lane;
      u32 wi[8] = {qi[u].x, qi[u].y, qi[u].z, qi[u].w, 0, 0, 0, 0};
      u32 wv[4] = {qv[u].x, qv[u].y, 0, 0};
      if (D) {
        const uint4 n4 = make_uint4(__shfl_down_sync(0xffffffffu, qi[u].x, 1), __shfl_down_sync(0xffffffffu, qi[u].y, 1),
                                    __shfl_down_sync(0xffffffffu, qi[u].z, 1), __shfl_down_sync(0xffffffffu, qi[u].w, 1));
        const uint2 n2 = make_uint2(__shfl_down_sync(0xffffffffu, qv[u].x, 1), __shfl_down_sync(0xffffffffu, qv[u].y, 1));
        const bool l31 = lane == 31;
        wi[4] = l31 ? ni[u].x : n4.x;
        wi[5] = l31 ? ni[u].y : n4.y;
        wi[6] = l31 ? ni[u].z : n4.z;
        wi[7] = l31 ? ni[u].w : n4.w;
        wv[2] = l31 ? nv[u].x : n2.x;
        wv[3] = l31 ? nv[u].y : n2.y;
      }
      const u32 i0 = wi[D], i1 = wi[D + 1], i2 = wi[D + 2], i3 = wi[D + 3];
      // 16-bit values D .. D+3 of the 8-element window wv (element j = half j & 1 of word j >> 1)
      const u32 e0 = wv[D >> 1] >> (16 * (D & 1)), e1 = wv[(D + 1) >> 1] >> (16 * ((D + 1) & 1));
      const u32 e2 = wv[(D + 2) >> 1] >> (16 * ((D + 2) & 1)), e3 = wv[(D + 3) >> 1] >> (16 * ((D + 3) & 1));
      if (mode == 0) {
        u32 prev = __shfl_up_sync(0xffffffffu, i3, 1);
        if (lane == 0) prev = pred[u];
        *reinterpret_cast<uint2*>(D16 + q) = make_uint2(__byte_perm(i0 - prev, i1 - i0, 0x5410),
                                                        __byte_perm(i2 - i1, i3 - i2, 0x5410));
      } else {
        *reinterpret_cast<uint4*>(A32 + q) = make_uint4(i0, i1, i2, i3);
      }
      if (!e8)
        *reinterpret_cast<u32*>(L + q) = (e0 & 0xFFu) | ((e1 & 0xFFu) << 8) | ((e2 & 0xFFu) << 16) | ((e3 & 0xFFu) << 24);
    }
  }
  return nr * 512;
}

// One CTA per chunk (16384 values; persistent CTAs claim chunks from a counter). All threads write the chunk's slices of the
// index stream and of the lo plane (packed 32-bit stores) and copy the chunk's
// rANS block (states, model, words) that k_chunk_stats already produced.
__global__ void __launch_bounds__(kCThreads, SS_ENC_MINB) k_encode(Plan p, const u32* I, const u16* V, const u64* counts,
                                                     u8* enc) {
  __shared__ u32 s_t;
  __shared__ u64 s_g[2];
  const u32 tid = threadIdx.x;
  const u64 n_chunks = p.totals[kTotChunks];
  const bool comp = p.codec == SYNC_CODEC_COMPRESSED;
  const bool e8 = p.dtype == SYNC_DTYPE_FP8;   // FP8: one value plane (the byte), no lo plane
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(p.work + 1);
  if (tid == 0) s_g[0] = atomicAdd(ctr, 1ull);
  for (u32 it = 0;; ++it) {
    __syncthreads();
    const u64 g = s_g[it & 1];
    if (g >= n_chunks) break;
    if (tid == 0) s_g[(it + 1) & 1] = atomicAdd(ctr, 1ull);   // claim the next chunk now: its latency hides
                                                                // behind this chunk's work
    // the compressed codec's stats pass recorded each chunk's tensor (no search)
    const ChunkPos c = comp ? chunk_at(p, counts, g, p.chunk_t[g], I, V) : locate_chunk(p, counts, g, s_t, I, V);
    const u32 t = c.t;
    const u64 nnz = c.nnz, k = c.k, p0 = c.p0;
    const u32 nk = c.nk;
    const u64 n_ch = p.chunk_off[t + 1] - p.chunk_off[t];
    const bool last = (k + 1 == n_ch);
    const u32* Ir = c.Ir;
    const u16* Vc = c.Vc;
    u8* rec = enc + p.rec_dst[t];
    const u64 rb = p.rec_bytes[t];
    const u32 mode = p.rec_mode[t];

    if (k == 0 && tid == 0) {
      u32* h = reinterpret_cast<u32*>(rec);
      h[0] = t;
      h[1] = mode == kModeFull ? (u32)p.numel[t] : (u32)nnz;
      h[2] = (u32)rb;
      h[3] = mode | (p.dtype << 8) | ((comp ? 1u : 0u) << 16);
    }

    if (mode == kModeFull) {
      // f3 FULL record: the tensor's current values. The record's n_ch chunks (counted
      // from its nnz) split the copy at multiples of 8 elements (16-byte stores into the 16-aligned body).
      const u64 numel = p.numel[t];
      const u64 lo = (numel * k / n_ch) & ~15ull;
      const u64 hi = last ? numel : ((numel * (k + 1) / n_ch) & ~15ull);
      if (e8) {   // bytes
        const u8* src8 = reinterpret_cast<const u8*>(p.cur[t]);
        u8* dst8 = rec + 16;
        for (u64 q = lo + tid; q < hi; q += kCThreads) dst8[q] = src8[q];
        if (last) zero_bytes(rec + 16 + numel, rb - (16 + numel));
        continue;
      }
      const u16* src = p.cur[t];
      u16* dst = reinterpret_cast<u16*>(rec + 16);
      if ((((uintptr_t)src) & 15u) == 0) {
        const u64 v_end = lo + ((hi - lo) & ~7ull);
        for (u64 q = lo + 8ull * tid; q < v_end; q += 8ull * kCThreads)
          *reinterpret_cast<uint4*>(dst + q) = *reinterpret_cast<const uint4*>(src + q);
        for (u64 q = v_end + tid; q < hi; q += kCThreads) dst[q] = src[q];
      } else {
        for (u64 q = lo + tid; q < hi; q += kCThreads) dst[q] = src[q];
      }
      if (last) zero_bytes(rec + 16 + 2 * numel, rb - (16 + 2 * numel));
      continue;
    }

    if (!comp) {
      u32* Io = reinterpret_cast<u32*>(rec + 16) + p0;
      u8* Vb = rec + 16 + 4 * nnz;
      constexpr int kR = 8;   // coalesced, 8 values per thread in flight (one at a time was latency-bound)
      for (u32 q0 = 0; q0 < nk; q0 += kCThreads * kR) {
        u32 iv[kR], vv[kR];
#pragma unroll
        for (int u = 0; u < kR; ++u) {
          const u32 q = q0 + u * kCThreads + tid;
          iv[u] = q < nk ? Ir[p0 + q] : 0u;
          vv[u] = q < nk ? (u32)Vc[q] : 0u;
        }
#pragma unroll
        for (int u = 0; u < kR; ++u) {
          const u32 q = q0 + u * kCThreads + tid;
          if (q < nk) {
            Io[q] = iv[u];
            if (e8) Vb[p0 + q] = (u8)vv[u];
            else reinterpret_cast<u16*>(Vb)[p0 + q] = (u16)vv[u];
          }
        }
      }
      const u64 used = 16 + (e8 ? 5 : 6) * nnz;
      if (last) zero_bytes(rec + used, rb - used);
      continue;
    }

    // ---- index stream + lo plane slices: groups of 4 positions per thread, kG groups in flight
    //      (DELTA16: one 64-bit store of 4 deltas; ABS32: one 128-bit store; lo: one 32-bit store)
    const bool esc = mode == kModeDelta16E;
    const u64 ch0 = p.chunk_off[t];
    const u64 ne_rec = esc ? p.chunk_escoff[ch0 + n_ch] - p.chunk_escoff[ch0] : 0;
    const u64 s0 = esc ? 16 + 4 * (n_ch + 1) : 16;          // f4: word-offset table after the header
    const u64 ib = esc ? 2 * (nnz + ne_rec) : (mode ? 4 : 2) * nnz;
    const u64 lo_off = s0 + pad_to(ib, 4);
    const u64 dir_off = lo_off + (e8 ? 0 : pad_to(nnz, 4));
    const u64 hi_base = dir_off + 16 * n_ch;
    if (esc) {
      // f4 DELTA16E: rounds of 4 positions per thread; a block scan of the word counts (1, or
      // 2 for an escape) places every thread's words after the chunk's first word w0
      __shared__ u32 s_ws[kCThreads / 32 + 1];
      const u64 w0 = (u64)p0 + (p.chunk_escoff[g] - p.chunk_escoff[ch0]);
      u32* tbl = reinterpret_cast<u32*>(rec + 16);
      if (tid == 0) {
        tbl[k] = (u32)w0;
        if (last) tbl[n_ch] = (u32)(nnz + ne_rec);
      }
      u16* Ws = reinterpret_cast<u16*>(rec + s0);
      u8* L = rec + lo_off + p0;
      u64 wrun = w0;
      for (u32 r0 = 0; r0 < nk; r0 += 4 * kCThreads) {
        const u32 q = r0 + 4 * tid;
        u32 d[4];
        u32 cnt = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const u64 pp = p0 + q + j;
          d[j] = 0;
          if (q + j < nk) {
            d[j] = Ir[pp] - (pp ? Ir[pp - 1] : 0u);
            cnt += d[j] > 32767u ? 2u : 1u;
            if (!e8) L[q + j] = (u8)(Vc[q + j] & 0xFFu);
          }
        }
        // exclusive block scan of cnt (kCThreads threads)
        const u32 lane = tid & 31, wp = tid >> 5;
        const u32 inc = warp_incl_scan(cnt);
        if (lane == 31) s_ws[wp] = inc;
        __syncthreads();
        if (tid == 0) {
          u32 acc = 0;
          for (u32 i = 0; i < kCThreads / 32; ++i) {
            const u32 v = s_ws[i];
            s_ws[i] = acc;
            acc += v;
          }
          s_ws[kCThreads / 32] = acc;
        }
        __syncthreads();
        u64 w = wrun + s_ws[wp] + inc - cnt;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (q + j < nk) {
            if (d[j] <= 32767u) {
              Ws[w++] = (u16)d[j];
            } else {
              Ws[w++] = (u16)(0x8000u | (d[j] >> 16));
              Ws[w++] = (u16)(d[j] & 0xFFFFu);
            }
          }
        }
        wrun += s_ws[kCThreads / 32];
        __syncthreads();
      }
    } else {
      // thread tid owns positions q = q0 + u * kCThreads + tid (u < kU): every load / store instruction of a
      // warp covers 32 consecutive values (coalesced), kU values per thread in flight; Δ from the value of
      // lane l - 1 (a shuffle), lane 0 loads its predecessor (Δ_0 = I_0 at a record's first value)
      constexpr int kU = 8;   // the remainder after the vectorised rounds (and unaligned I / V): one value per thread
      const u32 lane = tid & 31;
      const u32* Ic = Ir + p0;
      u16* D16 = reinterpret_cast<u16*>(rec + 16) + p0;
      u32* A32 = reinterpret_cast<u32*>(rec + 16) + p0;
      u8* L = rec + lo_off + p0;
      const u32 first_prev = p0 ? Ic[-1] : 0u;
      u32 qv = 0;   // values done by the vectorised rounds
      const u64 cs = (u64)(Ic - I);
      if (kCThreads == 128 && !(((uintptr_t)I) & 15u) && !(((uintptr_t)V) & 7u) && (u64)(Vc - V) == cs) {
        switch ((u32)(cs & 3u)) {
          case 0: qv = encode_vec<0>(I, V, cs, nk, p.cap, p0 == 0, mode, e8, D16, A32, L); break;
          case 1: qv = encode_vec<1>(I, V, cs, nk, p.cap, p0 == 0, mode, e8, D16, A32, L); break;
          case 2: qv = encode_vec<2>(I, V, cs, nk, p.cap, p0 == 0, mode, e8, D16, A32, L); break;
          default: qv = encode_vec<3>(I, V, cs, nk, p.cap, p0 == 0, mode, e8, D16, A32, L); break;
        }
      }
      for (u32 q0 = qv; q0 < nk; q0 += kCThreads * kU) {
        u32 iv[kU], pv[kU], vv[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const u32 q = q0 + u * kCThreads + tid;
          const bool in = q < nk;
          iv[u] = in ? Ic[q] : 0u;
          vv[u] = in ? (u32)Vc[q] : 0u;
          pv[u] = (lane == 0 && in && mode == 0) ? (q ? Ic[q - 1] : first_prev) : 0u;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const u32 q = q0 + u * kCThreads + tid;
          u32 prev = __shfl_up_sync(0xffffffffu, iv[u], 1);
          if (lane == 0) prev = pv[u];
          if (q < nk) {
            if (mode == 0) D16[q] = (u16)(iv[u] - prev);
            else A32[q] = iv[u];
            if (!e8) L[q] = (u8)(vv[u] & 0xFFu);
          }
        }
      }
    }
    if (last) {
      zero_bytes(rec + s0 + ib, pad_to(ib, 4) - ib);
      if (!e8) zero_bytes(rec + lo_off + nnz, pad_to(nnz, 4) - nnz);
    }
    // ---- directory entry + hi block
    const u32 hb = p.chunk_hi[g];
    const u32 cm = p.chunk_mode[g];
    const u64 hi_off = hi_base + (p.chunk_hioff[g] - p.chunk_hioff[p.chunk_off[t]]);
    if (tid == 0) {
      u32* d = reinterpret_cast<u32*>(rec + dir_off + 16 * k);
      d[0] = (u32)hi_off;
      d[1] = hb;
      d[2] = cm;
      d[3] = ((mode == 0 || mode == kModeDelta16E) && k > 0) ? Ir[p0 - 1] : 0u;
    }
    u8* blk = rec + hi_off;
    if (last) {
      const u64 hi_end = hi_base + (p.chunk_hioff[p.chunk_off[t + 1]] - p.chunk_hioff[p.chunk_off[t]]);
      zero_bytes(rec + hi_end, rb - hi_end);
    }
    if (cm == 0) {
      for (u32 q = tid; q < nk; q += kCThreads) blk[q] = e8 ? (u8)Vc[q] : (u8)(Vc[q] >> 8);
      zero_bytes(blk + nk, pad_to(nk, 4) - nk);
      continue;
    }
    // RANS block: states, model and words were produced by k_chunk_stats; copy them in
    // (words stored in reverse emission order)
    const u32* rh = p.chunk_rhdr + g * kRhdrWords;
    const u32 nsym = rh[33];
    const u32 nwords = rh[32];
    u32* hdr = reinterpret_cast<u32*>(blk);
    for (u32 i = tid; i < 34 + nsym; i += kCThreads) hdr[i] = rh[i];
    const u16* ws = p.word_scratch + chunk_words_base(p.rec_off[t] + p0, g);
    u16* words = reinterpret_cast<u16*>(blk + 136 + 4 * nsym);
    {
      constexpr int kW = 8;   // 8 loads in flight per thread (the copy is latency-bound otherwise)
      for (u32 i0 = tid; i0 < nwords; i0 += kCThreads * kW) {
        u16 w[kW];
#pragma unroll
        for (int j = 0; j < kW; ++j) {
          const u32 i = i0 + j * kCThreads;
          w[j] = i < nwords ? ws[nwords - 1 - i] : (u16)0;
        }
#pragma unroll
        for (int j = 0; j < kW; ++j) {
          const u32 i = i0 + j * kCThreads;
          if (i < nwords) words[i] = w[j];
        }
      }
    }
    if (tid == 0 && (hb & 3u)) *reinterpret_cast<u16*>(blk + hb) = 0;
  }
}

void launch_encode(const Plan& p, const u32* I, const u16* V, const u64* counts, u8* enc, int grid,
                   cudaStream_t s) {
  static int cap[kMaxDevices] = {};   // persistent: the resident CTAs claim chunks from a counter
  const int dev = current_device();
  if (!cap[dev]) {
    int n_sm = 148, per = 1;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_encode, kCThreads, 0);
    cap[dev] = n_sm * (per > 0 ? per : 1);
  }
  k_encode<<<grid < cap[dev] ? grid : cap[dev], kCThreads, 0, s>>>(p, I, V, counts, enc);
  count_launch();
}

}  // namespace ss
