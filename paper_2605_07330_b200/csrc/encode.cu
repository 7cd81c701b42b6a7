// encode.cu — K3: record encoding (rows a3 + a4), DESIGN §3.1 / §3.2.
//
// One warp per chunk (16384 values). COMPRESSED: the chunk's slice of the
// index stream (DELTA16 first differences with a prepended zero, or ABS32
// absolutes), its slice of the raw lo plane, its directory entry and
// its hi block — a static order-0 rANS over 32 interleaved lanes (lane j owns
// positions p = 32g + j, so a warp step encodes 32 symbols and the serial word
// order of DESIGN §3.3 is recovered with one ballot per step). RAW: u32 I and
// u16 V slices (the paper's measured raw path). Chunk 0 of a
// record writes the header; the last chunk writes the section paddings.
#include "common.cuh"
#include "kernels.h"

namespace ss {

__device__ __forceinline__ void zero_bytes(u8* p, u64 n, u32 lane) {
  for (u64 q = lane; q < n; q += 32) p[q] = 0;
}

__global__ void __launch_bounds__(256) k_encode(Plan p, const u32* I, const u16* V, const u64* counts, u8* enc) {
  __shared__ WarpModel s_model[8];
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpModel& m = s_model[warp];
  const u64 n_chunks = p.totals[kTotChunks];
  const u64 nwarps = (u64)gridDim.x * (blockDim.x >> 5);
  const u64* co = p.chunk_off;
  const bool comp = p.codec == SYNC_CODEC_COMPRESSED;
  for (u64 g = (u64)blockIdx.x * (blockDim.x >> 5) + warp; g < n_chunks; g += nwarps) {
    const u32 t = warp_upper_search(p.n_tensors, g, [&](u32 i) { return co[i]; });
    const u64 nnz = counts[t];
    const u64 n_ch = co[t + 1] - co[t];
    const u64 k = g - co[t];
    const u64 p0 = k * kChunk;
    const u32 nk = (u32)((nnz - p0) < kChunk ? (nnz - p0) : kChunk);
    const bool last = (k + 1 == n_ch);
    const u32* Ir = I + p.rec_off[t];
    const u16* Vr = V + p.rec_off[t];
    u8* rec = enc + p.enc_off[t];
    const u64 rb = p.rec_bytes[t];
    const u32 mode = p.rec_mode[t];

    if (k == 0 && lane == 0) {
      u32* h = reinterpret_cast<u32*>(rec);
      h[0] = t;
      h[1] = (u32)nnz;
      h[2] = (u32)rb;
      h[3] = mode | (1u << 8) | ((comp ? 1u : 0u) << 16);
    }

    if (!comp) {
      u32* Io = reinterpret_cast<u32*>(rec + 16);
      u16* Vo = reinterpret_cast<u16*>(rec + 16 + 4 * nnz);
      for (u32 q = lane; q < nk; q += 32) {
        Io[p0 + q] = Ir[p0 + q];
        Vo[p0 + q] = Vr[p0 + q];
      }
      if (last) zero_bytes(rec + 16 + 6 * nnz, rb - (16 + 6 * nnz), lane);
      continue;
    }

    // index stream slice
    const u64 ib = (mode ? 4 : 2) * nnz;
    if (mode == 0) {
      u16* D = reinterpret_cast<u16*>(rec + 16);
      for (u32 q = lane; q < nk; q += 32) {
        u64 pp = p0 + q;
        u32 prev = pp ? Ir[pp - 1] : 0u;
        D[pp] = (u16)(Ir[pp] - prev);
      }
    } else {
      u32* A = reinterpret_cast<u32*>(rec + 16);
      for (u32 q = lane; q < nk; q += 32) A[p0 + q] = Ir[p0 + q];
    }
    const u64 lo_off = 16 + pad_to(ib, 4);
    const u64 dir_off = lo_off + pad_to(nnz, 4);
    const u64 hi_base = dir_off + 16 * n_ch;
    if (last) {
      zero_bytes(rec + 16 + ib, pad_to(ib, 4) - ib, lane);
      zero_bytes(rec + lo_off + nnz, pad_to(nnz, 4) - nnz, lane);
    }
    // lo plane slice
    for (u32 q = lane; q < nk; q += 32) rec[lo_off + p0 + q] = (u8)(Vr[p0 + q] & 0xFFu);

    // directory entry + hi block
    const u32 hb = p.chunk_hi[g];
    const u32 cm = p.chunk_mode[g];
    const u64 hi_off = hi_base + (p.chunk_hioff[g] - p.chunk_hioff[co[t]]);
    if (lane == 0) {
      u32* d = reinterpret_cast<u32*>(rec + dir_off + 16 * k);
      d[0] = (u32)hi_off;
      d[1] = hb;
      d[2] = cm;
      d[3] = (mode == 0 && k > 0) ? Ir[p0 - 1] : 0u;
    }
    u8* blk = rec + hi_off;
    const u16* Vc = Vr + p0;
    if (cm == 0) {
      for (u32 q = lane; q < nk; q += 32) blk[q] = (u8)(Vc[q] >> 8);
      zero_bytes(blk + nk, pad_to(nk, 4) - nk, lane);
    } else {
      warp_histogram(m, nk, [&](u32 q) { return (u32)(Vc[q] >> 8); });
      const u32 nsym = warp_normalize(m, nk);
      const u32 nwords = (hb - 136u - 4u * nsym) / 2u;
      u16* words = reinterpret_cast<u16*>(blk + 136 + 4 * nsym);
      u32 x = kLow, e = 0;
      const u32 G = (nk + 31) / 32;
      const u32 lt = (1u << lane) - 1u;
      for (int gg = (int)G - 1; gg >= 0; --gg) {
        u32 q = (u32)gg * 32 + lane;
        bool act = q < nk;
        u32 s = act ? (u32)(Vc[q] >> 8) : 0u;
        u32 f = m.freq[s];
        bool emit = act && (x >> 20) >= f;
        u32 em = __ballot_sync(0xffffffffu, emit);
        if (emit) {
          words[nwords - 1u - (e + __popc(em & lt))] = (u16)(x & 0xFFFFu);
          x >>= 16;
        }
        e += __popc(em);
        if (act) {
          u32 r;
          u32 qq = div_by(x, f, m.rcp[s], &r);
          x = qq * kM + r + m.cum[s];
        }
      }
      u32* hdr = reinterpret_cast<u32*>(blk);
      hdr[lane] = x;                                   // final states, lane order
      if (lane == 0) {
        hdr[32] = nwords;
        hdr[33] = nsym;                                // u16 nsym | u16 0
      }
      // symbol entries ascending: lane owns symbols 8*lane .. 8*lane+7
      u32 present = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) present += m.freq[lane * 8 + j] ? 1u : 0u;
      u32 rank = warp_incl_scan(present) - present;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        u32 s = lane * 8 + j;
        u32 f = m.freq[s];
        if (f) hdr[34 + rank++] = s | (f << 16);
      }
      if (lane == 0 && (hb & 3u)) *reinterpret_cast<u16*>(blk + hb) = 0;
    }
    if (last) {
      const u64 hi_end = hi_base + (p.chunk_hioff[co[t + 1]] - p.chunk_hioff[co[t]]);
      zero_bytes(rec + hi_end, rb - hi_end, lane);
    }
  }
}

void launch_encode(const Plan& p, const u32* I, const u16* V, const u64* counts, u8* enc, int grid,
                   cudaStream_t s) {
  k_encode<<<grid, 256, 0, s>>>(p, I, V, counts, enc);
  count_launch();
}

}  // namespace ss
