// decode.cu — K5: bucket unpack, decompression and fused scatter-apply
// (rows a7 + a8; Alg. 3 l.5-6; "exact inverse" and "fused kernel").
//
// One warp per chunk of the bucket (the record directory maps a global chunk
// index to its record with a 32-ary warp search). For a rANS hi block the
// warp builds the slot -> symbol table in shared memory, then decodes 32
// symbols per step (lane j owns positions 32g + j); renormalisation words are
// taken in lane order 31..0 with one ballot, exactly as DESIGN §3.3. The lo
// byte and the DELTA16 delta of each position are plain coalesced loads; the
// index is rebuilt with a warp inclusive scan from the chunk's base_idx, and
// V = hi << 8 | lo is scattered straight into the weights (APPLY) or written
// out as (I, V) (EMIT, the debug path). Every chunk checks the end states
// (all lanes back at 2^16) and that every word was consumed.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

// decode launch variants (CTAs per SM, prefetch depth) for dense / sparse calls; dev overrides for A/B builds.
// Dense (decode-bound): with the general loop, 4 CTAs / 3-deep beat 3 / 4-deep by 13% at rho = 10% (BF16 and
// FP8); with the specialised loop of the common record kind, 3 CTAs / 4-deep (80 registers, no spill) is best
// (4 / 3-deep spills: +3.5%); sparse (scatter-bound): 2 CTAs / 8-deep, more CTAs lose 1-3% (round 2)
#ifndef SS_DEC_FAST
#define SS_DEC_FAST 1
#endif
#ifndef SS_DEC_DMINB
#define SS_DEC_DMINB 3
#endif
#ifndef SS_DEC_DPF
#define SS_DEC_DPF 4
#endif
#ifndef SS_DEC_SMINB
#define SS_DEC_SMINB 1
#endif
#ifndef SS_DEC_SPF
#define SS_DEC_SPF 8
#endif

namespace ss {

struct BucketHdr {
  u32 n_records, n_chunks, flags;
  u64 bytes;
};

constexpr u32 kDecodeBatch = 32;
struct DecodeBatch {            // passed by value (kernel parameter)
  const u8* bk[kDecodeBatch];
  u64 bytes[kDecodeBatch];
  u32 n;
  // table mode (t_hdr != null): the buckets b0 .. b0 + 31 of a device bucket table (a sender's plan: t_hdr[0]
  // buckets at t_base + t_off[b], t_size[b] bytes) instead of the host-filled arrays above
  const u64* t_hdr;
  const u64* t_off;
  const u64* t_size;
  const u8* t_base;
  u32 t_b0;
  u32 t_stride;                  // u64 words between consecutive entries of t_off / t_size
};

__device__ __forceinline__ int read_bucket_header(const u8* bk, u64 avail, BucketHdr* h) {
  if (avail < 32) return SYNC_ERR_TRUNCATED;
  const u32* w = reinterpret_cast<const u32*>(bk);
  if (w[0] != kMagic) return SYNC_ERR_BAD_MAGIC;
  if ((w[1] & 0xFFFFu) != kVersion) return SYNC_ERR_VERSION;
  h->flags = w[1] >> 16;
  h->n_records = w[3];
  h->n_chunks = w[4];
  h->bytes = *reinterpret_cast<const u64*>(bk + 24);
  if (h->bytes > avail || h->bytes < 32 + pad_to(8ull * h->n_records, 16)) return SYNC_ERR_TRUNCATED;
  return SYNC_OK;
}

struct RecHdr {
  u32 tid, nnz, rb, mode, dtype, codec;
};

__device__ __forceinline__ bool read_record(const u8* bk, const BucketHdr& h, u32 ro, u32 n_tensors,
                                            const u64* numel, RecHdr* r, u32 dtype) {
  if ((ro & 15u) || (u64)ro + 16 > h.bytes) return false;
  const u32* w = reinterpret_cast<const u32*>(bk + ro);
  r->tid = w[0];
  r->nnz = w[1];
  r->rb = w[2];
  r->mode = w[3] & 0xFFu;
  r->dtype = (w[3] >> 8) & 0xFFu;
  r->codec = (w[3] >> 16) & 0xFFu;
  if (r->rb < 16 || (r->rb & 15u) || (u64)ro + r->rb > h.bytes) return false;
  if (r->tid >= n_tensors || r->dtype != dtype || r->mode > 3 || r->codec > 1 || r->nnz == 0) return false;
  if (r->mode == kModeDelta16E && r->codec != SYNC_CODEC_COMPRESSED) return false;
  if ((u64)r->nnz > numel[r->tid]) return false;
  const u64 eb = dtype == SYNC_DTYPE_FP8 ? 1 : 2;           // element bytes
  const u64 lo = eb == 1 ? 0 : pad_to(r->nnz, 4);            // lo plane (16-bit elements only)
  if (r->mode == kModeFull) return (u64)r->nnz == numel[r->tid] && 16 + eb * r->nnz <= r->rb;
  if (r->codec == SYNC_CODEC_RAW) return r->mode == 1 && 16 + (4 + eb) * r->nnz <= r->rb;
  const u64 nch = (r->nnz + kChunk - 1) / kChunk;
  if (r->mode == kModeDelta16E) {   // f4: word-offset table + total words after the header
    const u64 s0 = 16 + 4 * (nch + 1);
    if (s0 > r->rb) return false;
    const u64 total = reinterpret_cast<const u32*>(bk + ro + 16)[nch];
    if (total < r->nnz || total > 2ull * r->nnz) return false;
    return s0 + pad_to(2 * total, 4) + lo + 16 * nch <= r->rb;
  }
  const u64 ib = (r->mode ? 4ull : 2ull) * r->nnz;
  return 16 + pad_to(ib, 4) + lo + 16 * nch <= r->rb;
}

// ---------------------------------------------------------------------------- unpack
__global__ void __launch_bounds__(1024) k_unpack(const u8* bk, u64 bytes, u32 n_tensors, const u64* numel,
                                                 sync_record_view* views, u32 max_views, u32* n_out, u32* status,
                                                 u32 dtype) {
  __shared__ u64 s_w[33];
  __shared__ int s_err;
  BucketHdr h;
  int err = read_bucket_header(bk, bytes, &h);
  if (err != SYNC_OK || h.n_records > max_views) {
    if (threadIdx.x == 0) {
      latch(status, err != SYNC_OK ? err : SYNC_ERR_CAPACITY);
      *n_out = 0;
    }
    return;
  }
  if (threadIdx.x == 0) s_err = 0;
  __syncthreads();
  const u32* dir = reinterpret_cast<const u32*>(bk + 32);
  u64 carry = 0;
  u32 chunk_carry = 0;
  for (u32 b = 0; b < h.n_records; b += blockDim.x) {
    u32 q = b + threadIdx.x;
    RecHdr r{};
    u64 nnz = 0;
    if (q < h.n_records) {
      u32 ro = dir[2 * q];
      if (!read_record(bk, h, ro, n_tensors, numel, &r, dtype)) {
        s_err = (ro + 16 <= h.bytes && bk[ro + 13] != dtype) ? 2 : 1;
      } else {
        nnz = r.nnz;
        sync_record_view v;
        v.tensor_id = r.tid;
        v.nnz = r.nnz;
        v.offset = ro;
        v.record_bytes = r.rb;
        v.first_chunk = dir[2 * q + 1];
        v.idx_mode = (u8)r.mode;
        v.dtype = (u8)r.dtype;
        v.codec = (u8)r.codec;
        v.reserved = 0;
        v.out_offset = 0;
        views[q] = v;
      }
    }
    // inclusive/exclusive scan of nnz and chunk counts (block of 1024)
    const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    u64 packed = (nnz << 24) | ((nnz + kChunk - 1) / kChunk);  // chunks per record < 2^24
    u64 inc = warp_incl_scan64(packed);
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      u64 w = lane < (blockDim.x >> 5) ? s_w[lane] : 0;
      u64 wi = warp_incl_scan64(w);
      s_w[lane] = wi - w;
      if (lane == 31) s_w[32] = wi;
    }
    __syncthreads();
    u64 ex = s_w[warp] + inc - packed;
    if (q < h.n_records) {
      views[q].out_offset = carry + (ex >> 24);
      if (views[q].first_chunk != chunk_carry + (u32)(ex & 0xFFFFFFull)) s_err = 1;
    }
    u64 tot = s_w[32];
    carry += tot >> 24;
    chunk_carry += (u32)(tot & 0xFFFFFFull);
    __syncthreads();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_err || chunk_carry != h.n_chunks) {
      latch(status, s_err == 2 ? SYNC_ERR_DTYPE : SYNC_ERR_CORRUPT);
      *n_out = 0;
    } else {
      *n_out = h.n_records;
    }
  }
}

// ---------------------------------------------------------------------------- decode
constexpr int kEscWin = 320;   // f4: index words staged per 8-step block (256 elements + 64 escapes; more: global)
struct DecodeModel {
  u8 slot2sym[kM];
  u16 freq[256];
  u16 cum[256];
  u16 win[kEscWin];            // f4: the block's escape-coded index words
};

// One launch decodes up to kDecodeBatch buckets (the chunks of all of them form one grid-stride range), so
// many small buckets do not each pay a launch that fills a fraction of the GPU.
template <bool kApply, int kMinB, int kPF>
__global__ void __launch_bounds__(256, kMinB) k_decode(DecodeBatch bb, u32 n_tensors, const u64* numel,
                                               u16* const* weights, const sync_record_view* views, u32* I_out,
                                               u16* V_out, u64 out_cap, u32* status, const u32* crc_bad,
                                               u32 dtype) {
  __shared__ DecodeModel s_dm[8];
  __shared__ BucketHdr s_h[kDecodeBatch];
  __shared__ u64 s_pre[kDecodeBatch + 1];
  __shared__ const u8* s_bk[kDecodeBatch];
  __shared__ u32 s_n;
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  DecodeModel& dm = s_dm[warp];
  const bool e8 = dtype == SYNC_DTYPE_FP8;   // FP8: one value plane (the byte), no lo plane, byte stores
  u64 my_bytes = 0;
  if (bb.t_hdr) {             // table mode: this launch's slice of the device bucket table
    const u64 nt = *(volatile const u64*)bb.t_hdr;
    const u32 n = nt > bb.t_b0 ? (u32)(nt - bb.t_b0 < kDecodeBatch ? nt - bb.t_b0 : kDecodeBatch) : 0u;
    if (threadIdx.x == 0) s_n = n;
    if (threadIdx.x < n) {
      s_bk[threadIdx.x] = bb.t_base + bb.t_off[(u64)(bb.t_b0 + threadIdx.x) * bb.t_stride];
      my_bytes = bb.t_size[(u64)(bb.t_b0 + threadIdx.x) * bb.t_stride];
    }
  } else {
    if (threadIdx.x == 0) s_n = bb.n;
    if (threadIdx.x < bb.n) {
      s_bk[threadIdx.x] = bb.bk[threadIdx.x];
      my_bytes = bb.bytes[threadIdx.x];
    }
  }
  __syncthreads();
  const u32 nb = s_n;
  if (threadIdx.x < nb) {   // headers; a bucket with a bad header or failed CRC contributes no chunks
    const u32 i = threadIdx.x;
    BucketHdr h;
    int herr = read_bucket_header(s_bk[i], my_bytes, &h);
    if (herr != SYNC_OK) {
      if (blockIdx.x == 0) latch(status, herr);
      h.n_chunks = 0;
    }
    if (crc_bad && crc_bad[i]) h.n_chunks = 0;
    if (h.n_records == 0) h.n_chunks = 0;
    s_h[i] = h;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 acc = 0;
    for (u32 i = 0; i < nb; ++i) {
      s_pre[i] = acc;
      acc += s_h[i].n_chunks;
    }
    s_pre[nb] = acc;
  }
  __syncthreads();
  const u64 total = s_pre[nb];
  const u64 nwarps = (u64)gridDim.x * (blockDim.x >> 5);
  for (u64 gg = (u64)blockIdx.x * (blockDim.x >> 5) + warp; gg < total; gg += nwarps) {
    // bucket of global chunk gg: the last i with s_pre[i] <= gg (kDecodeBatch <= 32: one ballot)
    const u32 bi = 31 - __clz(__ballot_sync(0xffffffffu, lane < nb && s_pre[lane] <= gg));
    const u8* bk = s_bk[bi];
    const BucketHdr h = s_h[bi];
    const u64 g = gg - s_pre[bi];
    const u32* dir = reinterpret_cast<const u32*>(bk + 32);
    const u32 q = warp_upper_search(h.n_records, g, [&](u32 i) { return (u64)dir[2 * i + 1]; });
    const u32 ro = dir[2 * q];
    RecHdr r;
    const u64 fc = dir[2 * q + 1];
    bool ok = read_record(bk, h, ro, n_tensors, numel, &r, dtype);
    const u64 nch = ok ? (r.nnz + kChunk - 1) / kChunk : 0;
    const u64 k = g - fc;
    if (!ok || k >= nch) {
      const bool tag = (u64)ro + 16 <= h.bytes && bk[ro + 13] != dtype;   // another element type
      if (lane == 0) latch(status, tag ? SYNC_ERR_DTYPE : SYNC_ERR_CORRUPT);
      continue;
    }
    const u8* rec = bk + ro;
    const u64 nnz = r.nnz;
    const u64 p0 = k * kChunk;
    const u32 nk = (u32)((nnz - p0) < kChunk ? (nnz - p0) : kChunk);
    const u64 lim = numel[r.tid];
    u16* W = nullptr;
    u32* Io = nullptr;
    u16* Vo = nullptr;
    if (kApply) {
      W = weights[r.tid];
    } else {
      const u64 oo = views[q].out_offset + p0;
      if (oo + nk > out_cap) {
        if (lane == 0) latch(status, SYNC_ERR_CAPACITY);
        continue;
      }
      Io = I_out + oo;
      Vo = V_out + oo;
    }
    bool bad = false;

    if (r.mode == kModeFull) {   // f3 FULL record: element i of the tensor = the i-th value
      const u16* Vr = reinterpret_cast<const u16*>(rec + 16);
      const u8* Vr8 = rec + 16;
      for (u32 qq = lane; qq < nk; qq += 32) {
        const u64 i = p0 + qq;
        const u16 v = e8 ? (u16)Vr8[i] : Vr[i];
        if (kApply) {
          if (e8) reinterpret_cast<u8*>(W)[i] = (u8)v;
          else W[i] = v;
        } else {
          Io[qq] = (u32)i;
          Vo[qq] = v;
        }
      }
      continue;
    }

    if (r.codec == SYNC_CODEC_RAW) {
      const u32* Ir = reinterpret_cast<const u32*>(rec + 16) + p0;
      const u16* Vr = reinterpret_cast<const u16*>(rec + 16 + 4 * nnz) + p0;
      const u8* Vr8 = rec + 16 + 4 * nnz + p0;
      for (u32 qq = lane; qq < nk; qq += 32) {
        u32 idx = Ir[qq];
        u16 v = e8 ? (u16)Vr8[qq] : Vr[qq];
        if (kApply) {
          if (idx < lim) {
            if (e8) reinterpret_cast<u8*>(W)[idx] = (u8)v;
            else W[idx] = v;
          } else {
            bad = true;
          }
        } else {
          Io[qq] = idx;
          Vo[qq] = v;
        }
      }
      if (__any_sync(0xffffffffu, bad) && lane == 0) latch(status, SYNC_ERR_INDEX_RANGE);
      continue;
    }

    const bool esc = r.mode == kModeDelta16E;
    const u32* tbl = reinterpret_cast<const u32*>(rec + 16);
    const u64 s0 = esc ? 16 + 4 * (nch + 1) : 16;
    const u64 ib = esc ? 2ull * tbl[nch] : (r.mode ? 4ull : 2ull) * nnz;
    const u64 lo_off = s0 + pad_to(ib, 4);
    const u64 dir_off = lo_off + (e8 ? 0 : pad_to(nnz, 4));   // FP8: no lo plane
    const u32* de = reinterpret_cast<const u32*>(rec + dir_off + 16 * k);
    const u32 hi_off = de[0], hb = de[1], cm = de[2], base = de[3];
    bool corrupt = ((u64)hi_off + hb > r.rb) || (hi_off & 3u) || cm > 1 || (cm == 0 && hb != nk);
    const u8* blk = rec + hi_off;
    const u8* lo = rec + lo_off + p0;
    const u16* D = reinterpret_cast<const u16*>(rec + 16) + p0;
    const u32* A = reinterpret_cast<const u32*>(rec + 16) + p0;

    // f4 DELTA16E: this chunk's words [tbl[k], tbl[k+1]) of the escape-coded stream
    const u16* Ws = reinterpret_cast<const u16*>(rec + s0);
    u32 wptr = esc ? tbl[k] : 0u;
    const u32 wend = esc ? tbl[k + 1] : 0u;   // tbl[nch] = total words
    bool esc_bad = esc && (wptr > wend || (u64)wend > (ib >> 1));
    u32 x = kLow, nwords = 0;
    const u16* words = nullptr;
    if (!corrupt && cm == 1) {
      if (hb < 136) {
        corrupt = true;
      } else {
        const u32* bh = reinterpret_cast<const u32*>(blk);
        x = bh[lane];
        nwords = bh[32];
        u32 nsym = bh[33] & 0xFFFFu;
        if (nsym < 1 || nsym > 256 || 136ull + 4ull * nsym + 2ull * nwords != hb) {
          corrupt = true;
        } else {
          // entries owned lane-contiguously: lane handles entries [8*lane, 8*lane+8)
          u32 fsum = 0, e_s[8], e_f[8];
          bool eok = true;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            u32 e = lane * 8 + j;
            e_s[j] = 0;
            e_f[j] = 0;
            if (e < nsym) {
              u32 ent = bh[34 + e];
              e_s[j] = ent & 0xFFFFu;
              e_f[j] = ent >> 16;
              if (e_s[j] > 255 || e_f[j] == 0) eok = false;
              fsum += e_f[j];
            }
          }
          // ascending symbols: compare with the previous entry
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            u32 e = lane * 8 + j;
            if (e < nsym && e > 0) {
              u32 ps = (j > 0) ? e_s[j - 1] : 0xFFFFFFFFu;
              if (j == 0) ps = bh[34 + e - 1] & 0xFFFFu;
              if (e_s[j] <= ps) eok = false;
            }
          }
          u32 incl = warp_incl_scan(fsum);
          u32 total = __shfl_sync(0xffffffffu, incl, 31);
          if (!__all_sync(0xffffffffu, eok) || total != kM) {
            corrupt = true;
          } else {
            u32 c = incl - fsum;
            for (u32 s = lane; s < 256; s += 32) dm.freq[s] = 0;
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              if (e_f[j]) {
                dm.freq[e_s[j]] = (u16)e_f[j];
                dm.cum[e_s[j]] = (u16)c;
                c += e_f[j];
              }
            }
            __syncwarp();
            // fill slot -> symbol: entry by entry, lanes stride the entry's slot range
            for (u32 e = 0; e < nsym; ++e) {
              u32 ent = bh[34 + e];
              u32 s = ent & 0xFFFFu;
              u32 f = ent >> 16;
              u32 c0 = dm.cum[s];
              for (u32 sl = lane; sl < f; sl += 32) dm.slot2sym[c0 + sl] = (u8)s;
            }
            __syncwarp();
            words = reinterpret_cast<const u16*>(blk + 136 + 4 * nsym);
          }
        }
      }
    }
    if (__any_sync(0xffffffffu, corrupt)) {
      if (lane == 0) latch(status, SYNC_ERR_CORRUPT);
      continue;
    }

    const u32 G = (nk + 31) / 32;
    u32 ptr = 0;
    u32 carry = (r.mode == 0 || esc) ? base : 0u;
    bool range_bad = false, word_bad = false;
#if SS_DEC_FAST
    if (kApply && cm == 1 && r.mode == 0 && !esc && !e8) {
      // the common record kind (rANS hi chunk, DELTA16 indices, 16-bit values, apply) without the per-step
      // mode branches of the general loop below: same steps, same checks. A chunk is one warp's dependent
      // chain, so in a small sync (fewer chunks than warps) its instruction count is the launch's latency
      // (small syncs): 4B in 24 groups 6.68 -> 5.20 ms of decode, 30B at rho = 1% +-0, and the dense
      // variant at 3 CTAs / 4-deep with it beats 4 CTAs / 3-deep without it by 1-4% (rho = 10% / 5%).
      u32 nlb2[kPF], ndd2[kPF];
#pragma unroll
      for (int i = 0; i < kPF; ++i) {
        const u32 qq = (u32)i * 32 + lane;
        nlb2[i] = qq < nk ? (u32)lo[qq] : 0u;
        ndd2[i] = qq < nk ? (u32)D[qq] : 0u;
      }
      for (u32 g0 = 0; g0 < G; g0 += kPF) {
        u32 lb[kPF], dd[kPF];
#pragma unroll
        for (int i = 0; i < kPF; ++i) {
          lb[i] = nlb2[i];
          dd[i] = ndd2[i];
        }
        if (g0 + kPF < G) {
#pragma unroll
          for (int i = 0; i < kPF; ++i) {
            const u32 qq = (g0 + kPF + (u32)i) * 32 + lane;
            nlb2[i] = qq < nk ? (u32)lo[qq] : 0u;
            ndd2[i] = qq < nk ? (u32)D[qq] : 0u;
          }
        }
        if (lane < 8 && ptr + 64 * (lane + 1) < nwords)  // warm L1 with the next words
          asm volatile("prefetch.global.L1 [%0];" ::"l"(words + ptr + 64 * (lane + 1)));
#pragma unroll
        for (int i = 0; i < kPF; ++i) {
          const u32 gs = g0 + i;
          if (gs >= G) break;
          const u32 qq = gs * 32 + lane;
          const bool act = qq < nk;
          u32 sym = 0;
          if (act) {
            const u32 slot = x & (kM - 1);
            sym = dm.slot2sym[slot];
            x = (u32)dm.freq[sym] * (x >> 12) + slot - dm.cum[sym];
          }
          const bool need = act && x < kLow;
          const u32 nm = __ballot_sync(0xffffffffu, need);
          if (need) {
            const u32 pos = ptr + __popc(nm >> lane >> 1);
            if (pos < nwords) x = (x << 16) | words[pos];
            else word_bad = true;
          }
          ptr += __popc(nm);
          const u32 idx = carry + warp_incl_scan(dd[i]);
          carry = __shfl_sync(0xffffffffu, idx, 31);
          if (act) {
            if (idx < lim) W[idx] = (u16)((sym << 8) | lb[i]);
            else range_bad = true;
          }
        }
      }
      const bool endbad = word_bad || x != kLow || ptr != nwords;
      if (__any_sync(0xffffffffu, endbad) && lane == 0) latch(status, SYNC_ERR_CORRUPT);
      if (__any_sync(0xffffffffu, range_bad) && lane == 0) latch(status, SYNC_ERR_INDEX_RANGE);
      continue;
    }
#endif
    // software pipeline: the lo bytes and the index words (DELTA16 delta or
    // ABS32 index) of the next 8 steps are loaded while the current 8 decode
    u32 nlb[kPF], ndd[kPF];
    auto load_block = [&](u32 g0, u32* lb_, u32* dd_) {
#pragma unroll
      for (int i = 0; i < kPF; ++i) {
        const u32 qq = (g0 + i) * 32 + lane;
        const bool act = qq < nk;
        lb_[i] = (act && !e8) ? (u32)lo[qq] : 0u;
        dd_[i] = (act && !esc) ? (r.mode == 0 ? (u32)D[qq] : A[qq]) : 0u;
      }
    };
    load_block(0, nlb, ndd);
    for (u32 g0 = 0; g0 < G; g0 += kPF) {
      u32 lb[kPF], dd[kPF];
#pragma unroll
      for (int i = 0; i < kPF; ++i) {
        lb[i] = nlb[i];
        dd[i] = ndd[i];
      }
      if (g0 + kPF < G) load_block(g0 + kPF, nlb, ndd);
      if (cm == 1 && lane < 8 && ptr + 64 * (lane + 1) < nwords)  // warm L1 with the next words
        asm volatile("prefetch.global.L1 [%0];" ::"l"(words + ptr + 64 * (lane + 1)));
      // f4: stage this block's index words (from wptr) in shared memory, one coalesced pass, so the
      // per-step parse below reads shared memory instead of waiting on a global load every step
      const u32 wbase = wptr;
      if (esc) {
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kEscWin / 32; ++j) {
          const u32 o = (u32)j * 32 + lane;
          dm.win[o] = (wbase + o < wend) ? Ws[wbase + o] : (u16)0;
        }
        __syncwarp();
      }
#pragma unroll
      for (int i = 0; i < kPF; ++i) {
        const u32 gs = g0 + i;
        if (gs >= G) break;
        const u32 qq = gs * 32 + lane;
        const bool act = qq < nk;
        u32 s;
        if (cm == 1) {
          s = 0;
          if (act) {
            const u32 slot = x & (kM - 1);
            s = dm.slot2sym[slot];
            x = (u32)dm.freq[s] * (x >> 12) + slot - dm.cum[s];
          }
          const bool need = act && x < kLow;
          const u32 nm = __ballot_sync(0xffffffffu, need);
          if (need) {
            const u32 pos = ptr + __popc(nm >> lane >> 1);
            if (pos < nwords) x = (x << 16) | words[pos];
            else word_bad = true;
          }
          ptr += __popc(nm);
        } else {
          s = act ? blk[qq] : 0u;
        }
        u32 idx;
        if (r.mode == 0) {
          idx = carry + warp_incl_scan(dd[i]);
          carry = __shfl_sync(0xffffffffu, idx, 31);
        } else if (esc) {
          // parse the 32 elements of this step: lane l reads word wptr + l, shifted by one word for every
          // escape (two-word element) among the lanes before it; one ballot per escape in the step
          u32 pos = wptr + lane, dv = 0, n_esc = 0;
          bool done = !act;
          while (true) {
            const bool in = !done && pos < wend;
            if (!done && !in) {
              esc_bad = true;
              done = true;
            }
            const u32 w = in ? (u32)(pos - wbase < (u32)kEscWin ? dm.win[pos - wbase] : Ws[pos]) : 0u;
            const u32 m = __ballot_sync(0xffffffffu, in && (w & 0x8000u));
            if (m == 0) {
              if (in) dv = w;
              break;
            }
            const u32 e = __ffs(m) - 1;
            ++n_esc;                      // every round resolves exactly one escape (two words)
            if (in && lane < e) {
              dv = w;
              done = true;
            } else if (lane == e) {
              if (pos + 1 < wend)
                dv = ((w & 0x7FFFu) << 16) | (pos + 1 - wbase < (u32)kEscWin ? dm.win[pos + 1 - wbase] : Ws[pos + 1]);
              else esc_bad = true;
              done = true;
            } else if (in) {
              pos += 1;
            }
          }
          // the step consumed one word per active element plus one per escape
          wptr += __popc(__ballot_sync(0xffffffffu, act)) + n_esc;
          idx = carry + warp_incl_scan(dv);
          carry = __shfl_sync(0xffffffffu, idx, 31);
        } else {
          idx = dd[i];
        }
        if (act) {
          const u16 v = e8 ? (u16)s : (u16)((s << 8) | lb[i]);
          if (kApply) {
            if (idx < lim) {
              if (e8) reinterpret_cast<u8*>(W)[idx] = (u8)v;
              else W[idx] = v;
            } else {
              range_bad = true;
            }
          } else {
            Io[qq] = idx;
            Vo[qq] = v;
            if (idx >= lim) range_bad = true;
          }
        }
      }
    }
    if (cm == 1) {
      bool endbad = word_bad || x != kLow || ptr != nwords;
      if (__any_sync(0xffffffffu, endbad) && lane == 0) latch(status, SYNC_ERR_CORRUPT);
    }
    if (esc && __any_sync(0xffffffffu, esc_bad || wptr != wend) && lane == 0) latch(status, SYNC_ERR_CORRUPT);
    if (__any_sync(0xffffffffu, range_bad) && lane == 0) latch(status, SYNC_ERR_INDEX_RANGE);
  }
}

void launch_unpack(const u8* bucket, u64 bytes, u32 n_tensors, const u64* numel, sync_record_view* views,
                   u32 max_views, u32* n_records, u32* status, u32 dtype, cudaStream_t s) {
  k_unpack<<<1, 1024, 0, s>>>(bucket, bytes, n_tensors, numel, views, max_views, n_records, status, dtype);
  count_launch();
}

template <int kMinB, int kPF>
static void run_decode(const DecodeBatch& bb, u32 n_tensors, const u64* numel, u16* const* weights,
                       const sync_record_view* views, u32* I_out, u16* V_out, u64 out_cap, u32* status,
                       const u32* bad, u32 dtype, int grid, cudaStream_t s) {
  if (weights)
    k_decode<true, kMinB, kPF><<<grid, 256, 0, s>>>(bb, n_tensors, numel, weights, nullptr, nullptr, nullptr, 0,
                                                    status, bad, dtype);
  else
    k_decode<false, kMinB, kPF><<<grid, 256, 0, s>>>(bb, n_tensors, numel, nullptr, views, I_out, V_out, out_cap,
                                                     status, bad, dtype);
}

void launch_decode(const u8* const* buckets, const u64* bytes, u32 n_buckets, u32 n_tensors, const u64* numel,
                   u16* const* weights, const sync_record_view* views, u32* I_out, u16* V_out, u64 out_cap,
                   u32* status, const u32* crc_bad, u32 dtype, int grid, bool dense, cudaStream_t s) {
  for (u32 b0 = 0; b0 < n_buckets; b0 += kDecodeBatch) {
    DecodeBatch bb{};
    bb.n = n_buckets - b0 < kDecodeBatch ? n_buckets - b0 : kDecodeBatch;
    for (u32 i = 0; i < bb.n; ++i) {
      bb.bk[i] = buckets[b0 + i];
      bb.bytes[i] = bytes[b0 + i];
    }
    const u32* bad = crc_bad ? crc_bad + b0 : nullptr;
    // dense syncs are decode-bound: the 3-CTA / 4-deep variant keeps more chunks in flight; sparse ones are
    // scatter-bound and keep the 8-deep load pipeline
    if (dense && dtype == SYNC_DTYPE_FP8)   // no specialised loop for 8-bit values: the general loop's best
      run_decode<4, 3>(bb, n_tensors, numel, weights, views, I_out, V_out, out_cap, status, bad, dtype, grid, s);
    else if (dense)
      run_decode<SS_DEC_DMINB, SS_DEC_DPF>(bb, n_tensors, numel, weights, views, I_out, V_out, out_cap, status, bad,
                                           dtype, grid, s);
    else
      run_decode<SS_DEC_SMINB, SS_DEC_SPF>(bb, n_tensors, numel, weights, views, I_out, V_out, out_cap, status, bad,
                                           dtype, grid, s);
    count_launch();
  }
}

void launch_decode_table(const u64* t_hdr, const u64* t_off, const u64* t_size, u32 stride, const u8* base,
                         u32 max_buckets, u32 n_tensors, const u64* numel, u16* const* weights, u32* status,
                         u32 dtype, int grid, bool dense, cudaStream_t s) {
  for (u32 b0 = 0; b0 < max_buckets; b0 += kDecodeBatch) {   // a launch past the table's count decodes nothing
    DecodeBatch bb{};
    bb.t_hdr = t_hdr;
    bb.t_off = t_off;
    bb.t_size = t_size;
    bb.t_base = base;
    bb.t_b0 = b0;
    bb.t_stride = stride;
    if (dense && dtype == SYNC_DTYPE_FP8)
      run_decode<4, 3>(bb, n_tensors, numel, weights, nullptr, nullptr, nullptr, 0, status, nullptr, dtype, grid, s);
    else if (dense)
      run_decode<SS_DEC_DMINB, SS_DEC_DPF>(bb, n_tensors, numel, weights, nullptr, nullptr, nullptr, 0, status,
                                           nullptr, dtype, grid, s);
    else
      run_decode<SS_DEC_SMINB, SS_DEC_SPF>(bb, n_tensors, numel, weights, nullptr, nullptr, nullptr, 0, status,
                                           nullptr, dtype, grid, s);
    count_launch();
  }
}

}  // namespace ss
