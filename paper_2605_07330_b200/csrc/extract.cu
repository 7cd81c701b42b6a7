// extract.cu — K1: lossless sparse extraction (row a1).
//
// I = ascending { i : bits(old_i) != bits(new_i) }, V = new[I] per tensor,
// records contiguous in manifest order (Alg. 1 l.6; Alg. 2 l.5, P:312;
// sorted; bitwise compare, DESIGN C1).
//
// One pass over old+new (2S bytes, ~97% of a sync's HBM traffic at 1%
// density). Persistent, warp-specialised kernel (DESIGN §6 K1). A tile (the
// look-back unit) is 32768 elements of one tensor, streamed as four 8192-
// element sub-tiles (16 KB of old + 16 KB of new each):
//   * scheduler warp: claims the CTA's next tile from a global ticket
//     (atomicAdd), so tiles are taken in increasing order by CTAs that are
//     already running; resolves tile -> tensor / pointers a few tiles ahead
//     (tile table + one round of loads);
//   * copier warp: TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx)
//     of each sub-tile into one of kStages shared-memory stages;
//   * 8 consumer warps: per sub-tile, an 8-bit change mask per 128-bit vector,
//     one block scan, append (local index | value << 16) to the
//     tile's staging slot (a per-CTA ring of kSlots slots in global memory,
//     L2-resident); at the end of the tile publish its aggregate at once;
//   * writer warps: per tile, the global offset from the CTA's own previous
//     tile's prefix plus the counts published in between (the only wait on
//     other CTAs), then the coalesced write of (I, V).
//     The ring gives the writer kSlots tiles of slack, so the look-back
//     latency never stalls the stream.
//   * tiles denser than a slot (> 12.5%) take a slow path: the writer re-reads
//     the tile from global and writes directly.
// Forward progress without co-residency: a writer of tile j waits only for
// counts of tiles < j, all claimed (the ticket is monotonic) by CTAs that are
// running. By induction on the smallest unpublished tile m: its CTA's earlier
// tiles are < m, so their writers' windows are complete, the ring drains and
// m gets counted. Any number of resident CTAs (MPS, green contexts, a kernel
// spinning on another stream) therefore finishes the launch.
#include <cstdio>
#include <type_traits>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace ss {

constexpr int kXConsumers = kXThreads;            // 256 consumer threads (8 warps)
constexpr int xblock(int writers) { return kXConsumers + 64 + 32 * writers; }  // + copier, scheduler, writers
constexpr int kXQueue = 4;                        // tiles claimed + resolved ahead by the scheduler
constexpr u32 kStageBytes = (u32)kSub * 2 * 2;    // old + new, 16 KB each

struct ExtractArgs {
  const u16* const* old_ptrs;  // batched: device arrays of tensor pointers
  const u16* const* new_ptrs;
  const u16* old_single;       // single-tensor mode
  const u16* new_single;
  const u64* tile_prefix;      // [T+1]
  const u32* tile_tensor;      // [n_tiles] tile -> tensor
  const u64* numel;            // [T]
  u64 numel_single;
  u64 n_tiles;
  u32 n_tensors;
  u32* I;
  u16* V;
  u64 cap;
  u64* counts;                 // [T]
  u64* tile_state;             // [n_tiles]
  u32* ticket;                 // next unclaimed tile (zeroed before the launch)
  u32* stage_ring;             // [grid][kSlots][kSlotCap]
  u32* status;
  unsigned long long* prof;    // debug cycle counters (SS_XPROF=1), else null
};

struct TileJob {               // scheduler -> copier
  u64 tile;                    // ~0 = no more tiles
  u64 base;
  const u16* po;
  const u16* pn;
  u64 n;                       // tensor numel
  u32 t;
  u32 n_sub;
};

struct SubInfo {               // copier -> consumers, one per stage
  u64 tile;                    // ~0 = no more tiles
  u64 base;                    // first element of the sub-tile within its tensor
  const u16* po;
  const u16* pn;
  u32 t;
  u32 n_valid;                 // elements of this sub-tile inside the tensor
  u32 bulk;                    // elements delivered by the bulk copies (multiple of 8)
  u16 sub;                     // sub-tile index within the tile
  u16 n_sub;                   // sub-tiles in this tile
};

struct StagedTile {            // consumers -> writer, one per ring slot
  u64 tile;                    // ~0 = no more tiles
  u64 tile_base;               // first element of the tile within its tensor
  u64 tile_end;
  u64 prev;                    // the CTA's previous tile (~0 = none): the writer's window starts after it
  const u16* po;
  const u16* pn;
  u32 t;
  u32 count;
  u32 overflow;
  u32 pad;
};

__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kXConsumers) : "memory"); }

// ---------------------------------------------------------------- cross-CTA prefix
// Tile states: bit 63 = published, [62:0] = the tile's change count. Consumers
// publish a tile's count as soon as it is counted. The writer of CTA c already
// knows the inclusive prefix of c's previous tile p (claimed earlier from the
// ticket), so
//     excl(j) = incl(p) + sum_{i = p+1}^{j-1} count(i)
// needs only the counts in between (about G-1 of them when all CTAs run) —
// published by consumers, never by other writers, so no chain of look-backs
// forms. A CTA's first tile sums from tile 0. One L2 round trip reads 32 x kLB
// contiguous states; entries not yet published are re-polled alone, with a
// short back-off.
constexpr int kLB = 16;  // window 512 >= G - 1 for G <= 513 CTAs
constexpr u64 kPublished = 1ull << 63;

__device__ __forceinline__ void publish_count(u64* state, u64 tile, u64 cnt) {
  st_relaxed(&state[tile], kPublished | cnt);
}

// Sum of the published counts of tiles [lo, hi) (full warp; waits until all are published).
__device__ __forceinline__ u64 window_sum(u64* state, u64 lo, u64 hi) {
  const u32 lane = lane_id();
  u64 acc = 0;
  for (u64 base = lo; base < hi; base += 32 * kLB) {
    u32 pending = 0;
    u64 part = 0;
#pragma unroll
    for (int i = 0; i < kLB; ++i)
      if (base + lane * kLB + i < hi) pending |= 1u << i;
    while (true) {
#pragma unroll
      for (int i = 0; i < kLB; ++i) {
        if (pending & (1u << i)) {
          const u64 v = ld_relaxed(&state[base + lane * kLB + i]);
          if (v & kPublished) {
            part += v & ~kPublished;
            pending &= ~(1u << i);
          }
        }
      }
      if (!__any_sync(0xffffffffu, pending != 0)) break;
      __nanosleep(128);
    }
    acc += warp_sum64(part);
  }
  return acc;
}

// ---------------------------------------------------------------- per-vector helpers
__device__ __forceinline__ uint4 load8_direct(const u16* p, u64 e, u64 n) {
  u16 h[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) h[k] = (e + k < n) ? p[e + k] : (u16)0;
  return make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16), h[6] | (h[7] << 16));
}

__device__ __forceinline__ u32 change_mask(const uint4& o, const uint4& n) {
  u32 x0 = o.x ^ n.x, x1 = o.y ^ n.y, x2 = o.z ^ n.z, x3 = o.w ^ n.w;
  return ((x0 & 0xFFFFu) ? 1u : 0u) | ((x0 >> 16) ? 2u : 0u) | ((x1 & 0xFFFFu) ? 4u : 0u) |
         ((x1 >> 16) ? 8u : 0u) | ((x2 & 0xFFFFu) ? 16u : 0u) | ((x2 >> 16) ? 32u : 0u) |
         ((x3 & 0xFFFFu) ? 64u : 0u) | ((x3 >> 16) ? 128u : 0u);
}

// 8-bit elements (FP8, f2): 16 bytes per vector
__device__ __forceinline__ uint4 load16_direct8(const uint8_t* p, u64 e, u64 n) {
  u32 w[4] = {0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < 16; ++k)
    if (e + k < n) w[k >> 2] |= (u32)p[e + k] << (8 * (k & 3));
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// bit 4j + b <-> byte b of word j differs. Per word: the high bit of every nonzero byte of x
// ((x & 0x7F..) + 0x7F.. sets it for nonzero low 7 bits, | x for the top bit), then one multiply
// gathers bits 7, 15, 23, 31 into bits 28..31 (the partial products land on distinct bits: no carries).
__device__ __forceinline__ u32 byte_nz4(u32 x) {
  const u32 t = (((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;
  return (t * 0x00204081u) >> 28;
}
__device__ __forceinline__ u32 change_mask8(const uint4& o, const uint4& n) {
  return byte_nz4(o.x ^ n.x) | (byte_nz4(o.y ^ n.y) << 4) | (byte_nz4(o.z ^ n.z) << 8) |
         (byte_nz4(o.w ^ n.w) << 12);
}

__device__ __forceinline__ u16 lane8(const uint4& v, int b) {
  const u32 w[4] = {v.x, v.y, v.z, v.w};
  return (u16)((w[b >> 2] >> (8 * (b & 3))) & 0xFFu);
}

__device__ __forceinline__ u16 lane16(const uint4& v, int b) {
  const u64 lo64 = v.x | ((u64)v.y << 32), hi64 = v.z | ((u64)v.w << 32);
  return (u16)(((b < 4) ? lo64 : hi64) >> ((b & 3) * 16));
}

// kB = element bytes: 2 (BF16 / FP16) or 1 (FP8, f2). A 16-byte vector holds kEPV = 16 / kB elements; a
// sub-tile (one stage: 16 KB of old + 16 KB of new) holds kSubE = 256 threads x 4 vectors x kEPV elements;
// a tile is always kTile = 32768 elements (local indices fit 16 bits; the tile tables are shared).
template <bool kSingle, int kStages, int kWriters, int kB = 2>
__global__ void __launch_bounds__(xblock(kWriters), 2) k_extract(ExtractArgs a) {
  constexpr u32 kEPV = 16 / kB;
  constexpr u64 kSubE = (u64)kXThreads * kXVec * kEPV;
  extern __shared__ __align__(128) u8 smem[];
  u8* data = smem;
  u64* full = reinterpret_cast<u64*>(smem + kStages * kStageBytes);
  u64* empty = full + kStages;
  u64* qfull = empty + kStages;
  u64* qempty = qfull + kXQueue;
  u64* sfull = qempty + kXQueue;
  u64* sempty = sfull + kSlots;
  SubInfo* info = reinterpret_cast<SubInfo*>(sempty + kSlots);
  TileJob* jobs = reinterpret_cast<TileJob*>(info + kStages);
  StagedTile* meta = reinterpret_cast<StagedTile*>(jobs + kXQueue);
  u64* s_wsum = reinterpret_cast<u64*>(meta + kSlots);  // [0..7] scan (2 x 8 u32)
  u64* s_incl = s_wsum + 8;                              // writer hand-off: inclusive prefix
  u32* s_done = reinterpret_cast<u32*>(s_wsum + 9);      // tiles whose prefix is known
  u32* ring = a.stage_ring + (size_t)blockIdx.x * kSlots * kSlotCap;
  const u32 tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (tid == 0) {
    *s_done = 0;
    *s_incl = 0;
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kXConsumers / 32);
    }
    for (int q = 0; q < kXQueue; ++q) {
      mbar_init(&qfull[q], 1);
      mbar_init(&qempty[q], 1);
    }
    for (int q = 0; q < (int)kSlots; ++q) {
      mbar_init(&sfull[q], 1);
      mbar_init(&sempty[q], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kXConsumers / 32 + 1) {
    // ------------------------------------------------------------ scheduler warp
    for (u32 k = 0;; ++k) {
      const u32 q = k % kXQueue;
      if (k >= (u32)kXQueue) mbar_wait(&qempty[q], ((k / kXQueue) - 1) & 1);
      u32 tk = 0;
      if (lane == 0) tk = atomicAdd(a.ticket, 1u);
      const u64 tile = __shfl_sync(0xffffffffu, tk, 0);
      if (tile >= a.n_tiles) {
        if (lane == 0) {
          jobs[q].tile = ~0ull;
          mbar_arrive(&qfull[q]);
        }
        break;
      }
      const u32 t = kSingle ? 0u : a.tile_tensor[tile];
      u64 v = 0;
      if (lane == 0) v = kSingle ? a.numel_single : a.numel[t];
      if (lane == 1) v = (u64)(kSingle ? a.old_single : a.old_ptrs[t]);
      if (lane == 2) v = (u64)(kSingle ? a.new_single : a.new_ptrs[t]);
      if (lane == 3) v = kSingle ? 0ull : a.tile_prefix[t];
      const u64 n = __shfl_sync(0xffffffffu, v, 0);
      const u64 po = __shfl_sync(0xffffffffu, v, 1);
      const u64 pn = __shfl_sync(0xffffffffu, v, 2);
      const u64 tp = __shfl_sync(0xffffffffu, v, 3);
      if (lane == 0) {
        TileJob j;
        j.tile = tile;
        j.base = (tile - tp) * kTile;
        j.po = reinterpret_cast<const u16*>(po);
        j.pn = reinterpret_cast<const u16*>(pn);
        j.n = n;
        j.t = t;
        const u64 rem = n - j.base;
        const u64 nv = rem < kTile ? rem : kTile;
        j.n_sub = (u32)((nv + kSubE - 1) / kSubE);
        jobs[q] = j;
        mbar_arrive(&qfull[q]);
      }
      __syncwarp();
    }
    return;
  }

  if (warp == kXConsumers / 32) {
    // ------------------------------------------------------------ copier warp
    const u64 pol = policy_evict_first();
    u32 it = 0;
    long long p_copy = 0;
    for (u32 k = 0;; ++k) {
      const u32 q = k % kXQueue;
      mbar_wait(&qfull[q], (k / kXQueue) & 1);
      const TileJob j = jobs[q];
      __syncwarp();
      if (lane == 0) mbar_arrive(&qempty[q]);
      const bool done = j.tile == ~0ull;
      const u32 n_sub = done ? 1u : j.n_sub;
      const bool aligned = ((((uintptr_t)j.po) | ((uintptr_t)j.pn)) & 15u) == 0;
      for (u32 sub = 0; sub < n_sub; ++sub, ++it) {
        const u32 s = it % kStages;
        if (it >= (u32)kStages) {
          const long long c0 = clock64();
          mbar_wait(&empty[s], ((it / kStages) - 1) & 1);
          p_copy += clock64() - c0;
        }
        if (lane == 0) {
          SubInfo si;
          if (done) {
            si.tile = ~0ull;
            info[s] = si;
            mbar_arrive(&full[s]);
          } else {
            const u64 sb = j.base + (u64)sub * kSubE;
            const u64 rem = j.n - sb;
            const u32 n_valid = (u32)(rem < kSubE ? rem : kSubE);
            const u32 bulk = aligned ? (n_valid & ~(kEPV - 1)) : 0u;   // whole 16-byte vectors
            si.tile = j.tile;
            si.base = sb;
            si.po = j.po;
            si.pn = j.pn;
            si.t = j.t;
            si.n_valid = n_valid;
            si.bulk = bulk;
            si.sub = (u16)sub;
            si.n_sub = (u16)n_sub;
            info[s] = si;
            u8* dst = data + (size_t)s * kStageBytes;
            if (bulk) {
              const u8* po8 = reinterpret_cast<const u8*>(j.po) + kB * sb;
              const u8* pn8 = reinterpret_cast<const u8*>(j.pn) + kB * sb;
              mbar_arrive_tx(&full[s], 2u * kB * bulk);
              bulk_g2s(dst, po8, kB * bulk, &full[s], pol);
              bulk_g2s(dst + kStageBytes / 2, pn8, kB * bulk, &full[s], pol);
            } else {
              mbar_arrive(&full[s]);
            }
          }
        }
        __syncwarp();
      }
      if (done) break;
    }
    if (a.prof && lane == 0) atomicAdd(&a.prof[2], (unsigned long long)p_copy);
    return;
  }

  if (warp >= kXConsumers / 32 + 2) {
    // ------------------------------------------------------------ writer warps
    // kWriters warps take the CTA's tiles round-robin. The expensive part — the
    // window of G-1 published counts — runs concurrently in every writer; only
    // the cheap inclusive-prefix hand-off between consecutive tiles is serial
    // (through shared memory).
    const u32 w = warp - (kXConsumers / 32 + 2);
    const u64 keep = policy_evict_last();
    long long p_w = 0, p_lb = 0, p_wr = 0, n_t = 0, p_win = 0, p_span = 0;
    for (u32 k = w;; k += kWriters) {
      const u32 b = k % kSlots;
      long long c0 = clock64();
      mbar_wait(&sfull[b], (k / kSlots) & 1);
      long long c1 = clock64();
      p_w += c1 - c0;
      const StagedTile m = meta[b];
      if (m.tile == ~0ull) break;
      const bool first = m.prev == ~0ull;
      const u64 win = window_sum(a.tile_state, first ? 0ull : m.prev + 1, m.tile);
      const long long c1b = clock64();
      p_win += c1b - c1;
      p_span += first ? 0 : (long long)(m.tile - m.prev - 1);
      // wait for the inclusive prefix of this CTA's previous tile (k - 1)
      while (*(volatile u32*)s_done != k) __nanosleep(32);
      const u64 prefix = (first ? 0ull : *(volatile u64*)s_incl) + win;
      __syncwarp();
      if (lane == 0) {
        *(volatile u64*)s_incl = prefix + m.count;
        __threadfence_block();
        *(volatile u32*)s_done = k + 1;
      }
      long long c2 = clock64();
      p_lb += c2 - c1;
      ++n_t;
      if (lane == 0 && m.count) atomicAdd((unsigned long long*)&a.counts[m.t], (unsigned long long)m.count);
      const u32* stg = ring + b * kSlotCap;
      if (!m.overflow) {
        // lane l writes entries q0 + 32c + l: every store instruction covers 32 consecutive I (128 B) and
        // V (64 B) slots; 16 staged entries per lane in flight, the next batch loaded before this one is
        // stored (the ring is L2-resident)
        constexpr int kE = 16;
        const bool room = prefix + m.count <= a.cap;
        u32 nx[kE];
#pragma unroll
        for (int c = 0; c < kE; ++c) {
          const u32 q = c * 32 + lane;
          nx[c] = q < m.count ? ld_hint(stg + q, keep) : 0u;
        }
        for (u32 q0 = 0; q0 < m.count; q0 += 32 * kE) {
          u32 ev[kE];
#pragma unroll
          for (int c = 0; c < kE; ++c) ev[c] = nx[c];
          if (q0 + 32 * kE < m.count) {
#pragma unroll
            for (int c = 0; c < kE; ++c) {
              const u32 q = q0 + 32 * kE + c * 32 + lane;
              nx[c] = q < m.count ? ld_hint(stg + q, keep) : 0u;
            }
          }
#pragma unroll
          for (int c = 0; c < kE; ++c) {
            const u32 q = q0 + c * 32 + lane;
            if (q < m.count) {
              const u64 pos = prefix + q;
              if (room || pos < a.cap) {   // streaming stores: the output is not re-read by this kernel
                __stcs(a.I + pos, (u32)(m.tile_base + (ev[c] & 0xFFFFu)));
                __stcs(a.V + pos, (u16)(ev[c] >> 16));
              } else {
                latch(a.status, SYNC_ERR_CAPACITY);
              }
            }
          }
        }
      } else {
        // slow path (tile denser than a slot): re-read it from global
        u64 run = prefix;
        for (u64 e0 = m.tile_base; e0 < m.tile_end; e0 += 32 * kEPV) {
          const u64 e = e0 + lane * kEPV;
          uint4 vo, vd;
          u32 mk;
          if (kB == 1) {
            vo = load16_direct8(reinterpret_cast<const u8*>(m.po), e, m.tile_end);
            vd = load16_direct8(reinterpret_cast<const u8*>(m.pn), e, m.tile_end);
            mk = change_mask8(vo, vd);
          } else {
            vo = load8_direct(m.po, e, m.tile_end);
            vd = load8_direct(m.pn, e, m.tile_end);
            mk = change_mask(vo, vd);
          }
          const u32 c = __popc(mk);
          const u32 inc = warp_incl_scan(c);
          u64 pos = run + inc - c;
          while (mk) {
            int bb = __ffs(mk) - 1;
            mk &= mk - 1;
            if (pos < a.cap) {
              a.I[pos] = (u32)(e + bb);
              a.V[pos] = kB == 1 ? lane8(vd, bb) : lane16(vd, bb);
            } else {
              latch(a.status, SYNC_ERR_CAPACITY);
            }
            ++pos;
          }
          run += __shfl_sync(0xffffffffu, inc, 31);
        }
      }
      __syncwarp();
      p_wr += clock64() - c2;
      if (lane == 0) mbar_arrive(&sempty[b]);
    }
    if (a.prof && lane == 0) {
      atomicAdd(&a.prof[3], (unsigned long long)p_w);
      atomicAdd(&a.prof[4], (unsigned long long)p_lb);
      atomicAdd(&a.prof[5], (unsigned long long)p_wr);
      atomicAdd(&a.prof[8], (unsigned long long)n_t);
      atomicAdd(&a.prof[10], (unsigned long long)p_win);
      atomicAdd(&a.prof[11], (unsigned long long)p_span);
    }
    return;
  }

  // -------------------------------------------------------------- consumer warps
  const u64 keep = policy_evict_last();   // the staging ring: written here, read back by the writers
  u32 tile_cnt = 0, tseq = 0, b = 0;
  u64 prev_tile = ~0ull;
  bool overflow = false;
  long long p_full = 0, p_se = 0, n_s = 0;
  const long long c_start = clock64();
  for (u32 it = 0;; ++it) {
    const u32 s = it % kStages;
    const long long c0 = clock64();
    mbar_wait(&full[s], (it / kStages) & 1);
    p_full += clock64() - c0;
    ++n_s;
    const SubInfo si = info[s];
    if (si.tile == ~0ull) {
      for (u32 kk = tseq; kk < tseq + kWriters; ++kk) {  // one sentinel per writer warp
        b = kk % kSlots;
        if (kk >= kSlots) mbar_wait(&sempty[b], ((kk / kSlots) - 1) & 1);
        if (tid == 0) {
          meta[b].tile = ~0ull;
          mbar_arrive(&sfull[b]);
        }
      }
      break;
    }
    if (si.sub == 0) {
      b = tseq % kSlots;
      const long long c1 = clock64();
      if (tseq >= kSlots) mbar_wait(&sempty[b], ((tseq / kSlots) - 1) & 1);  // writer done with slot b
      p_se += clock64() - c1;
      tile_cnt = 0;
      overflow = false;
    }
    const uint4* so = reinterpret_cast<const uint4*>(data + (size_t)s * kStageBytes);
    const uint4* sn = reinterpret_cast<const uint4*>(data + (size_t)s * kStageBytes + kStageBytes / 2);
    const u16* sn16 = reinterpret_cast<const u16*>(data + (size_t)s * kStageBytes + kStageBytes / 2);
    const u8* sn8 = data + (size_t)s * kStageBytes + kStageBytes / 2;

    // Thread t owns the 4 consecutive vectors 4t..4t+3 (elements 32t..32t+31), so
    // thread order == index order and one u32 scan places every change. Load u
    // reads vector 4t + ((t/2 + u) & 3): the 8 threads of each LDS.128 phase hit
    // 8 distinct 16-byte columns (conflict-free).
    // bit kEPV*j + b <-> element 4*kEPV*t + kEPV*j + b (32 elements per thread for 16-bit, 64 for 8-bit)
    using MaskT = typename std::conditional<kB == 1, u64, u32>::type;
    MaskT masks = 0;
    const u32 rot = (tid >> 1) & 3;
#pragma unroll
    for (int u = 0; u < kXVec; ++u) {
      const u32 j = (rot + (u32)u) & 3;
      const u32 v = 4 * tid + j;  // vector index within the sub-tile
      uint4 vo, vd;
      if (v * kEPV + kEPV <= si.bulk) {
        vo = so[v];
        vd = sn[v];
      } else if (v * kEPV < si.n_valid) {
        if (kB == 1) {
          vo = load16_direct8(reinterpret_cast<const u8*>(si.po), si.base + v * kEPV, si.base + si.n_valid);
          vd = load16_direct8(reinterpret_cast<const u8*>(si.pn), si.base + v * kEPV, si.base + si.n_valid);
        } else {
          vo = load8_direct(si.po, si.base + v * 8, si.base + si.n_valid);
          vd = load8_direct(si.pn, si.base + v * 8, si.base + si.n_valid);
        }
      } else {
        vo = vd = make_uint4(0, 0, 0, 0);
      }
      masks |= (MaskT)(kB == 1 ? change_mask8(vo, vd) : change_mask(vo, vd)) << (kEPV * j);
    }
    const u32 cnt = kB == 1 ? (u32)__popcll((u64)masks) : (u32)__popc((u32)masks);
    // block exclusive scan (one barrier; s_wsum double-buffered by sub-tile parity)
    const u32 incl = warp_incl_scan(cnt);
    u32* wsum = reinterpret_cast<u32*>(s_wsum) + (it & 1) * 8;
    if (lane == 31) wsum[warp] = incl;
    consumer_bar();
    u32 wexcl = 0, st_total = 0;
#pragma unroll
    for (int w = 0; w < kXConsumers / 32; ++w) {
      const u32 x = wsum[w];
      wexcl += (w < (int)warp) ? x : 0u;
      st_total += x;
    }
    if (!overflow && tile_cnt + st_total <= kSlotCap) {
      u32* stg = ring + b * kSlotCap;
      u32 pos = tile_cnt + wexcl + incl - cnt;
      constexpr u32 kPerT = 4 * kEPV;   // elements per thread
      const u32 local = (u32)si.sub * (u32)kSubE + kPerT * tid;
      MaskT mk = masks;
      if (kPerT * tid + kPerT <= si.bulk) {
        // all of this thread's elements are in the stage: values from shared memory, a running
        // ring pointer, (local | value << 16) in one byte permute (local < 2^15 within a tile)
        u32* sp = stg + pos;
        while (mk) {
          const int bb = (kB == 1 ? __ffsll((long long)mk) : __ffs((int)mk)) - 1;
          mk &= mk - 1;
          const u32 val = kB == 1 ? (u32)sn8[kPerT * tid + bb] : (u32)sn16[kPerT * tid + bb];
          st_hint(sp++, __byte_perm(local + (u32)bb, val, 0x5410), keep);
        }
      }
      while (mk) {
        const int bb = (kB == 1 ? __ffsll((long long)mk) : __ffs((int)mk)) - 1;
        mk &= mk - 1;
        u16 val;
        if (kB == 1) {
          if (kPerT * tid + bb + 1 <= si.bulk) val = sn8[kPerT * tid + bb];
          else val = reinterpret_cast<const u8*>(si.pn)[si.base + kPerT * tid + bb];
        } else {
          if (kPerT * tid + bb + 1 <= si.bulk) val = sn16[kPerT * tid + bb];
          else val = si.pn[si.base + kPerT * tid + bb];
        }
        st_hint(stg + pos++, (local + bb) | ((u32)val << 16), keep);
      }
    } else {
      overflow = true;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // 8 warp arrivals release the stage to the copier
    tile_cnt += st_total;
    if (si.sub + 1 < si.n_sub) continue;

    // ---- end of tile: publish the aggregate now, hand the staged list to the writer
    consumer_bar();                                     // all staging writes done
    if (tid == 0) {
      publish_count(a.tile_state, si.tile, tile_cnt);
      StagedTile m;
      m.tile = si.tile;
      m.tile_base = si.base - (u64)si.sub * kSubE;
      m.tile_end = si.base + si.n_valid;
      m.prev = prev_tile;
      m.po = si.po;
      m.pn = si.pn;
      m.t = si.t;
      m.count = tile_cnt;
      m.overflow = overflow ? 1u : 0u;
      m.pad = 0;
      meta[b] = m;
      mbar_arrive(&sfull[b]);
    }
    prev_tile = si.tile;
    ++tseq;
  }
  if (a.prof && tid == 0) {
    atomicAdd(&a.prof[0], (unsigned long long)p_full);
    atomicAdd(&a.prof[1], (unsigned long long)p_se);
    atomicAdd(&a.prof[6], (unsigned long long)(clock64() - c_start));
    atomicAdd(&a.prof[9], (unsigned long long)n_s);
  }
}

template <int kStages>
static size_t extract_smem() {
  return (size_t)kStages * kStageBytes + 2 * (kStages + kXQueue + kSlots) * 8 + kStages * sizeof(SubInfo) +
         kXQueue * sizeof(TileJob) + kSlots * sizeof(StagedTile) + 16 * 8;
}

template <bool kSingle, int kStages, int kWriters, int kB = 2>
static void launch_k(const ExtractArgs& a, cudaStream_t s) {
  constexpr int kXBlock = xblock(kWriters);
  static int grid_cap[kMaxDevices] = {};   // per device: the attribute is a per-device setting
  const size_t sm = extract_smem<kStages>();
  const int dev = current_device();
  if (!grid_cap[dev]) {
    cudaFuncSetAttribute(k_extract<kSingle, kStages, kWriters, kB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    int n_sm = 148, per = 1;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_extract<kSingle, kStages, kWriters, kB>, kXBlock, sm);
    int cap = n_sm * (per > 0 ? per : 1);
    grid_cap[dev] = cap > (int)kMaxExtractCtas ? (int)kMaxExtractCtas : cap;
  }
  static int env_cap = -1;   // SS_XCTAS: a K1-only grid cap (dev experiments: leave SMs to concurrent kernels)
  if (env_cap < 0) env_cap = getenv("SS_XCTAS") ? atoi(getenv("SS_XCTAS")) : 0;
  u64 cap = (u64)clamp_ctas(grid_cap[dev]);
  if (env_cap > 0 && (u64)env_cap < cap) cap = (u64)env_cap;
  u64 grid = a.n_tiles < cap ? a.n_tiles : cap;
  static unsigned long long* prof = nullptr;
  static int want_prof = -1;
  if (want_prof < 0) want_prof = getenv("SS_XPROF") ? 1 : 0;
  ExtractArgs b = a;
  if (want_prof) {  // debug instrumentation only
    if (!prof) cudaMalloc(&prof, 16 * sizeof(unsigned long long));
    cudaMemsetAsync(prof, 0, 16 * sizeof(unsigned long long), s);
    b.prof = prof;
  }
  k_extract<kSingle, kStages, kWriters, kB><<<(unsigned)grid, kXBlock, sm, s>>>(b);
  count_launch();
  if (want_prof) {
    unsigned long long h[16];
    cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const double G = (double)grid;
    fprintf(stderr,
            "[xprof] grid %llu tiles/cta %.1f subs/cta %.1f | per CTA kcycles: consumer total %.1f wait_full %.1f "
            "wait_slot %.1f | copier wait_empty %.1f | writer wait %.1f lookback %.1f (window %.1f, mean window "
            "%.0f tiles) write %.1f\n",
            (unsigned long long)grid, h[8] / G, h[9] / G, h[6] / G / 1e3, h[0] / G / 1e3, h[1] / G / 1e3,
            h[2] / G / 1e3, h[3] / G / 1e3, h[4] / G / 1e3, h[10] / G / 1e3, h[8] ? (double)h[11] / h[8] : 0.0,
            h[5] / G / 1e3);
  }
}

// 3 stages (two CTAs per SM) and 4 writer warps by default (round 2, with ticketed tiles, same-box A/B: 4 writers
// beat 3 by 0.4% at 1% density and 1.6% at 10%; round 1's static schedule had preferred 3); SS_XWRITERS=2|3 and
// (with 2 writers) SS_XSTAGES=2|4 select other instantiations for experiments.
template <bool kSingle>
static void launch(const ExtractArgs& a, cudaStream_t s) {
  static int stages = 0, writers = 0;
  if (!stages) {
    const char* e = getenv("SS_XSTAGES");
    stages = e ? atoi(e) : 3;
    const char* w = getenv("SS_XWRITERS");
    writers = w ? atoi(w) : 4;
  }
  if (writers == 2) {
    if (stages == 2) launch_k<kSingle, 2, 2>(a, s);
    else if (stages == 4) launch_k<kSingle, 4, 2>(a, s);
    else launch_k<kSingle, 3, 2>(a, s);
  } else if (writers == 3) {
    launch_k<kSingle, 3, 3>(a, s);
  } else {
    launch_k<kSingle, 3, 4>(a, s);
  }
}

void launch_extract_batched(const u16* const* d_old, const u16* const* d_new, const u64* tile_prefix,
                            const u32* tile_tensor, const u64* numel, u32 n_tensors, u64 n_tiles, u32* I, u16* V,
                            u64 cap, u64* counts, u64* tile_state, u32* ticket, u32* stage_ring, u32* status,
                            cudaStream_t s, int elem_bytes) {
  if (n_tiles == 0) return;
  ExtractArgs a{};
  a.old_ptrs = d_old;
  a.new_ptrs = d_new;
  a.tile_prefix = tile_prefix;
  a.tile_tensor = tile_tensor;
  a.numel = numel;
  a.n_tiles = n_tiles;
  a.n_tensors = n_tensors;
  a.I = I;
  a.V = V;
  a.cap = cap;
  a.counts = counts;
  a.tile_state = tile_state;
  a.ticket = ticket;
  a.stage_ring = stage_ring;
  a.status = status;
  if (elem_bytes == 1) launch_k<false, 3, 4, 1>(a, s);   // FP8: the same pipeline on 8-bit elements
  else launch<false>(a, s);
}

void launch_extract_single(const u16* d_old, const u16* d_new, u64 n, u32* I, u16* V, u64 cap, u64* count,
                           u64* tile_state, u32* ticket, u32* stage_ring, u32* status, cudaStream_t s) {
  u64 n_tiles = (n + kTile - 1) / kTile;
  if (n_tiles == 0) return;
  ExtractArgs a{};
  a.old_single = d_old;
  a.new_single = d_new;
  a.numel_single = n;
  a.n_tiles = n_tiles;
  a.n_tensors = 1;
  a.I = I;
  a.V = V;
  a.cap = cap;
  a.counts = count;
  a.tile_state = tile_state;
  a.ticket = ticket;
  a.stage_ring = stage_ring;
  a.status = status;
  launch<true>(a, s);
}

}  // namespace ss
