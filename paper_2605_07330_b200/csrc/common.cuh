// common.cuh — device helpers shared by the sm_100a kernels of libsparsesync.
// (Product code; shares nothing with oracle/.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cuda/atomic>

#include "../../include/sparsesync.h"

namespace ss {

typedef uint64_t u64;
typedef uint32_t u32;
typedef uint16_t u16;
typedef uint8_t u8;

constexpr u32 kChunk = SYNC_CHUNK;         // values per chunk
constexpr u32 kLanes = 32;                  // rANS interleave width == warp width
constexpr u32 kProbBits = 12;
constexpr u32 kM = 1u << kProbBits;         // 4096
constexpr u32 kLow = 1u << 16;              // rANS lower bound
constexpr u32 kMagic = 0x424C5253u;         // "SRLB"
constexpr u32 kVersion = 1;
constexpr u64 kBucketAlign = 256;
constexpr u64 kCrcSegBytes = 65536;         // CRC-32 segment (one CTA of k_crc_seg)
// rANS block head kept by the stats pass: 32 lane states, nwords, nsym, <= 256 entries
constexpr u32 kRhdrWords = 34 + 256;

// Extract tiling: a sub-tile is 256 threads x 4 x uint4 (8 bf16) = 8192 elements
// (one TMA stage: 16 KB of old + 16 KB of new); a tile (the look-back unit) is
// kSubPerTile sub-tiles = 32768 elements (local indices fit 16 bits).
constexpr int kXThreads = 256;
constexpr int kXVec = 4;
constexpr u64 kSub = (u64)kXThreads * kXVec * 8;
constexpr u32 kSubPerTile = 4;
constexpr u64 kTile = kSub * kSubPerTile;
// Per-CTA staging ring (global memory, L2-resident) between the extract
// consumers and its writer warp: kSlots tiles of up to kSlotCap changes.
constexpr u32 kSlots = 16;
constexpr u32 kSlotCap = 4096;
constexpr u32 kMaxExtractCtas = 512;
// bytes of the extract staging ring for a launch over n_tiles tiles
__host__ __device__ inline u64 stage_ring_bytes(u64 n_tiles) {
  const u64 ctas = n_tiles < kMaxExtractCtas ? n_tiles : kMaxExtractCtas;
  return ctas * kSlots * kSlotCap * 4;
}

// Look-back tile state: [63:62] flag, [61:0] value.
constexpr u64 kFlagA = 1ull << 62;
constexpr u64 kFlagP = 2ull << 62;
constexpr u64 kValMask = (1ull << 62) - 1;

__host__ __device__ inline u64 pad_to(u64 x, u64 a) { return (x + a - 1) / a * a; }

__device__ __forceinline__ u64 ld_relaxed(const u64* p) {
  return cuda::atomic_ref<u64, cuda::thread_scope_device>(*const_cast<u64*>(p))
      .load(cuda::std::memory_order_relaxed);
}
__device__ __forceinline__ void st_relaxed(u64* p, u64 v) {
  cuda::atomic_ref<u64, cuda::thread_scope_device>(*p).store(v, cuda::std::memory_order_relaxed);
}

// Streaming 128-bit load: read once, no L1 allocation.
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Latch the first error into the device status word (stored as -code).
__device__ __forceinline__ void latch(u32* status, int code) {
  if (status) atomicCAS(status, 0u, (u32)(-code));
}

__device__ __forceinline__ u32 lane_id() { return threadIdx.x & 31u; }

// Warp-cooperative search: largest idx in [0, n) with key_at(idx) <= key,
// for a non-decreasing key_at with key_at(0) <= key. 32-ary, ceil(log32 n) rounds.
template <typename F>
__device__ __forceinline__ u32 warp_upper_search(u32 n, u64 key, F key_at) {
  const u32 lane = lane_id();
  u32 lo = 0, hi = n;
  while (hi - lo > 1) {
    u32 step = (hi - lo + 31) / 32;
    u32 idx = lo + lane * step;
    bool ok = idx < hi && key_at(idx) <= key;
    u32 m = __ballot_sync(0xffffffffu, ok);
    u32 last = 31 - __clz(m);  // bit 0 is always set
    u32 nlo = lo + last * step;
    u32 nhi = nlo + step;
    lo = nlo;
    hi = nhi < hi ? nhi : hi;
  }
  return lo;
}

// Warp inclusive scan (u32 / u64).
__device__ __forceinline__ u32 warp_incl_scan(u32 v) {
  const u32 lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    u32 t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= (u32)o) v += t;
  }
  return v;
}
__device__ __forceinline__ u64 warp_incl_scan64(u64 v) {
  const u32 lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    u64 t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= (u32)o) v += t;
  }
  return v;
}
__device__ __forceinline__ u64 warp_sum64(u64 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Exact floor(x / f) for 1 <= f <= 4096 and x < 2^32 from rcp = rcp_of(f):
// floor(2^32 / f) for f >= 2 (so umulhi(x, rcp) > x/f - 1) and 2^32 - 1 for f = 1
// (umulhi = x - 1): the estimate is at most one below the quotient.
__host__ __device__ __forceinline__ u32 rcp_of(u32 f) { return f == 1 ? 0xFFFFFFFFu : (u32)((1ull << 32) / f); }
__device__ __forceinline__ u32 div_by(u32 x, u32 f, u32 rcp, u32* rem) {
  u32 q = __umulhi(x, rcp);
  u32 r = x - q * f;
  if (r >= f) {
    q++;
    r -= f;
  }
  *rem = r;
  return q;
}

// Per-warp rANS model built from a hi-byte histogram.
struct WarpModel {
  u32 hist[256];
  u16 freq[256];
  // per symbol {freq | cum << 16, rcp_of(freq)}: one 64-bit load per step in the encode loop; entry 256 is a
  // no-op symbol (freq 4096, cum 0) for the padding positions past a chunk's end: it never emits and
  // x + q * (4096 - 4096) + 0 leaves the state unchanged
  uint2 fr[257];
};

// fills freq, cum, rcp; returns nsym.
__device__ __forceinline__ u32 warp_normalize(WarpModel& m, u32 n) {
  const u32 lane = lane_id();
  u32 f[8], c[8];
  u32 sum = 0, nsym = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    u32 s = lane * 8 + k;
    c[k] = m.hist[s];
    u32 v = 0;
    if (c[k]) {
      v = (c[k] * kM) / n;  // c <= 16384: fits 32 bits
      if (v < 1) v = 1;
      nsym++;
    }
    f[k] = v;
    sum += v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    nsym += __shfl_xor_sync(0xffffffffu, nsym, o);
  }
  if (sum < kM) {
    // argmax count, lowest symbol on ties: key = count << 8 | (255 - s)
    u32 best = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      u32 s = lane * 8 + k;
      if (c[k]) {
        u32 key = (c[k] << 8) | (255u - s);
        best = key > best ? key : best;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      u32 t = __shfl_xor_sync(0xffffffffu, best, o);
      best = t > best ? t : best;
    }
    const u32 bs = 255u - (best & 0xFFu);
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] += (lane * 8 + (u32)k == bs) ? kM - sum : 0u;   // registers, no local
    sum = kM;
  }
  while (sum > kM) {
    u32 best = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      u32 s = lane * 8 + k;
      if (f[k] > 1) {
        u32 key = (f[k] << 8) | (255u - s);
        best = key > best ? key : best;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      u32 t = __shfl_xor_sync(0xffffffffu, best, o);
      best = t > best ? t : best;
    }
    const u32 bs = 255u - (best & 0xFFu);
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] -= (lane * 8 + (u32)k == bs) ? 1u : 0u;
    sum -= 1;
  }
  // exclusive prefix over symbols (lane-major, 8 per lane)
  u32 local = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) local += f[k];
  u32 incl = warp_incl_scan(local);
  u32 run = incl - local;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    u32 s = lane * 8 + k;
    m.freq[s] = (u16)f[k];
    m.fr[s] = make_uint2(f[k] | (run << 16), f[k] ? rcp_of(f[k]) : 0u);
    run += f[k];
  }
  if (lane == 0) m.fr[256] = make_uint2((u32)kM, rcp_of((u32)kM));
  __syncwarp();
  return nsym;
}

// Device-side launch counter (diagnostics, sync_launch_count).
}  // namespace ss
