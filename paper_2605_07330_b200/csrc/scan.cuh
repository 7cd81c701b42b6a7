// scan.cuh — grid-wide exclusive scans for the plan kernels (K2, K4 planning).
//
// One item per thread, kGScan threads per CTA, up to three u64 lanes per item. A CTA takes its rank j from a
// ticket (so every CTA it waits for has already started: forward progress without co-residency, as in K1),
// scans its items in shared memory, publishes its three totals with the call's epoch as the flag, and adds
// the totals of CTAs 0..j-1 (every one read directly — aggregates only, no chain of inclusive prefixes, so
// the wait is one round of loads once they have published). Tickets count up forever: a kernel with a fixed
// grid G uses ticket mod G, and every launch consumes exactly G tickets. The state words are never reset:
// a CTA publishes (values, epoch) and a reader accepts only the current epoch. The epoch lives in device
// memory (one counter per scan): every CTA reads it at its start, and the last CTA advances it once it has
// seen every other CTA's totals (so all of them have read the old value) — no host bookkeeping, so a plan
// captured in a CUDA graph stays correct on every replay.
#pragma once
#include "common.cuh"

namespace ss {

constexpr int kGScan = 1024;

struct GScanState {     // one per CTA of one scan: 3 totals + the epoch flag (32 B)
  u64 v[3];
  u64 epoch;
};

// Block-wide exclusive scan of three u64 lanes (kGScan threads); returns the block totals in tot[].
__device__ __forceinline__ void block_scan3(const u64 (&v)[3], u64 (&ex)[3], u64 (&tot)[3], u64* s_w /*[3][33]*/) {
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u64 inc[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    inc[k] = warp_incl_scan64(v[k]);
    if (lane == 31) s_w[k * 33 + warp] = inc[k];
  }
  __syncthreads();
  if (warp < 3) {
    const u64 w = s_w[warp * 33 + lane];
    const u64 wi = warp_incl_scan64(w);
    s_w[warp * 33 + lane] = wi - w;
    if (lane == 31) s_w[warp * 33 + 32] = wi;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    ex[k] = s_w[k * 33 + warp] + inc[k] - v[k];
    tot[k] = s_w[k * 33 + 32];
  }
  __syncthreads();
}

// This launch's epoch (block-uniform): the counter's value + 1 (a zeroed workspace starts at epoch 1).
__device__ __forceinline__ u64 gscan_epoch(const u32* ctr, u64* s_e) {
  if (threadIdx.x == 0) *s_e = (u64)*(volatile const u32*)ctr + 1;
  __syncthreads();
  return *s_e;
}
// The last CTA, after gscan_publish_and_prefix: advance the counter to this launch's epoch.
__device__ __forceinline__ void gscan_advance(u32* ctr, u64 epoch) {
  if (threadIdx.x == 0) *(volatile u32*)ctr = (u32)epoch;
}

// This CTA's rank in ticket order (block-uniform).
__device__ __forceinline__ u32 gscan_rank(u32* ticket, u32 grid, u32* s_j) {
  if (threadIdx.x == 0) *s_j = atomicAdd(ticket, 1u) % grid;
  __syncthreads();
  return *s_j;
}

// Publish this CTA's totals, then return the sum of the totals of CTAs 0..j-1 (all threads).
__device__ __forceinline__ void gscan_publish_and_prefix(GScanState* st, u32 j, u64 epoch, const u64 (&tot)[3],
                                                         u64 (&pre)[3], u64* s_r /*[3][33]*/) {
  if (threadIdx.x == 0) {
    GScanState* me = st + j;
    me->v[0] = tot[0];
    me->v[1] = tot[1];
    me->v[2] = tot[2];
    __threadfence();
    cuda::atomic_ref<u64, cuda::thread_scope_device>(me->epoch).store(epoch, cuda::std::memory_order_release);
  }
  u64 acc[3] = {0, 0, 0};
  for (u32 i = threadIdx.x; i < j; i += blockDim.x) {
    cuda::atomic_ref<u64, cuda::thread_scope_device> f(st[i].epoch);
    while (f.load(cuda::std::memory_order_acquire) != epoch) __nanosleep(64);
    acc[0] += st[i].v[0];
    acc[1] += st[i].v[1];
    acc[2] += st[i].v[2];
  }
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    acc[k] = warp_sum64(acc[k]);
    if (lane == 0) s_r[k * 33 + warp] = acc[k];
  }
  __syncthreads();
  if (warp < 3) {
    u64 x = lane < blockDim.x / 32 ? s_r[warp * 33 + lane] : 0;
    x = warp_sum64(x);
    if (lane == 0) s_r[warp * 33 + 32] = x;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 3; ++k) pre[k] = s_r[k * 33 + 32];
  __syncthreads();
}

}  // namespace ss
