// bucket.cu — K4 planning on the device: the greedy bucket plan of DESIGN C11 (row a5).
//
// Buckets are filled greedily in record (manifest) order: a record never splits, a bucket closes when the
// next record would push it past L (header and record directory included), and a record larger than L sits
// alone. From the record table of k_plan_sizes (rec_list, srec = byte prefix, crec = chunk prefix):
//  * k_bucket_next (grid)   nxt[i] = one past the last record of a bucket that starts at record i:
//                           the largest j with 32 + pad16(8 (j - i)) + srec[j] - srec[i] <= L (at least
//                           i + 1). The size is increasing in j, so a binary search finds it.
//  * k_bucket_plan (1 CTA)  walks the chain 0 -> nxt[0] -> ... (one step per bucket; nxt staged in shared
//                           memory first when many buckets are expected), then in parallel: bucket sizes,
//                           256-aligned bases, CRC segment offsets; capacity checks (bytes, bucket count)
//                           latch SYNC_ERR_CAPACITY and leave nothing to encode. The bucket count, offsets
//                           and sizes go to the context's mapped pinned table (no copy, no host sync).
//  * k_bucket_records (grid) per record: its bucket (binary search over the starts), destination and
//                           directory entry.
// The host never sees a record size: sync_compress_pack is enqueue-only up to reading the final table.
#include "common.cuh"
#include "kernels.h"

namespace ss {

constexpr int kBThreads = 1024;

__global__ void __launch_bounds__(256) k_bucket_next(BucketPlan b) {
  const u64 R = b.totals[kTotRecords];
  if (b.totals[kTotOverflow]) return;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < R; i += (u64)gridDim.x * blockDim.x) {
    const u64 s0 = b.srec[i];
    u64 lo = i + 1, hi = R;   // answer in [lo, hi]; lo always allowed
    while (lo < hi) {
      const u64 mid = (lo + hi + 1) / 2;
      const u64 size = 32 + pad_to(8 * (mid - i), 16) + (b.srec[mid] - s0);
      if (size <= b.limit) lo = mid;
      else hi = mid - 1;
    }
    b.nxt[i] = (u32)lo;
  }
}

// Block-wide exclusive scan of a u64 (kBThreads threads); returns the block total.
__device__ __forceinline__ u64 bscan64(u64 v, u64* excl, u64* s_w) {
  const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u64 inc = warp_incl_scan64(v);
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const u64 w = s_w[lane];
    const u64 wi = warp_incl_scan64(w);
    s_w[lane] = wi - w;
    if (lane == 31) s_w[32] = wi;
  }
  __syncthreads();
  *excl = s_w[warp] + inc - v;
  const u64 total = s_w[32];
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(kBThreads) k_bucket_plan(BucketPlan b, u32 smem_nxt) {
  extern __shared__ u32 s_nxt[];
  __shared__ u64 s_w[33];
  __shared__ u32 s_nb;
  __shared__ u32 s_fail;
  __shared__ u64 s_need;
  const u32 tid = threadIdx.x;
  const u64 R = b.totals[kTotRecords];
  const bool over = b.totals[kTotOverflow] != 0;
  if (tid == 0) {
    s_fail = over ? 1u : 0u;
    s_need = 0;
  }
  // stage nxt in shared memory only when the walk is long (expected buckets = payload / L): a short walk
  // reads the few entries it needs from L2 directly
  const u64 est = R ? b.srec[R] / (b.limit ? b.limit : 1) + 1 : 0;
  const bool in_smem = !over && est > 64 && R <= smem_nxt;
  if (in_smem) {
#pragma unroll 8
    for (u64 i = tid; i < R; i += kBThreads) s_nxt[i] = b.nxt[i];
  }
  __syncthreads();
  // ---- 1. bucket starts: one step per bucket along the greedy chain
  if (tid == 0) {
    u32 nb = 0;
    if (!over) {
      u64 i = 0;
      while (i < R) {
        b.bstart[nb++] = (u32)i;
        i = in_smem ? s_nxt[i] : b.nxt[i];
      }
    }
    b.bstart[nb] = (u32)R;
    s_nb = nb;
    if (nb > b.max_buckets) s_fail = 1;
  }
  __syncthreads();
  const u32 nb = s_nb;
  // ---- 2. bucket sizes, bases (each padded to kBucketAlign), CRC segments; rounds of kBThreads buckets
  u64 base_carry = 0, seg_carry = 0;
  for (u32 r0 = 0; r0 < nb; r0 += kBThreads) {
    const u32 k = r0 + tid;
    u64 bytes = 0, segs = 0;
    u32 s = 0, e = 0;
    if (k < nb) {
      s = b.bstart[k];
      e = b.bstart[k + 1];
      bytes = 32 + pad_to(8ull * (e - s), 16) + (b.srec[e] - b.srec[s]);
      segs = (bytes - 32 + kCrcSegBytes - 1) / kCrcSegBytes;
    }
    u64 bex, sex;
    const u64 btot = bscan64(pad_to(bytes, kBucketAlign), &bex, s_w);
    const u64 stot = bscan64(segs, &sex, s_w);
    if (k < nb) {
      BucketDesc d;
      d.base = base_carry + bex;
      d.bytes = bytes;
      d.n_records = e - s;
      d.n_chunks = (u32)(b.crec[e] - b.crec[s]);
      d.first_record = s;
      d.seq = k;
      b.bks[k] = d;
      b.seg_off[k] = seg_carry + sex;
      if (k + 1 == nb) s_need = d.base + bytes;
      b.out_off[k] = d.base;   // the context's mapped table holds T + 1 entries (nb <= records <= T)
      b.out_size[k] = bytes;
    }
    base_carry += btot;
    seg_carry += stot;
  }
  __syncthreads();
  const u64 need = s_need;
  if (tid == 0) {
    b.seg_off[nb] = seg_carry;
    if (need > b.cap_bytes) s_fail = 1;
  }
  __syncthreads();
  const bool fail = s_fail != 0;
  if (tid == 0) {
    b.out_hdr[0] = fail ? 0 : nb;
    b.out_hdr[1] = fail ? 1 : 0;
    b.out_hdr[2] = need;
    b.totals[kTotBuckets] = fail ? 0 : nb;
    b.totals[kTotBucketBytes] = need;
    b.totals[kTotSegs] = fail ? 0 : seg_carry;
    if (fail) {
      if (!over) latch(b.status, SYNC_ERR_CAPACITY);
      b.totals[kTotOverflow] = 1;
      b.totals[kTotChunks] = 0;   // nothing gets encoded, packed or CRC'd
    }
    __threadfence_system();
  }
}

// per record: its bucket (the last start <= k), destination, directory entry
__global__ void __launch_bounds__(256) k_bucket_records(BucketPlan b) {
  const u64 R = b.totals[kTotRecords];
  if (b.totals[kTotOverflow]) return;
  const u32 nb = (u32)b.totals[kTotBuckets];
  for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < R; k += (u64)gridDim.x * blockDim.x) {
    u32 lo = 0, hi = nb - 1;
    while (lo < hi) {
      const u32 mid = (lo + hi + 1) / 2;
      if (b.bstart[mid] <= k) lo = mid;
      else hi = mid - 1;
    }
    const BucketDesc d = b.bks[lo];
    const u64 s = d.first_record;
    const u64 rec0 = 32 + pad_to(8ull * d.n_records, 16);
    const u32 t = b.rec_list[k];
    RecordDesc r;
    r.src = b.enc_off[t];
    r.bytes = (u32)(b.srec[k + 1] - b.srec[k]);
    r.dir_offset = (u32)(rec0 + b.srec[k] - b.srec[s]);
    r.dst = d.base + r.dir_offset;
    r.first_chunk = (u32)(b.crec[k] - b.crec[s]);
    r.tensor = t;
    b.recs[k] = r;
    if (b.rec_dst) b.rec_dst[t] = r.dst;
  }
}

void launch_bucket_plan(const BucketPlan& b, u32 n_tensors, int sm_count, cudaStream_t s) {
  // nxt for up to T records: grid-stride, one thread per record
  const u32 T = n_tensors ? n_tensors : 1;
  u32 g = (T + 255) / 256;
  const u32 gmax = (u32)(sm_count * 8);
  k_bucket_next<<<g < gmax ? g : gmax, 256, 0, s>>>(b);
  count_launch();
  // nxt staged in shared memory when it fits (<= 200 KB: 51,200 records; the 235B manifest has 36,945)
  constexpr u32 kSmemNxt = 51200;
  const u32 n_sm = T <= kSmemNxt ? T : 0;
  static bool attr[kMaxDevices] = {};
  const int dev = current_device();
  if (!attr[dev]) {
    cudaFuncSetAttribute(k_bucket_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(4 * kSmemNxt));
    attr[dev] = true;
  }
  k_bucket_plan<<<1, kBThreads, 4 * (size_t)n_sm, s>>>(b, n_sm);
  count_launch();
  k_bucket_records<<<g < gmax ? g : gmax, 256, 0, s>>>(b);
  count_launch();
}

}  // namespace ss
