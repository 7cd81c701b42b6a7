// pack.cu — K4: bucket assembly (row a5) and CRC-32 (C11, C14).
//
// The greedy bucket plan comes from the device planner (bucket.cu); every
// kernel here reads the bucket and record tables from device memory, so the
// whole sender is enqueued without a host round trip. They write every byte
// of the buckets:
//  * k_pack_meta : header (32 B) + record directory + directory padding
//  * k_pack_copy : records, 16 B units, enc -> bucket position (unfused path)
//  * k_crc_seg / k_crc_fin : parallel CRC-32/IEEE of [32, bytes) — slicing-by-4
//    CRCs of 128-byte pieces, combined per 64 KB segment and then across segments
//    with multiplications by x^(8n) mod P (the CRC is linear over GF(2)), then
//    the init/xorout terms. The sender fills every bucket's CRC in two launches
//    (segments of all buckets, then one CTA per bucket); the receiver checks one
//    bucket at a time.
// multmodp / x8n: GF(2) polynomial multiplication modulo P and x^(8n) mod P by
// squaring, the same construction as zlib's crc32.c (multmodp, x2nmodp), here
// with a fixed 32-step loop.
#include "common.cuh"
#include "kernels.h"

namespace ss {

constexpr u32 kPoly = 0xEDB88320u;  // reflected IEEE polynomial
constexpr int kCrcThreads = 512;    // one CTA per segment
constexpr u32 kCrcPiece = 128;      // bytes per thread (8 x 16-byte loads)
constexpr u32 kCrcSeg = kCrcThreads * kCrcPiece;   // 64 KB per segment
static_assert(kCrcSeg == kCrcSegBytes, "bucket.cu plans CRC segments of kCrcSegBytes");

struct CrcTables {
  u32 x2n[32];  // x^(2^k) mod P, reflected
};

// a * b mod P in the reflected representation (bit 31 = x^0); fixed 32 steps.
__host__ __device__ __forceinline__ u32 multmodp(u32 a, u32 b) {
  u32 r = 0;
  for (int i = 0; i < 32; ++i) {
    if (a & (0x80000000u >> i)) r ^= b;
    b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
  }
  return r;
}

// x^(8n) mod P
__host__ __device__ __forceinline__ u32 x8n(const CrcTables& tb, u64 n) {
  u32 r = 1u << 31;
  int k = 3;
  while (n) {
    if (n & 1) r = multmodp(tb.x2n[k & 31], r);
    n >>= 1;
    ++k;
  }
  return r;
}

// x^(8 * kCrcPiece * (kCrcThreads - 1 - t)): shifts piece t's CRC to the end of its segment
__constant__ u32 c_piece_shift[kCrcThreads];

// The bytes [0, len) are viewed as a virtual stream of S * kCrcSeg bytes with pad = S*kCrcSeg - len
// leading zero bytes (leading zeros leave an init-0 CRC unchanged). len is a multiple of 16, so every
// 128-byte piece of the virtual stream starts 16-byte aligned in memory. Thread t of CTA s computes the
// raw CRC (init 0, no xorout) of its piece with slicing-by-4 tables and shifts it to the segment end;
// the XOR of the shifted pieces is the segment's raw CRC (the CRC is linear over GF(2)).
__device__ __forceinline__ void crc_tables(u32 (*T)[256]) {
  for (u32 i = threadIdx.x; i < 256; i += blockDim.x) {
    u32 c = i;
    for (int k = 0; k < 8; ++k) c = (c >> 1) ^ (kPoly & (0u - (c & 1u)));
    T[0][i] = c;
  }
  __syncthreads();
  for (u32 i = threadIdx.x; i < 256; i += blockDim.x) {
    u32 c = T[0][i];
    for (int k = 1; k < 4; ++k) {
      c = (c >> 8) ^ T[0][c & 0xFFu];
      T[k][i] = c;
    }
  }
  __syncthreads();
}

// raw CRC of segment `seg` of the virtual stream (data, len, pad) -> *seg_crc (whole CTA)
__device__ __forceinline__ void crc_segment(const u32 (*T)[256], u32* s_x, const u8* data, u64 pad, u64 seg,
                                            u32* seg_crc) {
  const long long v0 = (long long)seg * kCrcSeg + (long long)threadIdx.x * kCrcPiece - (long long)pad;
  uint4 w[kCrcPiece / 16];
#pragma unroll
  for (int j = 0; j < (int)(kCrcPiece / 16); ++j) {
    const long long o = v0 + 16 * j;
    w[j] = o >= 0 ? *reinterpret_cast<const uint4*>(data + o) : make_uint4(0, 0, 0, 0);
  }
  u32 c = 0;
#pragma unroll
  for (int j = 0; j < (int)(kCrcPiece / 16); ++j) {
    const u32 ws[4] = {w[j].x, w[j].y, w[j].z, w[j].w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      c ^= ws[k];
      c = T[3][c & 0xFFu] ^ T[2][(c >> 8) & 0xFFu] ^ T[1][(c >> 16) & 0xFFu] ^ T[0][c >> 24];
    }
  }
  c = multmodp(c, c_piece_shift[threadIdx.x]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c ^= __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) s_x[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x < 32) {
    c = threadIdx.x < kCrcThreads / 32 ? s_x[threadIdx.x] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c ^= __shfl_xor_sync(0xffffffffu, c, o);
    if (threadIdx.x == 0) *seg_crc = c;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kCrcThreads) k_crc_seg(const u8* data, u64 len, u64 pad, u32* seg_crc) {
  __shared__ u32 T[4][256];
  __shared__ u32 s_x[kCrcThreads / 32];
  crc_tables(T);
  crc_segment(T, s_x, data, pad, blockIdx.x, seg_crc + blockIdx.x);
}

// Every bucket of a sender plan: global segment g of bucket b (seg_off[b] <= g < seg_off[b + 1]) covers the
// bucket's bytes [32, bytes) like k_crc_seg does for one bucket. Grid-stride over the segments.
__global__ void __launch_bounds__(kCrcThreads) k_crc_seg_all(const u8* buckets, const BucketDesc* bks,
                                                             const u64* seg_off, const u64* totals, u32* seg_crc) {
  __shared__ u32 T[4][256];
  __shared__ u32 s_x[kCrcThreads / 32];
  crc_tables(T);
  const u32 nb = (u32)totals[kTotBuckets];
  const u64 n_seg = totals[kTotSegs];
  for (u64 g = blockIdx.x; g < n_seg; g += gridDim.x) {
    u32 lo = 0, hi = nb - 1;
    while (lo < hi) {
      const u32 mid = (lo + hi + 1) / 2;
      if (seg_off[mid] <= g) lo = mid;
      else hi = mid - 1;
    }
    const BucketDesc d = bks[lo];
    const u64 len = d.bytes - 32;
    const u64 S = seg_off[lo + 1] - seg_off[lo];
    crc_segment(T, s_x, buckets + d.base + 32, S * kCrcSeg - len, g - seg_off[lo], seg_crc + g);
  }
}

// Combine the S segment CRCs (thread j: Horner over its block of consecutive segments, then one shift to
// the stream end, XOR-reduced), apply the init / xorout terms of CRC-32/IEEE over the real len bytes, and
// store into *out (or compare with the header's value).
// Combine the S segment CRCs (thread j: Horner over its block of consecutive segments, then one shift to
// the stream end, XOR-reduced), apply the init / xorout terms of CRC-32/IEEE over the real len bytes, and
// store into *out (or compare with the header's value). Whole CTA of 1024 threads.
__device__ __forceinline__ void crc_finish(u32* s_x, const u32* seg_crc, u64 S, u64 len, const CrcTables& tb,
                                           u32* out, const u8* hdr_crc, u32* status, u32* bad) {
  const u64 B = (S + blockDim.x - 1) / blockDim.x;
  const u64 s0 = (u64)threadIdx.x * B, s1 = s0 + B < S ? s0 + B : S;
  u32 acc = 0;
  if (s0 < S) {
    const u32 shift = x8n(tb, kCrcSeg);
    for (u64 s = s0; s < s1; ++s) acc = multmodp(acc, shift) ^ seg_crc[s];
    acc = multmodp(acc, x8n(tb, (u64)kCrcSeg * (S - s1)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s_x[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < blockDim.x / 32 ? s_x[threadIdx.x] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) {
      const u32 crc = acc ^ multmodp(0xFFFFFFFFu, x8n(tb, len)) ^ 0xFFFFFFFFu;
      if (out) *out = crc;
      if (hdr_crc) {
        u32 want = (u32)hdr_crc[0] | ((u32)hdr_crc[1] << 8) | ((u32)hdr_crc[2] << 16) | ((u32)hdr_crc[3] << 24);
        if (want != crc) {
          latch(status, SYNC_ERR_CRC);
          if (bad) *bad = 1;
        }
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(1024) k_crc_fin(const u32* seg_crc, u64 S, u64 len, CrcTables tb, u32* out,
                                                  const u8* hdr_crc, u32* status, u32* bad) {
  __shared__ u32 s_x[32];
  crc_finish(s_x, seg_crc, S, len, tb, out, hdr_crc, status, bad);
}

// one CTA per bucket (grid-stride): the bucket's CRC into its header
__global__ void __launch_bounds__(1024) k_crc_fin_all(u8* buckets, const BucketDesc* bks, const u64* seg_off,
                                                      const u64* totals, const u32* seg_crc, CrcTables tb) {
  __shared__ u32 s_x[32];
  const u32 nb = (u32)totals[kTotBuckets];
  for (u32 b = blockIdx.x; b < nb; b += gridDim.x) {
    const BucketDesc d = bks[b];
    crc_finish(s_x, seg_crc + seg_off[b], seg_off[b + 1] - seg_off[b], d.bytes - 32, tb,
               reinterpret_cast<u32*>(buckets + d.base + 20), nullptr, nullptr, nullptr);
  }
}

static CrcTables host_crc_tables() {
  CrcTables tb;
  u32 p = 1u << 30;  // x^1
  tb.x2n[0] = p;
  for (int k = 1; k < 32; ++k) tb.x2n[k] = p = multmodp(p, p);
  return tb;
}

static const CrcTables& crc_tb() {
  static const CrcTables tb = host_crc_tables();
  return tb;
}

// c_piece_shift is __constant__ memory: per device (context), so uploaded once per device
static void crc_shifts() {
  static bool done[kMaxDevices] = {};
  const int dev = current_device();
  if (done[dev]) return;
  u32 h[kCrcThreads];
  for (int t = 0; t < kCrcThreads; ++t) h[t] = x8n(crc_tb(), (u64)kCrcPiece * (kCrcThreads - 1 - t));
  cudaMemcpyToSymbol(c_piece_shift, h, sizeof(h));
  done[dev] = true;
}

// scratch: >= ceil(len / kCrcSeg) u32
static void crc_bucket(const u8* bucket, u64 bytes, u32* scratch, u32* out, const u8* hdr_crc, u32* status,
                       u32* bad, cudaStream_t s) {
  crc_shifts();
  const u64 len = bytes > 32 ? bytes - 32 : 0;   // bytes is a multiple of 16
  const u64 S = (len + kCrcSeg - 1) / kCrcSeg;
  if (S) {
    k_crc_seg<<<(unsigned)S, kCrcThreads, 0, s>>>(bucket + 32, len, S * kCrcSeg - len, scratch);
    count_launch();
  }
  k_crc_fin<<<1, 1024, 0, s>>>(scratch, S, len, crc_tb(), out, hdr_crc, status, bad);
  count_launch();
}

// grid-stride over the buckets of the device plan
__global__ void k_pack_meta(u8* buckets, const RecordDesc* recs, const BucketDesc* bks, const u64* totals,
                            u32 flags) {
  const u32 nb = (u32)totals[kTotBuckets];
  for (u32 k = blockIdx.x; k < nb; k += gridDim.x) {
    const BucketDesc b = bks[k];
    u8* bk = buckets + b.base;
    if (threadIdx.x == 0) {
      u32* h = reinterpret_cast<u32*>(bk);
      h[0] = kMagic;
      h[1] = kVersion | ((flags & SYNC_FLAG_CRC) << 16);
      h[2] = b.seq;
      h[3] = b.n_records;
      h[4] = b.n_chunks;
      h[5] = 0;  // CRC filled by k_crc_fin_all
      *reinterpret_cast<u64*>(bk + 24) = b.bytes;
    }
    u32* dir = reinterpret_cast<u32*>(bk + 32);
    for (u32 q = threadIdx.x; q < b.n_records; q += blockDim.x) {
      const RecordDesc r = recs[b.first_record + q];
      dir[2 * q] = r.dir_offset;
      dir[2 * q + 1] = r.first_chunk;
    }
    u64 dir_end = 32 + 8ull * b.n_records, dir_pad = 32 + pad_to(8ull * b.n_records, 16);
    for (u64 q = dir_end + threadIdx.x; q < dir_pad; q += blockDim.x) bk[q] = 0;
  }
}

// 16-byte units of enc (totals[kTotEnc] / 16 of them); each warp handles 32 consecutive units.
__global__ void __launch_bounds__(256) k_pack_copy(const uint4* enc, u8* buckets, const RecordDesc* recs,
                                                    const u64* totals) {
  const u32 lane = threadIdx.x & 31;
  const u64 nwarps = (u64)gridDim.x * (blockDim.x >> 5);
  const u32 n_records = totals[kTotBuckets] ? (u32)totals[kTotRecords] : 0u;
  const u64 n_units = n_records ? totals[kTotEnc] / 16 : 0;
  for (u64 w = (u64)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w * 32 < n_units; w += nwarps) {
    const u64 u0 = w * 32;
    const u64 u = u0 + lane;
    u32 r = warp_upper_search(n_records, u0 * 16, [&](u32 i) { return recs[i].src; });
    if (u < n_units) {
      const u64 byte = u * 16;
      while (r + 1 < n_records && recs[r + 1].src <= byte) ++r;
      const RecordDesc& d = recs[r];
      uint4 v = enc[u];
      *reinterpret_cast<uint4*>(buckets + d.dst + (byte - d.src)) = v;
    }
  }
}

void launch_pack(const u8* enc, u8* buckets, const RecordDesc* recs, const BucketDesc* bks, const u64* totals,
                 u32 max_buckets, u32 flags, int grid, cudaStream_t s) {
  const u32 g = max_buckets < (u32)grid ? (max_buckets ? max_buckets : 1u) : (u32)grid;
  k_pack_meta<<<g, 256, 0, s>>>(buckets, recs, bks, totals, flags);
  count_launch();
  if (enc) {   // unfused path: copy the contiguous encoded stream into the bucket positions
    k_pack_copy<<<grid, 256, 0, s>>>(reinterpret_cast<const uint4*>(enc), buckets, recs, totals);
    count_launch();
  }
}

// every bucket's CRC (SYNC_FLAG_CRC): segments of all buckets, then one CTA per bucket. scratch: >=
// totals[kTotSegs] u32 (workspace: the encoded-stream bound / 64 KB + one per tensor)
void crc_fill(u8* buckets, const BucketDesc* bks, const u64* seg_off, const u64* totals, u32 max_buckets,
              u32* scratch, int grid, cudaStream_t s) {
  crc_shifts();
  k_crc_seg_all<<<grid, kCrcThreads, 0, s>>>(buckets, bks, seg_off, totals, scratch);
  count_launch();
  const u32 g = max_buckets < 1024u ? (max_buckets ? max_buckets : 1u) : 1024u;
  k_crc_fin_all<<<g, 1024, 0, s>>>(buckets, bks, seg_off, totals, scratch, crc_tb());
  count_launch();
}

void launch_crc_check(const u8* bucket, u64 bytes, u32* seg_scratch, u32* bad_flag, u32* status, cudaStream_t s) {
  crc_bucket(bucket, bytes, seg_scratch, nullptr, bucket + 20, status, bad_flag, s);
}

}  // namespace ss
