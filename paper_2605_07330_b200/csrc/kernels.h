// kernels.h — host-side launchers of the sm_100a kernels (internal to libsparsesync).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sparsesync.h"

namespace ss {

void count_launch();
// Launch sizing (api.cu). Per-device caches are indexed by the current device (< kMaxDevices).
constexpr int kMaxDevices = 64;
int current_device();
// grid of a persistent / grid-stride kernel after the process-wide sync_set_max_ctas() limit
int clamp_ctas(int grid);

// Device views of the workspace (all arrays live in the caller's workspace).
struct Plan {
  uint32_t n_tensors;
  uint64_t cap;                  // I/V capacity
  uint32_t codec;
  uint64_t max_chunks;
  uint64_t enc_cap;              // capacity of the caller's enc buffer (bytes)
  const uint64_t* numel;         // [T]
  uint64_t* rec_off;             // [T+1] value offset of tensor t in I/V
  uint64_t* chunk_off;           // [T+1] first global chunk of tensor t
  uint32_t* maxgap;              // [T]
  uint32_t* rec_mode;            // [T] DELTA16 / ABS32 / FULL
  uint64_t* rec_bytes;           // [T]
  uint64_t* enc_off;             // [T+1]
  const uint64_t* rec_dst;       // [T] where k_encode writes record t (enc_off, or bucket positions)
  uint32_t* chunk_hi;            // [max_chunks] hi block bytes (unpadded)
  uint32_t* chunk_mode;          // [max_chunks]
  uint64_t* chunk_hioff;         // [max_chunks+1] exclusive prefix of pad4(chunk_hi)
  uint32_t* chunk_rhdr;          // [max_chunks][kRhdrWords] rANS block head from the stats pass
  uint16_t* word_scratch;        // renormalisation words in emission order (see chunk_words_base)
  uint64_t* totals;              // [16]
  uint32_t* status;
  int prof;                      // debug instrumentation switch
  int route;                     // f3: SYNC_FLAG_ROUTE
  uint32_t dtype;                // record dtype tag (SYNC_DTYPE_*)
  int escape;                    // f4: SYNC_FLAG_ESCAPE
  uint32_t* chunk_esc;           // [max_chunks] index gaps > 32767 in the chunk (f4)
  uint32_t* chunk_t;             // [max_chunks] tensor of each chunk (k_chunk_stats -> k_encode)
  uint64_t* chunk_escoff;        // [max_chunks+1] exclusive prefix of chunk_esc
  const uint16_t* const* cur;    // f3: current weights (FULL records), device pointer table
  uint32_t* rec_list;            // [T] tensor of record k (records = tensors with a change, manifest order)
  uint64_t* srec;                // [T+1] exclusive prefix of the record bytes over records
  uint64_t* crec;                // [T+1] exclusive prefix of the on-wire chunk counts over records
  uint64_t* work;                // [2] chunk claim counters (k_chunk_stats, k_encode), zeroed by k_plan_scan
  uint32_t* tickets;             // [3] CTA tickets of the grid scans (scan.cuh); never reset
  uint64_t* gscan;               // GScanState [gscan_T + gscan_C + gscan_T]: plan_scan, plan_chunks, plan_records
  uint32_t gscan_T;              // CTAs of the per-tensor scans = ceil(T / 1024)
  uint32_t gscan_C;              // CTAs of the per-chunk scan = ceil(max_chunks / 1024)
  uint32_t* epochs;              // [3] device epoch counters of the three grid scans (scan.cuh)
};

enum TotalsIdx {
  kTotNnz = 0, kTotChunks = 1, kTotRecords = 2, kTotEnc = 3, kTotDelta16 = 4, kTotAbs32 = 5,
  kTotRansChunks = 6, kTotOverflow = 7, kTotIndexBytes = 8, kTotValueBytes = 9, kTotFull = 10,
  kTotDelta16E = 11, kTotBuckets = 12, kTotBucketBytes = 13, kTotSegs = 14
};
constexpr uint32_t kModeFull = 2;     // record idx_mode of a FULL record (f3)
constexpr uint32_t kModeDelta16E = 3;  // record idx_mode of an escape-coded DELTA16 record (f4)

void launch_extract_batched(const uint16_t* const* d_old, const uint16_t* const* d_new, const uint64_t* tile_prefix,
                            const uint32_t* tile_tensor, const uint64_t* numel, uint32_t n_tensors, uint64_t n_tiles,
                            uint32_t* I, uint16_t* V, uint64_t cap, uint64_t* counts, uint64_t* tile_state,
                            uint32_t* ticket, uint32_t* stage_ring, uint32_t* status, cudaStream_t s,
                            int elem_bytes = 2);   // 1: FP8
// ticket: a zeroed device u32 (the tile claim counter)
void launch_extract_single(const uint16_t* d_old, const uint16_t* d_new, uint64_t n, uint32_t* I, uint16_t* V,
                           uint64_t cap, uint64_t* count, uint64_t* tile_state, uint32_t* ticket,
                           uint32_t* stage_ring, uint32_t* status, cudaStream_t s);

// plan.cu
void launch_plan_scan(const Plan& p, const uint64_t* counts, cudaStream_t s);
void launch_chunk_stats(const Plan& p, const uint32_t* I, const uint16_t* V, const uint64_t* counts, int grid,
                        cudaStream_t s);
void launch_plan_sizes(const Plan& p, const uint64_t* counts, cudaStream_t s);

// encode.cu
void launch_encode(const Plan& p, const uint32_t* I, const uint16_t* V, const uint64_t* counts, uint8_t* enc,
                   int grid, cudaStream_t s);

// pack.cu
struct BucketDesc {              // one bucket of the device plan (bucket.cu)
  uint64_t base;                 // byte offset of the bucket in the caller's buffer
  uint64_t bytes;
  uint32_t n_records;
  uint32_t n_chunks;
  uint32_t first_record;         // index into the record table
  uint32_t seq;
};
struct RecordDesc {              // one per record, manifest order
  uint64_t src;                  // offset in enc
  uint64_t dst;                  // offset in the bucket buffer
  uint32_t bytes;
  uint32_t dir_offset;           // record offset from its bucket start
  uint32_t first_chunk;          // within its bucket
  uint32_t tensor;
};
// bucket.cu: the greedy bucket plan on the device (DESIGN C11)
struct BucketPlan {
  const uint32_t* rec_list;      // Plan::rec_list / srec / crec (from k_plan_sizes)
  const uint64_t* srec;
  const uint64_t* crec;
  const uint64_t* enc_off;       // [T] record t's offset in the contiguous encoded stream (unfused path)
  uint32_t* nxt;                 // [T] scratch
  uint32_t* bstart;              // [T+1] first record of each bucket (+ sentinel)
  uint64_t* seg_off;             // [T+1] first CRC segment of each bucket
  RecordDesc* recs;              // [T]
  BucketDesc* bks;               // [T]
  uint64_t* rec_dst;             // [T] where k_encode writes record t (fused path), or null
  uint64_t* totals;
  uint32_t* status;
  uint64_t limit;                // L
  uint64_t cap_bytes;            // the caller's bucket buffer
  uint32_t max_buckets;          // the caller's table
  uint64_t* out_hdr;             // mapped pinned host: {n_buckets, failed, need}
  uint64_t* out_off;             // mapped pinned host: [T+1] bucket offsets
  uint64_t* out_size;            // mapped pinned host: [T+1] bucket sizes
};
void launch_bucket_plan(const BucketPlan& b, uint32_t n_tensors, int sm_count, cudaStream_t s);

// bucket headers + directories for the device plan (counts read from totals); enc != null: also copy the
// contiguous encoded stream into the bucket positions (unfused path)
void launch_pack(const uint8_t* enc, uint8_t* buckets, const RecordDesc* recs, const BucketDesc* bks,
                 const uint64_t* totals, uint32_t max_buckets, uint32_t flags, int grid, cudaStream_t s);
void crc_fill(uint8_t* buckets, const BucketDesc* bks, const uint64_t* seg_off, const uint64_t* totals,
              uint32_t max_buckets, uint32_t* scratch, int grid, cudaStream_t s);

// decode.cu
// CRC-32 of one bucket vs its header: mismatch latches SYNC_ERR_CRC and sets *bad_flag (device u32).
void launch_crc_check(const uint8_t* bucket, uint64_t bytes, uint32_t* seg_scratch, uint32_t* bad_flag,
                      uint32_t* status, cudaStream_t s);
void launch_unpack(const uint8_t* bucket, uint64_t bytes, uint32_t n_tensors, const uint64_t* numel,
                   sync_record_view* views, uint32_t max_views, uint32_t* n_records, uint32_t* status,
                   uint32_t dtype, cudaStream_t s);
// buckets / bytes: HOST arrays of n_buckets device addresses and sizes; crc_bad: device flags [n_buckets]
// (or null). One kernel per 32 buckets.
void launch_decode(const uint8_t* const* buckets, const uint64_t* bytes, uint32_t n_buckets, uint32_t n_tensors,
                   const uint64_t* numel, uint16_t* const* weights, const sync_record_view* views, uint32_t* I_out,
                   uint16_t* V_out, uint64_t out_cap, uint32_t* status, const uint32_t* crc_bad, uint32_t dtype,
                   int grid, bool dense, cudaStream_t s);
// the same, from a device bucket table (a sender context's plan: t_hdr[0] buckets, offsets / sizes every
// `stride` u64 words);
// ceil(max_buckets / 32) launches, each decoding its slice of the table (no host knowledge of the count)
void launch_decode_table(const uint64_t* t_hdr, const uint64_t* t_off, const uint64_t* t_size, uint32_t stride,
                         const uint8_t* base, uint32_t max_buckets, uint32_t n_tensors, const uint64_t* numel, uint16_t* const* weights,
                         uint32_t* status, uint32_t dtype, int grid, bool dense, cudaStream_t s);
// a decode call is "dense" when its buckets carry >= 0.1 byte per model element (rho >~ 3%)
inline bool decode_is_dense(const uint64_t* bytes, uint32_t n, uint64_t model_elems) {
  uint64_t t = 0;
  for (uint32_t i = 0; i < n; ++i) t += bytes[i];
  return t * 10 >= model_elems && t > 0;
}

// track.cu (f1 cast-fused tracking, Alg. 1)
struct TrackArgs {
  uint64_t n_tiles;
  uint32_t n_tensors;
  const uint32_t* tile_tensor;   // [n_tiles]
  const uint64_t* tile_prefix;   // [T+1]
  const uint64_t* numel;         // [T]
  const uint64_t* bm_off;        // [T+1] bitmap word offset of each tensor
  uint32_t* bitmap;
  uint64_t* tile_off;            // [n_tiles] tile counts -> offsets within their group
  uint64_t* group_sum;           // [n_groups+1]
  uint64_t* counts;              // [T]
  uint32_t* I;
  uint16_t* V;
  uint64_t cap;
  uint64_t* totals;
  uint32_t* status;
};
void launch_cast_track(const TrackArgs& a, const float* const* master, uint16_t* const* W, int grid, cudaStream_t s);
void launch_extract_tracked(const TrackArgs& a, uint16_t* const* W, int clear, int grid, cudaStream_t s,
                            bool k8 = false);
// FP8 (8-bit elements): bitwise diff into the bitmap, then the tracked compaction (V = new[I] bytes)
void launch_extract8(const TrackArgs& a, const uint8_t* const* olds, const uint8_t* const* news, int grid,
                     cudaStream_t s);

// apply.cu
void launch_apply(uint16_t* W, const uint32_t* I, const uint16_t* V, uint64_t count, uint64_t numel,
                  uint32_t* status, cudaStream_t s);
void launch_commit_batched(const Plan& p, uint16_t* const* snaps, const uint32_t* I, const uint16_t* V, int grid,
                           cudaStream_t s);

}  // namespace ss
