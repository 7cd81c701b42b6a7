/*
 * sparsesync.h — C ABI of the B200-native SparseRL-Sync hot path
 * (arxiv 2605.07330, "§3 Method").
 *
 * Implemented by paper_2605_07330_b200/libsparsesync.so (hand-written sm_100a
 * CUDA). No torch types cross this boundary: pointers are plain host or device
 * pointers, sizes are integers, every function returns an int status
 * (SYNC_OK = 0, negative = error) and nothing throws.
 *
 * Conventions (apply to every call unless stated):
 *  - "d_" pointers are DEVICE pointers owned by the caller; "h_" pointers are
 *    host pointers owned by the caller. The library never allocates device
 *    memory; the caller allocates the workspace whose size the *_workspace_size
 *    calls return, and keeps it alive for the lifetime of the context.
 *  - BF16 values travel as uint16_t raw bit patterns and are never converted,
 *    so NaN payloads and signed zeros survive (C1, C9).
 *  - Weight / snapshot / I / V pointers must be 16-byte aligned
 *    (else SYNC_ERR_ALIGNMENT) — torch allocations are 256-byte aligned.
 *  - Every call is asynchronous on `stream` unless documented as blocking.
 *    Errors detected on the device (index range, capacity, corrupt stream,
 *    CRC) are latched in a device status word and returned by sync_status().
 *  - Indices are tensor-local row-major flat element indices, numel < 2^31
 *    ("Indices are kept in int32 ... fits in 2^31 flattened elements").
 *  - The wire format (records, chunks, buckets) is DESIGN.md §3, version 1.
 */
#ifndef SPARSESYNC_H
#define SPARSESYNC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* sync_stream_t; /* == cudaStream_t; NULL = legacy default stream */

/* ---- status codes -------------------------------------------------------- */
#define SYNC_OK 0
#define SYNC_ERR_ARG -1          /* bad argument (NULL, size out of range) */
#define SYNC_ERR_ALIGNMENT -2    /* device pointer not 16-byte aligned */
#define SYNC_ERR_DTYPE -3        /* unsupported dtype, or a record whose dtype tag differs from the context's */
#define SYNC_ERR_WORKSPACE -4    /* workspace too small */
#define SYNC_ERR_CUDA -5         /* a CUDA runtime call failed */
#define SYNC_ERR_INDEX_RANGE -6  /* an index >= numel (S:327 IndexOutOfRange); no OOB write happened */
#define SYNC_ERR_CAPACITY -7     /* output capacity exceeded; no OOB write happened */
#define SYNC_ERR_CORRUPT -8      /* malformed record / rANS end-state mismatch / unconsumed words */
#define SYNC_ERR_BAD_MAGIC -9    /* bucket magic != "SRLB" */
#define SYNC_ERR_VERSION -10     /* bucket version != 1 */
#define SYNC_ERR_TRUNCATED -11   /* bucket shorter than its header says */
#define SYNC_ERR_CRC -12         /* CRC-32 mismatch */

/* ---- configuration ------------------------------------------------------- */
#define SYNC_CODEC_RAW 0         /* u32 I + u16 V: the paper's measured raw path */
#define SYNC_CODEC_COMPRESSED 1  /* DELTA16/ABS32 indices + byte-plane rANS values (§3.3) */
#define SYNC_FLAG_CRC 1u         /* per-bucket CRC-32/IEEE */
#define SYNC_FLAG_ROUTE 2u       /* f3 per-parameter routing: a record goes FULL (the whole tensor,
                                    idx_mode 2) when that is smaller than its sparse record (DESIGN C19);
                                    needs sync_set_current()                                              */
#define SYNC_FLAG_ESCAPE 4u      /* f4 escape-coded DELTA16: a record with gaps > 32767 keeps
                                    2-byte deltas plus one escape word per large gap (idx_mode 3) instead
                                    of falling back to 4-byte absolute indices, when that is smaller       */
#define SYNC_CHUNK 16384u        /* values per chunk */

/* Ordered tensor list = record order (model iteration order). Host memory. */
typedef struct {
  uint32_t n_tensors;
  const uint64_t* numel;   /* [n_tensors], each < 2^31 (0 allowed) */
} sync_manifest;

typedef struct {
  uint64_t bucket_limit;   /* L: max bytes per bucket incl. header (DESIGN C11); >= 64 */
  uint64_t max_changed;    /* capacity of the caller's I/V arrays (elements) */
  uint32_t codec;          /* SYNC_CODEC_* */
  uint32_t flags;          /* SYNC_FLAG_* */
  uint32_t dtype;          /* SYNC_DTYPE_* of every manifest tensor (0 = BF16) */
} sync_config;

/* Element types (f2). BF16 / FP16 are 16-bit patterns: every step is the same integer work and the
 * record's dtype byte carries the tag; a receiver context only accepts records of its own dtype. */
#define SYNC_DTYPE_BF16 1u
#define SYNC_DTYPE_FP16 2u
/* FP8 E4M3 (8-bit elements): every pointer table / weight argument of an FP8 context points at
 * byte tensors (cast to the uint16_t* parameter types); V arrays still hold one value per u16 slot (the byte
 * in the low half). Records have one value plane. Not supported by sync_extract / sync_apply /
 * sync_commit_snapshot (single-tensor 16-bit calls) nor by the f1 tracking calls (round_BF16).           */
#define SYNC_DTYPE_FP8 3u

/* Per-sync statistics, filled by sync_ctx_stats() (blocking). */
typedef struct {
  uint64_t nnz;            /* Σ changed elements (|I|) */
  uint64_t n_records;      /* tensors with nnz > 0 */
  uint64_t n_delta16;      /* records coded DELTA16 (b_i = 2) */
  uint64_t n_abs32;        /* records coded ABS32 (b_i = 4) */
  uint64_t n_chunks;       /* Σ ceil(nnz_t / SYNC_CHUNK) */
  uint64_t n_chunks_rans;  /* hi chunks stored as rANS (rest RAW) */
  uint64_t enc_bytes;      /* Σ record_bytes (compressed or raw records) */
  uint64_t index_bytes;    /* Σ padded index-stream bytes */
  uint64_t value_bytes;    /* Σ (record_bytes - 16 - index bytes): α numerator (DESIGN C5) */
  uint64_t n_full;         /* records routed FULL (SYNC_FLAG_ROUTE, f3) */
  uint64_t n_delta16e;     /* records coded DELTA16E (SYNC_FLAG_ESCAPE, f4) */
} sync_stats;

/* Record view produced by sync_bucket_unpack (device memory, 32 B). */
typedef struct {
  uint32_t tensor_id;
  uint32_t nnz;
  uint32_t offset;         /* record offset from bucket start */
  uint32_t record_bytes;
  uint32_t first_chunk;    /* chunk index of the record's first chunk within the bucket */
  uint8_t idx_mode, dtype, codec, reserved;
  uint64_t out_offset;     /* Σ nnz of the preceding records in the bucket */
} sync_record_view;

typedef struct sync_ctx sync_ctx;   /* opaque host object */

/* ---- context --------------------------------------------------------------
 * sync_workspace_size: device bytes the context needs (tile look-back states,
 * manifest tables, record/chunk plan, status word).
 * sync_ctx_create: validates the manifest (numel < 2^31) and the dtype (BF16 or FP16),
 * uploads its tables into d_workspace on `stream`, and returns a host object.
 * The same context serves a sender (extract/compress/pack/commit) and a
 * receiver (unpack/decompress/apply) over the same manifest (the
 * receiver needs only the manifest, not the Trainer's layout).            */
int sync_workspace_size(const sync_manifest* m, const sync_config* c, size_t* bytes);
int sync_ctx_create(sync_ctx** out, const sync_manifest* m, const sync_config* c,
                    void* d_workspace, size_t workspace_bytes, sync_stream_t stream);
/* sync_ctx_destroy waits for the device first (enqueued copies may still read the context's pinned host
 * tables), then frees the host object; the workspace stays the caller's.  */
int sync_ctx_destroy(sync_ctx* ctx);

/* ---- a1 extract: Alg. 1 l.6 + Alg. 2 l.5 -------------------
 * Single tensor: I = ascending { i < n : old[i] != new_[i] bitwise },
 * V[k] = new_[I[k]], *d_count = |I| (device u64). n < 2^31. If |I| > cap,
 * only the first cap entries are written, *d_count is still the true count
 * and the status word latches SYNC_ERR_CAPACITY. Needs its own small
 * workspace (look-back tile states).                                       */
int sync_extract_workspace_size(uint64_t n, size_t* bytes);
int sync_extract(const uint16_t* d_old, const uint16_t* d_new, uint64_t n,
                 uint32_t* d_I, uint16_t* d_V, uint64_t cap, uint64_t* d_count,
                 void* d_workspace, size_t workspace_bytes, sync_stream_t stream);
/* Reads and clears the status word of a single-tensor workspace (blocking). */
int sync_extract_status(void* d_workspace, sync_stream_t stream);

/* Whole manifest in one launch: d_old_ptrs/d_new_ptrs are DEVICE arrays of
 * n_tensors device pointers. Records are contiguous in manifest order:
 * tensor t's entries occupy [Σ_{u<t} counts[u], +counts[t]) of I and V, with
 * tensor-local indices. d_counts: device u64[n_tensors]. Capacity =
 * config.max_changed.                                                      */
int sync_extract_batched(sync_ctx* ctx, const uint16_t* const* d_old_ptrs,
                         const uint16_t* const* d_new_ptrs, uint32_t* d_I, uint16_t* d_V,
                         uint64_t* d_counts, sync_stream_t stream);

/* ---- a2-a4 plan + encode: §3.3 --------------------------------
 * From the output of sync_extract_batched, build every record (DESIGN §3.1 or
 * §3.2 per config.codec) back to back into d_enc (capacity enc_cap bytes;
 * sync_enc_bound gives a safe capacity). Per-record sizes stay in the
 * workspace for sync_bucket_pack. Deterministic bytes.                     */
int sync_enc_bound(const sync_manifest* m, const sync_config* c, uint64_t* bytes);
int sync_compress(sync_ctx* ctx, const uint32_t* d_I, const uint16_t* d_V, const uint64_t* d_counts,
                  uint8_t* d_enc, uint64_t enc_cap, sync_stream_t stream);

/* ---- a5 bucket pack (Fig. workflow, C11) ----------------
 * Enqueues on `stream` the device bucket plan of the preceding sync_compress
 * (greedy, DESIGN C11), the copy of every record into d_buckets, the headers,
 * directories and (flag) CRC-32; then BLOCKS until the plan table is on the
 * host (as sync_pack_result; the bucket bytes are ready when `stream` reaches
 * that point). Bucket b starts at h_offsets[b] (256-aligned) and is
 * h_sizes[b] bytes. *n_buckets = 0 when nothing changed. SYNC_ERR_CAPACITY as
 * sync_compress_pack_async.                                                 */
int sync_bucket_pack(sync_ctx* ctx, const uint8_t* d_enc, uint8_t* d_buckets, uint64_t buckets_cap,
                     uint32_t* n_buckets, uint64_t* h_offsets, uint64_t* h_sizes, uint32_t max_buckets,
                     sync_stream_t stream);
/* Upper bound of the bucket buffer for the current plan (after sync_compress; blocking). */
int sync_buckets_bound(sync_ctx* ctx, uint64_t* bytes, sync_stream_t stream);

/* ---- a2-a5 fused: plan -> bucket plan -> encode in place -------------------
 * Same bytes as sync_compress + sync_bucket_pack, but every record is encoded
 * straight into its bucket position (no staging stream, no copy). Everything
 * runs on the device (bucketing and packing overlap the transfer):
 * record plan + per-chunk model (K2), the greedy bucket plan (DESIGN C11,
 * bucket.cu), the encode (K3), the bucket headers/directories (+ CRC, K4).
 *
 * sync_compress_pack_async: ENQUEUE-ONLY (never blocks; capturable in a CUDA
 * graph). The bucket count / offsets / sizes land in the context's page-locked
 * table once the bucket plan kernel has run; read them with sync_pack_result.
 * If d_buckets is too small (buckets_cap) or more than max_buckets buckets are
 * needed, SYNC_ERR_CAPACITY is latched in the device status word, nothing is
 * encoded or written, and sync_pack_result reports it with the needed bytes.
 *
 * sync_pack_result: BLOCKS until the last enqueued bucket plan of this context
 * is complete (an event right after the plan kernel: not the encode behind
 * it), then copies n_buckets, h_offsets[0..n) / h_sizes[0..n) (host arrays of
 * >= max_buckets entries) and *h_need (bytes of the bucket buffer the plan
 * needs; may be NULL). Returns SYNC_ERR_CAPACITY (n_buckets = 0) if the plan
 * did not fit, SYNC_ERR_ARG if nothing was enqueued.
 *
 * sync_compress_pack = sync_compress_pack_async + sync_pack_result (the host
 * waits for the plan while the encode kernels run).                         */
int sync_compress_pack_async(sync_ctx* ctx, const uint32_t* d_I, const uint16_t* d_V, const uint64_t* d_counts,
                             uint8_t* d_buckets, uint64_t buckets_cap, uint32_t max_buckets, sync_stream_t stream);
int sync_pack_result(sync_ctx* ctx, uint32_t* n_buckets, uint64_t* h_offsets, uint64_t* h_sizes,
                     uint32_t max_buckets, uint64_t* h_need);
int sync_compress_pack(sync_ctx* ctx, const uint32_t* d_I, const uint16_t* d_V, const uint64_t* d_counts,
                       uint8_t* d_buckets, uint64_t buckets_cap, uint32_t* n_buckets, uint64_t* h_offsets,
                       uint64_t* h_sizes, uint32_t max_buckets, uint64_t* h_need, sync_stream_t stream);

/* ---- device-side bucket table (no host in the loop) ------------------------
 * sync_pack_table: device pointers to the context's bucket table (device memory
 * in its workspace), which every bucket plan rewrites (stream-ordered):
 * d_hdr[0] = bucket count (0 after a capacity failure), d_off[b * stride] /
 * d_size[b * stride] = bucket b's offset in the bucket buffer and its bytes.
 * Valid for the life of the context.
 * sync_decompress_apply_table: K5 over the buckets such a table lists (same
 * GPU or a peer that can read it): d_base = the bucket buffer; it launches
 * ceil(max_buckets / 32) decode kernels, each taking its slice of the table,
 * so the whole sender + receiver can be captured in one CUDA graph. flags bit
 * 0 = the dense launch variant (payload >= ~0.1 B per weight). Not with
 * SYNC_FLAG_CRC (SYNC_ERR_ARG): the CRC pass needs host sizes. Asynchronous. */
int sync_pack_table(sync_ctx* ctx, const uint64_t** d_hdr, const uint64_t** d_off, const uint64_t** d_size,
                    uint32_t* stride);
int sync_decompress_apply_table(sync_ctx* ctx, const uint8_t* d_base, const uint64_t* d_hdr, const uint64_t* d_off,
                                const uint64_t* d_size, uint32_t stride, uint32_t max_buckets,
                                uint16_t* const* d_weight_ptrs, uint32_t flags, sync_stream_t stream);

/* ---- a7 unpack / decompress (Alg. 3 l.5; "exact inverse") ---
 * sync_bucket_unpack validates one bucket in device memory (magic, version,
 * sizes, CRC when flagged) and writes one sync_record_view per record into
 * d_views (device, max_views entries) and the record count into d_n_records
 * (device u32). Failures latch BAD_MAGIC / VERSION / TRUNCATED / CRC / CORRUPT.
 * sync_decompress decodes every record of the bucket into d_I / d_V at
 * view.out_offset (tensor-local indices), d_cap entries of capacity.       */
int sync_bucket_unpack(sync_ctx* ctx, const uint8_t* d_bucket, uint64_t bytes,
                       sync_record_view* d_views, uint32_t max_views, uint32_t* d_n_records,
                       sync_stream_t stream);
int sync_decompress(sync_ctx* ctx, const uint8_t* d_bucket, uint64_t bytes, uint32_t* d_I, uint16_t* d_V,
                    uint64_t d_cap, sync_stream_t stream);

/* ---- a7+a8 fused decode + scatter-apply (Alg. 3 l.5-6) --
 * Validates the bucket, decodes every chunk and scatters V into
 * d_weight_ptrs[tensor_id] (DEVICE array of n_tensors device pointers) in
 * place. Indices >= numel latch SYNC_ERR_INDEX_RANGE and are not written.  */
int sync_decompress_apply(sync_ctx* ctx, const uint8_t* d_bucket, uint64_t bytes,
                          uint16_t* const* d_weight_ptrs, sync_stream_t stream);

/* Batched form of sync_decompress_apply: h_buckets / h_bytes are HOST arrays of n_buckets device bucket
 * addresses and sizes (e.g. the buckets of one transfer span); one kernel decodes up to 32 buckets, so many
 * small buckets do not each pay a launch that fills a fraction of the GPU. Same validation and errors.   */
int sync_decompress_apply_batched(sync_ctx* ctx, const uint8_t* const* h_buckets, const uint64_t* h_bytes,
                                  uint32_t n_buckets, uint16_t* const* d_weight_ptrs, sync_stream_t stream);

/* ---- a8 scatter-apply / a9 snapshot commit (Alg. 3 l.6) -----
 * d_W[d_I[k]] = d_V[k] for k < count (superset-safe, idempotent).
 * Indices >= numel are skipped and latch SYNC_ERR_INDEX_RANGE into *d_status
 * (device u32, OR-ed; may be NULL). sync_commit_snapshot is the same
 * operation on the Trainer's snapshot; call it only after the transfer of
 * this sync completed (DESIGN C13).                                        */
int sync_apply(uint16_t* d_W, const uint32_t* d_I, const uint16_t* d_V, uint64_t count, uint64_t numel,
               uint32_t* d_status, sync_stream_t stream);
int sync_commit_snapshot(uint16_t* d_snapshot, const uint32_t* d_I, const uint16_t* d_V, uint64_t count,
                         uint64_t numel, uint32_t* d_status, sync_stream_t stream);
/* Batched commit over the manifest from the raw output of sync_extract_batched. */
int sync_commit_snapshot_batched(sync_ctx* ctx, uint16_t* const* d_snapshot_ptrs, const uint32_t* d_I,
                                 const uint16_t* d_V, const uint64_t* d_counts, sync_stream_t stream);

/* ---- f3 routing: the current weights a FULL record copies ---------------------------------------------
 * d_new_ptrs: device array of the manifest's current-weight pointers (the `new` of sync_extract_batched, or
 * W under f1 tracking), read by sync_compress / sync_compress_pack for records routed FULL. Required when
 * the context was created with SYNC_FLAG_ROUTE (else those calls return SYNC_ERR_ARG); kept until replaced. */
int sync_set_current(sync_ctx* ctx, const uint16_t* const* d_new_ptrs);

/* ---- f1 cast-fused tracking (Alg. 1; hook P:386) ----------
 * The paper's own hook: the changed indices are collected inside the optimizer-step epilogue that casts the
 * fp32 master weights into the bf16 model weights, and accumulate across steps into the cumulative set
 * I_T (Alg. 1 l.7), a superset of the true delta that is harmless because absolute values are sent.
 * No snapshot is kept; the sync reads the set (1 bit per element) and gathers V = W[I].
 * The set is a caller-allocated, 16-byte aligned device bitmap of sync_bitmap_words() u32 words (zero it
 * once); tensor t owns ceil(numel_t / 32) consecutive words in manifest order, starting at a multiple of 4
 * words; bit b of word w = element 32 w + b.
 * sync_cast_track_batched: for every manifest tensor, W[i] <- round_BF16(master[i]) (round to nearest even
 *   on the fp32 bits, NaN -> 0x7FC0, DESIGN C18) and bit i |= (bits(W[i]) changed) (Alg. 1 l.5-7).
 *   d_master_ptrs / d_weight_ptrs: device arrays of per-tensor pointers (fp32 / bf16 bits); 16-byte aligned
 *   tensors take the vector path, others a scalar one. Only W sectors that changed are written.
 * sync_extract_tracked: I = ascending set bits of each tensor (tensor-local, records contiguous in manifest
 *   order exactly like sync_extract_batched), V = W[I], d_counts[t] = |I_t|; clears the bitmap when `clear`
 *   (next interval, Alg. 1 l.1). Capacity = max_changed: beyond it nothing is written out of bounds,
 *   d_counts hold the true counts, SYNC_ERR_CAPACITY is latched and the bitmap is left intact (retry with
 *   a larger context). The output feeds sync_compress(_pack).                                             */
int sync_bitmap_words(sync_ctx* ctx, uint64_t* words);
int sync_cast_track_batched(sync_ctx* ctx, const float* const* d_master_ptrs, uint16_t* const* d_weight_ptrs,
                            uint32_t* d_bitmap, sync_stream_t stream);
int sync_extract_tracked(sync_ctx* ctx, uint16_t* const* d_weight_ptrs, uint32_t* d_bitmap, uint32_t* d_I,
                         uint16_t* d_V, uint64_t* d_counts, int clear, sync_stream_t stream);

/* ---- status ----------------------------------------------------------------
 * sync_status: BLOCKING; synchronises `stream`, reads and clears the device
 * status word, returns SYNC_OK or the first latched error.
 * sync_ctx_stats: BLOCKING; statistics of the last sync_compress.          */
int sync_status(sync_ctx* ctx, sync_stream_t stream);
int sync_ctx_stats(sync_ctx* ctx, sync_stats* out, sync_stream_t stream);
const char* sync_strerror(int status);
/* Number of kernels the library launched since load (diagnostics). */
uint64_t sync_launch_count(void);
/* Process-wide cap on the CTAs of every kernel the library launches from now on (0 = no cap: the persistent
 * kernels size their grid to the SM count x occupancy). For sharing the GPU with a concurrently running
 * training step (as NCCL_MAX_CTAS does for collectives). Correctness never depends on how many CTAs are
 * co-resident: K1 claims its tiles from a ticket, so any grid, and any number of resident CTAs, finishes
 * (DESIGN.md §6 K1 forward progress). Returns SYNC_ERR_ARG for a negative value. Not stream-ordered.      */
int sync_set_max_ctas(int max_ctas);

#ifdef __cplusplus
}
#endif
#endif /* SPARSESYNC_H */
