// api.cu — the C ABI of include/sparsesync.h: context, workspace layout,
// argument checks and launch sequencing. All arithmetic of the method runs in
// the kernels of extract.cu / plan.cu / encode.cu / pack.cu / decode.cu /
// apply.cu; the host only sequences launches, plans bucket boundaries from the
// record sizes (greedy, DESIGN C11) and reads back status words.
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "kernels.h"

using namespace ss;

namespace {
// NVTX range around each enqueueing entry point (named after it), so a trace (nsys, or ncu --nvtx
// --nvtx-include) attributes the kernels to the ABI call that launched them; a no-op without a tool attached
struct ApiRange {
  explicit ApiRange(const char* name) { nvtxRangePushA(name); }
  ~ApiRange() { nvtxRangePop(); }
};
}  // namespace

namespace ss {
static std::atomic<uint64_t> g_launches{0};
static std::atomic<int> g_max_ctas{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev >= 0 && dev < kMaxDevices ? dev : 0;
}
int clamp_ctas(int grid) {
  const int m = g_max_ctas.load(std::memory_order_relaxed);
  return (m > 0 && grid > m) ? m : grid;
}
}  // namespace ss

namespace {

constexpr u64 kAlign = 256;

struct Layout {
  u64 numel, tile_prefix, tile_tensor, misc, tile_state, stage_ring, rec_off, chunk_off, maxgap, rec_mode, rec_bytes, enc_off;
  u64 chunk_hi, chunk_mode, chunk_hioff, chunk_rhdr, word_scratch, rec_dst, totals, recs, bks, views, nviews, crc;
  u64 bm_off, group_sum, chunk_esc, chunk_escoff, chunk_t, bitmap8, rec_list, srec, crec, nxt, bstart, seg_off, gscan, total;
};

u64 crc_slots(u64 max_bucket_bytes) { return max_bucket_bytes / 4096 + 4 + 32; }  // + 32 bad flags

Layout make_layout(u32 T, u64 n_tiles, u64 max_chunks, u64 crc_n, u64 max_changed, u64 bm8_words = 0) {
  Layout L{};
  u64 o = 0;
  auto take = [&](u64 bytes) {
    u64 at = o;
    o = pad_to(o + (bytes ? bytes : 8), kAlign);
    return at;
  };
  L.numel = take(8ull * T);
  L.tile_prefix = take(8ull * (T + 1));
  L.tile_tensor = take(4ull * n_tiles);
  L.misc = take(4 * 64);
  L.tile_state = take(8ull * n_tiles);
  L.stage_ring = take(stage_ring_bytes(n_tiles));
  L.rec_off = take(8ull * (T + 1));
  L.chunk_off = take(8ull * (T + 1));
  L.maxgap = take(4ull * T);
  L.rec_mode = take(4ull * T);
  L.rec_bytes = take(8ull * T);
  L.enc_off = take(8ull * (T + 1));
  L.chunk_hi = take(4ull * max_chunks);
  L.chunk_mode = take(4ull * max_chunks);
  L.chunk_hioff = take(8ull * (max_chunks + 1));
  L.chunk_rhdr = take(4ull * kRhdrWords * max_chunks);
  L.word_scratch = take(2ull * (max_changed / 2 + max_chunks + 2));
  L.rec_dst = take(8ull * T);
  L.totals = take(8 * 16);
  L.recs = take(sizeof(RecordDesc) * (u64)T);
  L.bks = take(sizeof(BucketDesc) * (u64)(T + 1));
  L.views = take(sizeof(sync_record_view) * (u64)T);
  L.nviews = take(8);
  L.crc = take(4ull * crc_n);
  L.bm_off = take(8ull * (T + 1));                       // f1: bitmap word offset per tensor
  L.group_sum = take(8ull * (n_tiles / 1024 + 2));       // f1: tile-offset scan groups
  L.chunk_esc = take(4ull * max_chunks);                   // f4: escapes per chunk
  L.chunk_escoff = take(8ull * (max_chunks + 1));          // f4: their exclusive prefix
  L.chunk_t = take(4ull * max_chunks);                     // tensor of each chunk
  L.bitmap8 = take(4ull * bm8_words);                      // FP8: change bitmap of the extract
  L.rec_list = take(4ull * T);                             // device bucket plan (bucket.cu)
  L.srec = take(8ull * (T + 1));
  L.crec = take(8ull * (T + 1));
  L.nxt = take(4ull * T);
  L.bstart = take(4ull * (T + 1));
  L.seg_off = take(8ull * (T + 1));
  L.gscan = take(32ull * (2 * ((T + 1023) / 1024 + 1) + (max_chunks + 1023) / 1024 + 1));   // scan.cuh states
  L.total = o;
  return L;
}

struct Dims {
  u32 T;
  u64 n_tiles, max_chunks, max_record, crc_n, bm8_words;
};

int check_manifest(const sync_manifest* m, const sync_config* c, Dims* d) {
  if (!m || !c || (m->n_tensors && !m->numel)) return SYNC_ERR_ARG;
  if (c->codec > SYNC_CODEC_COMPRESSED || c->bucket_limit < 64) return SYNC_ERR_ARG;
  if (c->dtype > SYNC_DTYPE_FP8) return SYNC_ERR_DTYPE;
  d->T = m->n_tensors;
  d->n_tiles = 0;
  u64 maxn = 0;
  for (u32 t = 0; t < m->n_tensors; ++t) {
    if (m->numel[t] >= (1ull << 31)) return SYNC_ERR_ARG;
    d->n_tiles += (m->numel[t] + kTile - 1) / kTile;
    maxn = m->numel[t] > maxn ? m->numel[t] : maxn;
  }
  d->bm8_words = 0;   // FP8 contexts extract through a change bitmap (same per-tensor word layout as f1)
  if (c->dtype == SYNC_DTYPE_FP8)
    for (u32 t = 0; t < m->n_tensors; ++t) d->bm8_words += pad_to((m->numel[t] + 31) / 32, 4);
  d->max_chunks = (c->max_changed + kChunk - 1) / kChunk + d->T + 1;
  // largest possible record (one tensor fully changed): bounds a received bucket for the CRC scratch
  d->max_record = 6 * maxn + 20 * ((maxn + kChunk - 1) / kChunk) + 64;
  u64 mb = c->bucket_limit > d->max_record + 64 ? c->bucket_limit : d->max_record + 64;
  // CRC scratch: one received bucket (receiver), or the segments of every bucket of a sender plan: payload
  // <= the encoded-stream bound + bucket headers/directories, + one partial segment per bucket
  const u64 enc_bound = 6 * c->max_changed + 20 * d->max_chunks + 64ull * d->T + 64;
  const u64 send_segs = (enc_bound + 64ull * (d->T + 1) + 8ull * d->T) / 65536 + d->T + 1;
  d->crc_n = crc_slots(mb) > send_segs ? crc_slots(mb) : send_segs;
  return SYNC_OK;
}

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

#define CK(x)                                   \
  do {                                          \
    if ((x) != cudaSuccess) return SYNC_ERR_CUDA; \
  } while (0)

}  // namespace

struct sync_ctx {
  Dims d;
  sync_config cfg;
  std::vector<u64> numel, tile_prefix;
  u64 total_elems = 0;   // sum of numel (decode variant choice)
  std::vector<u32> tile_tensor;
  std::vector<u64> bm_off;   // f1: bitmap word offset of each tensor (ceil(numel / 32) words each)
  u8* ws;
  Layout L;
  Plan plan;
  u32* misc;  // [0] tile counter, [1] status, [2] crc bad flag
  int sm_count;
  int grid;   // grid-stride kernels: CTAs of 256 threads
  const u64* plan_counts;
  bool plan_valid;
  // the device bucket plan's result table, written by k_bucket_plan straight into mapped page-locked host
  // memory: {n_buckets, failed, need} + offsets[T + 1] + sizes[T + 1]; valid once pack_ev has completed
  u64* h_pack;
  u64* d_pack;
  cudaEvent_t pack_ev;
  bool pack_pending;
  ~sync_ctx() {
    if (h_pack) cudaFreeHost(h_pack);
    if (pack_ev) cudaEventDestroy(pack_ev);
  }
};

extern "C" {

int sync_workspace_size(const sync_manifest* m, const sync_config* c, size_t* bytes) {
  Dims d;
  int st = check_manifest(m, c, &d);
  if (st) return st;
  if (!bytes) return SYNC_ERR_ARG;
  *bytes = make_layout(d.T, d.n_tiles, d.max_chunks, d.crc_n, c->max_changed, d.bm8_words).total;
  return SYNC_OK;
}

int sync_ctx_create(sync_ctx** out, const sync_manifest* m, const sync_config* c, void* d_workspace,
                    size_t workspace_bytes, sync_stream_t stream) {
  if (!out) return SYNC_ERR_ARG;
  *out = nullptr;
  Dims d;
  int st = check_manifest(m, c, &d);
  if (st) return st;
  Layout L = make_layout(d.T, d.n_tiles, d.max_chunks, d.crc_n, c->max_changed, d.bm8_words);
  if (!d_workspace || workspace_bytes < L.total) return SYNC_ERR_WORKSPACE;
  if (!aligned16(d_workspace)) return SYNC_ERR_ALIGNMENT;
  sync_ctx* x = new (std::nothrow) sync_ctx();
  if (!x) return SYNC_ERR_ARG;
  x->d = d;
  x->cfg = *c;
  x->ws = static_cast<u8*>(d_workspace);
  x->L = L;
  x->numel.assign(m->numel, m->numel + d.T);
  for (u64 n : x->numel) x->total_elems += n;
  x->tile_prefix.resize(d.T + 1);
  u64 acc = 0;
  for (u32 t = 0; t < d.T; ++t) {
    x->tile_prefix[t] = acc;
    acc += (x->numel[t] + kTile - 1) / kTile;
  }
  x->tile_prefix[d.T] = acc;
  x->tile_tensor.resize(acc);
  for (u32 t = 0; t < d.T; ++t)
    for (u64 k = x->tile_prefix[t]; k < x->tile_prefix[t + 1]; ++k) x->tile_tensor[k] = t;
  x->bm_off.resize(d.T + 1);
  u64 wacc = 0;
  for (u32 t = 0; t < d.T; ++t) {
    x->bm_off[t] = wacc;
    wacc += pad_to((x->numel[t] + 31) / 32, 4);   // every tensor's words start 16-byte aligned
  }
  x->bm_off[d.T] = wacc;
  cudaStream_t s = (cudaStream_t)stream;
  u8* w = x->ws;
  if (d.T) {
    if (cudaMemcpyAsync(w + L.numel, x->numel.data(), 8ull * d.T, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(w + L.tile_prefix, x->tile_prefix.data(), 8ull * (d.T + 1), cudaMemcpyHostToDevice, s) !=
            cudaSuccess ||
        (acc && cudaMemcpyAsync(w + L.tile_tensor, x->tile_tensor.data(), 4ull * acc, cudaMemcpyHostToDevice, s) !=
                    cudaSuccess) ||
        cudaMemcpyAsync(w + L.bm_off, x->bm_off.data(), 8ull * (d.T + 1), cudaMemcpyHostToDevice, s) != cudaSuccess) {
      delete x;
      return SYNC_ERR_CUDA;
    }
  }
  if (cudaMemsetAsync(w + L.misc, 0, 4 * 64, s) != cudaSuccess ||
      cudaMemsetAsync(w + L.gscan, 0, L.seg_off < L.gscan ? L.total - L.gscan : 0, s) != cudaSuccess ||
      cudaMemsetAsync(w + L.totals, 0, 8 * 16, s) != cudaSuccess) {
    delete x;
    return SYNC_ERR_CUDA;
  }
  x->misc = reinterpret_cast<u32*>(w + L.misc);
  x->h_pack = nullptr;
  x->pack_ev = nullptr;
  x->pack_pending = false;
  if (cudaHostAlloc(&x->h_pack, 8ull * (4 + 2 * (d.T + 1)), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(&x->d_pack, x->h_pack, 0) != cudaSuccess ||
      cudaEventCreateWithFlags(&x->pack_ev, cudaEventDisableTiming) != cudaSuccess) {
    delete x;
    return SYNC_ERR_CUDA;
  }
  memset(x->h_pack, 0, 8ull * (4 + 2 * (d.T + 1)));
  Plan& p = x->plan;
  p.n_tensors = d.T;
  p.cap = c->max_changed;
  p.codec = c->codec;
  p.route = (c->flags & SYNC_FLAG_ROUTE) ? 1 : 0;
  p.dtype = c->dtype ? c->dtype : SYNC_DTYPE_BF16;
  p.escape = (c->flags & SYNC_FLAG_ESCAPE) ? 1 : 0;
  p.chunk_esc = reinterpret_cast<u32*>(w + L.chunk_esc);
  p.chunk_escoff = reinterpret_cast<u64*>(w + L.chunk_escoff);
  p.chunk_t = reinterpret_cast<u32*>(w + L.chunk_t);
  p.cur = nullptr;
  p.max_chunks = d.max_chunks;
  p.numel = reinterpret_cast<const u64*>(w + L.numel);
  p.rec_off = reinterpret_cast<u64*>(w + L.rec_off);
  p.chunk_off = reinterpret_cast<u64*>(w + L.chunk_off);
  p.maxgap = reinterpret_cast<u32*>(w + L.maxgap);
  p.rec_mode = reinterpret_cast<u32*>(w + L.rec_mode);
  p.rec_bytes = reinterpret_cast<u64*>(w + L.rec_bytes);
  p.enc_off = reinterpret_cast<u64*>(w + L.enc_off);
  p.rec_dst = p.enc_off;
  p.chunk_hi = reinterpret_cast<u32*>(w + L.chunk_hi);
  p.chunk_mode = reinterpret_cast<u32*>(w + L.chunk_mode);
  p.chunk_hioff = reinterpret_cast<u64*>(w + L.chunk_hioff);
  p.chunk_rhdr = reinterpret_cast<u32*>(w + L.chunk_rhdr);
  p.word_scratch = reinterpret_cast<u16*>(w + L.word_scratch);
  p.totals = reinterpret_cast<u64*>(w + L.totals);
  p.status = x->misc + 1;
  p.work = reinterpret_cast<u64*>(x->misc + 16);   // misc words 16..19
  p.tickets = x->misc + 24;                         // misc words 24..26 (zeroed at creation, never reset)
  p.gscan = reinterpret_cast<u64*>(w + L.gscan);
  p.gscan_T = (d.T + 1023) / 1024 + 1;
  p.gscan_C = (u32)((d.max_chunks + 1023) / 1024);
  p.epochs = x->misc + 28;                          // misc words 28..30 (zeroed at creation)
  p.rec_list = reinterpret_cast<u32*>(w + L.rec_list);
  p.srec = reinterpret_cast<u64*>(w + L.srec);
  p.crec = reinterpret_cast<u64*>(w + L.crec);
  int dev = 0;
  cudaGetDevice(&dev);
  x->sm_count = 148;
  cudaDeviceGetAttribute(&x->sm_count, cudaDevAttrMultiProcessorCount, dev);
  x->grid = x->sm_count * 8;
  x->plan_counts = nullptr;
  x->plan_valid = false;
  *out = x;
  return SYNC_OK;
}

int sync_ctx_destroy(sync_ctx* ctx) {
  if (ctx) cudaDeviceSynchronize();   // in-flight copies may still read the ctx's pinned host tables
  delete ctx;
  return SYNC_OK;
}

// ------------------------------------------------------------------------ extract
int sync_extract_workspace_size(uint64_t n, size_t* bytes) {
  if (!bytes || n >= (1ull << 31)) return SYNC_ERR_ARG;
  const u64 n_tiles = (n + kTile - 1) / kTile;
  *bytes = kAlign + pad_to(8 * n_tiles + 8, kAlign) + stage_ring_bytes(n_tiles);
  return SYNC_OK;
}

int sync_extract(const uint16_t* d_old, const uint16_t* d_new, uint64_t n, uint32_t* d_I, uint16_t* d_V,
                 uint64_t cap, uint64_t* d_count, void* d_workspace, size_t workspace_bytes, sync_stream_t stream) {
  ApiRange nvtx_range("sync_extract");
  size_t need;
  if (sync_extract_workspace_size(n, &need)) return SYNC_ERR_ARG;
  if (!d_count || !d_workspace || (n && (!d_old || !d_new))) return SYNC_ERR_ARG;
  if (workspace_bytes < need) return SYNC_ERR_WORKSPACE;
  if (!aligned16(d_I) || !aligned16(d_V)) return SYNC_ERR_ALIGNMENT;   // the header's I / V contract
  if (!aligned16(d_workspace)) return SYNC_ERR_ALIGNMENT;
  cudaStream_t s = (cudaStream_t)stream;
  u8* w = static_cast<u8*>(d_workspace);
  u32* misc = reinterpret_cast<u32*>(w);
  u64 n_tiles = (n + kTile - 1) / kTile;
  CK(cudaMemsetAsync(misc, 0, 4, s));  // tile counter (status is sticky until read)
  CK(cudaMemsetAsync(d_count, 0, 8, s));
  if (n_tiles) CK(cudaMemsetAsync(w + kAlign, 0, 8 * n_tiles, s));
  launch_extract_single(d_old, d_new, n, d_I, d_V, cap, d_count, reinterpret_cast<u64*>(w + kAlign), misc,
                        reinterpret_cast<u32*>(w + kAlign + pad_to(8 * n_tiles + 8, kAlign)), misc + 1,
                        s);
  CK(cudaGetLastError());
  return SYNC_OK;
}

int sync_extract_status(void* d_workspace, sync_stream_t stream) {
  if (!d_workspace) return SYNC_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  u32 v = 0;
  u32* st = reinterpret_cast<u32*>(d_workspace) + 1;
  CK(cudaStreamSynchronize(s));
  CK(cudaMemcpy(&v, st, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemset(st, 0, 4));
  return -(int)v;
}

static TrackArgs track_args(sync_ctx* x, uint32_t* d_bitmap);

int sync_extract_batched(sync_ctx* x, const uint16_t* const* d_old_ptrs, const uint16_t* const* d_new_ptrs,
                         uint32_t* d_I, uint16_t* d_V, uint64_t* d_counts, sync_stream_t stream) {
  ApiRange nvtx_range("sync_extract_batched");
  if (!x || (x->d.T && (!d_old_ptrs || !d_new_ptrs || !d_counts))) return SYNC_ERR_ARG;
  if (!aligned16(d_I) || !aligned16(d_V)) return SYNC_ERR_ALIGNMENT;   // the header's I / V contract
  cudaStream_t s = (cudaStream_t)stream;
  x->plan_valid = false;
  if (x->d.T == 0) return SYNC_OK;
  CK(cudaMemsetAsync(x->misc, 0, 4, s));
  CK(cudaMemsetAsync(d_counts, 0, 8ull * x->d.T, s));
  if (x->plan.dtype == SYNC_DTYPE_FP8 && getenv("SS_FP8_BITMAP")) {   // alternative: diff bitmap + compaction
    TrackArgs a = track_args(x, reinterpret_cast<u32*>(x->ws + x->L.bitmap8));
    a.counts = d_counts;
    a.I = d_I;
    a.V = d_V;
    launch_extract8(a, reinterpret_cast<const uint8_t* const*>(d_old_ptrs),
                    reinterpret_cast<const uint8_t* const*>(d_new_ptrs), clamp_ctas(16 * x->sm_count), s);
    CK(cudaGetLastError());
    return SYNC_OK;
  }
  if (x->d.n_tiles) CK(cudaMemsetAsync(x->ws + x->L.tile_state, 0, 8 * x->d.n_tiles, s));
  launch_extract_batched(d_old_ptrs, d_new_ptrs, reinterpret_cast<const u64*>(x->ws + x->L.tile_prefix),
                         reinterpret_cast<const u32*>(x->ws + x->L.tile_tensor), x->plan.numel, x->d.T, x->d.n_tiles, d_I, d_V, x->cfg.max_changed, d_counts,
                         reinterpret_cast<u64*>(x->ws + x->L.tile_state), x->misc,
                         reinterpret_cast<u32*>(x->ws + x->L.stage_ring), x->misc + 1, s,
                         x->plan.dtype == SYNC_DTYPE_FP8 ? 1 : 2);
  CK(cudaGetLastError());
  return SYNC_OK;
}

// ------------------------------------------------------------------------ f1 cast-fused tracking
static TrackArgs track_args(sync_ctx* x, uint32_t* d_bitmap) {
  TrackArgs a{};
  a.n_tiles = x->d.n_tiles;
  a.n_tensors = x->d.T;
  a.tile_tensor = reinterpret_cast<const u32*>(x->ws + x->L.tile_tensor);
  a.tile_prefix = reinterpret_cast<const u64*>(x->ws + x->L.tile_prefix);
  a.numel = x->plan.numel;
  a.bm_off = reinterpret_cast<const u64*>(x->ws + x->L.bm_off);
  a.bitmap = d_bitmap;
  a.tile_off = reinterpret_cast<u64*>(x->ws + x->L.tile_state);
  a.group_sum = reinterpret_cast<u64*>(x->ws + x->L.group_sum);
  a.cap = x->cfg.max_changed;
  a.totals = x->plan.totals;
  a.status = x->misc + 1;
  return a;
}

int sync_set_current(sync_ctx* x, const uint16_t* const* d_new_ptrs) {
  if (!x) return SYNC_ERR_ARG;
  x->plan.cur = d_new_ptrs;
  return SYNC_OK;
}

int sync_bitmap_words(sync_ctx* x, uint64_t* words) {
  if (!x || !words) return SYNC_ERR_ARG;
  *words = x->bm_off.empty() ? 0 : x->bm_off.back();
  return SYNC_OK;
}

int sync_cast_track_batched(sync_ctx* x, const float* const* d_master_ptrs, uint16_t* const* d_weight_ptrs,
                            uint32_t* d_bitmap, sync_stream_t stream) {
  ApiRange nvtx_range("sync_cast_track_batched");
  if (!x || (x->d.T && (!d_master_ptrs || !d_weight_ptrs || !d_bitmap))) return SYNC_ERR_ARG;
  if (x->d.T && !aligned16(d_bitmap)) return SYNC_ERR_ALIGNMENT;
  if (x->plan.dtype != SYNC_DTYPE_BF16) return SYNC_ERR_DTYPE;   // the cast is round_BF16 (Alg. 1 l.5)
  launch_cast_track(track_args(x, d_bitmap), d_master_ptrs, d_weight_ptrs, clamp_ctas(8 * x->sm_count), (cudaStream_t)stream);
  CK(cudaGetLastError());
  return SYNC_OK;
}

int sync_extract_tracked(sync_ctx* x, uint16_t* const* d_weight_ptrs, uint32_t* d_bitmap, uint32_t* d_I,
                         uint16_t* d_V, uint64_t* d_counts, int clear, sync_stream_t stream) {
  ApiRange nvtx_range("sync_extract_tracked");
  if (!x || (x->d.T && (!d_weight_ptrs || !d_bitmap || !d_counts))) return SYNC_ERR_ARG;
  if (!aligned16(d_I) || !aligned16(d_V)) return SYNC_ERR_ALIGNMENT;   // the header's I / V contract
  x->plan_valid = false;
  if (x->d.T == 0) return SYNC_OK;
  TrackArgs a = track_args(x, d_bitmap);
  a.counts = d_counts;
  a.I = d_I;
  a.V = d_V;
  launch_extract_tracked(a, d_weight_ptrs, clear, clamp_ctas(16 * x->sm_count), (cudaStream_t)stream);
  CK(cudaGetLastError());
  return SYNC_OK;
}

// ------------------------------------------------------------------------ compress
int sync_enc_bound(const sync_manifest* m, const sync_config* c, uint64_t* bytes) {
  Dims d;
  int st = check_manifest(m, c, &d);
  if (st) return st;
  if (!bytes) return SYNC_ERR_ARG;
  *bytes = 6 * c->max_changed + 20 * d.max_chunks + 64ull * d.T + 64;
  return SYNC_OK;
}

int sync_compress(sync_ctx* x, const uint32_t* d_I, const uint16_t* d_V, const uint64_t* d_counts, uint8_t* d_enc,
                  uint64_t enc_cap, sync_stream_t stream) {
  ApiRange nvtx_range("sync_compress");
  if (!x || (x->d.T && (!d_counts || !d_enc))) return SYNC_ERR_ARG;
  if (x->plan.route && !x->plan.cur) return SYNC_ERR_ARG;   // SYNC_FLAG_ROUTE needs sync_set_current
  if (!aligned16(d_enc)) return SYNC_ERR_ALIGNMENT;
  if (!aligned16(d_I) || !aligned16(d_V)) return SYNC_ERR_ALIGNMENT;   // the header's I / V contract
  cudaStream_t s = (cudaStream_t)stream;
  x->plan.enc_cap = enc_cap;
  launch_plan_scan(x->plan, d_counts, s);
  // CTA-per-chunk kernels of 128 threads: 2x the grid of the 256-thread kernels (~9 resident per SM)
  if (x->cfg.codec == SYNC_CODEC_COMPRESSED) launch_chunk_stats(x->plan, d_I, d_V, d_counts, clamp_ctas(2 * x->grid), s);
  launch_plan_sizes(x->plan, d_counts, s);
  launch_encode(x->plan, d_I, d_V, d_counts, d_enc, clamp_ctas(2 * x->grid), s);
  CK(cudaGetLastError());
  x->plan_counts = d_counts;
  x->plan_valid = true;
  return SYNC_OK;
}

// ------------------------------------------------------------------------ pack
static int read_totals(sync_ctx* x, u64* t, cudaStream_t s) {
  CK(cudaMemcpyAsync(t, x->plan.totals, 8 * 16, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return SYNC_OK;
}

int sync_buckets_bound(sync_ctx* x, uint64_t* bytes, sync_stream_t stream) {
  if (!x || !bytes || !x->plan_valid) return SYNC_ERR_ARG;
  u64 t[16];
  int st = read_totals(x, t, (cudaStream_t)stream);
  if (st) return st;
  u64 nr = t[kTotRecords];
  *bytes = t[kTotEnc] + 8 * nr + (nr + 1) * (32 + 16 + kBucketAlign);
  return SYNC_OK;
}

// Enqueue the device bucket plan (bucket.cu) and the bucket assembly after it. fused: the records are encoded
// straight into their bucket positions (k_encode after the plan); else d_enc holds the contiguous encoded
// stream of sync_compress and k_pack_copy moves it. pack_ev completes when the plan table is in host memory,
// ahead of the encode/copy kernels behind it.
static int enqueue_pack(sync_ctx* x, const uint32_t* d_I, const uint16_t* d_V, const uint64_t* d_counts,
                        const uint8_t* d_enc, uint8_t* d_buckets, uint64_t buckets_cap, uint32_t max_buckets,
                        cudaStream_t s) {
  const Layout& L = x->L;
  u8* w = x->ws;
  u64* d_dst = reinterpret_cast<u64*>(w + L.rec_dst);
  BucketPlan b{};
  b.rec_list = x->plan.rec_list;
  b.srec = x->plan.srec;
  b.crec = x->plan.crec;
  b.enc_off = x->plan.enc_off;
  b.nxt = reinterpret_cast<u32*>(w + L.nxt);
  b.bstart = reinterpret_cast<u32*>(w + L.bstart);
  b.seg_off = reinterpret_cast<u64*>(w + L.seg_off);
  b.recs = reinterpret_cast<RecordDesc*>(w + L.recs);
  b.bks = reinterpret_cast<BucketDesc*>(w + L.bks);
  b.rec_dst = d_enc ? nullptr : d_dst;
  b.totals = x->plan.totals;
  b.status = x->plan.status;
  b.limit = x->cfg.bucket_limit;
  b.cap_bytes = buckets_cap;
  b.max_buckets = max_buckets;
  b.out_hdr = x->d_pack;
  b.out_off = x->d_pack + 4;
  b.out_size = x->d_pack + 4 + (x->d.T + 1);
  launch_bucket_plan(b, x->d.T, x->sm_count, s);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(s, &cap));
  if (cap == cudaStreamCaptureStatusActive) CK(cudaEventRecordWithFlags(x->pack_ev, s, cudaEventRecordExternal));
  else CK(cudaEventRecord(x->pack_ev, s));
  x->pack_pending = true;
  if (!d_enc) {   // fused: encode every record into its bucket position
    x->plan.rec_dst = d_dst;
    launch_encode(x->plan, d_I, d_V, d_counts, d_buckets, clamp_ctas(2 * x->grid), s);
    x->plan.rec_dst = x->plan.enc_off;
  }
  const u32 T1 = x->d.T ? x->d.T : 1u;
  const u32 mb = max_buckets < T1 ? max_buckets : T1;
  launch_pack(d_enc, d_buckets, b.recs, b.bks, b.totals, mb, x->cfg.flags, clamp_ctas(x->grid), s);
  if (x->cfg.flags & SYNC_FLAG_CRC)
    crc_fill(d_buckets, b.bks, b.seg_off, b.totals, mb, reinterpret_cast<u32*>(w + L.crc), clamp_ctas(x->grid), s);
  CK(cudaGetLastError());
  return SYNC_OK;
}

int sync_pack_result(sync_ctx* x, uint32_t* n_buckets, uint64_t* h_offsets, uint64_t* h_sizes,
                     uint32_t max_buckets, uint64_t* h_need) {
  if (!x || !n_buckets) return SYNC_ERR_ARG;
  *n_buckets = 0;
  if (h_need) *h_need = 0;
  if (!x->pack_pending) return SYNC_ERR_ARG;
  CK(cudaEventSynchronize(x->pack_ev));
  const volatile u64* hp = x->h_pack;
  const u64 nb = hp[0], failed = hp[1];
  if (h_need) *h_need = hp[2];
  if (failed) return SYNC_ERR_CAPACITY;   // latched on the device too; nothing was encoded or packed
  if (nb > max_buckets) return SYNC_ERR_CAPACITY;
  const u64* off = x->h_pack + 4;
  const u64* sz = x->h_pack + 4 + (x->d.T + 1);
  for (u64 b = 0; b < nb; ++b) {
    if (h_offsets) h_offsets[b] = off[b];
    if (h_sizes) h_sizes[b] = sz[b];
  }
  *n_buckets = (u32)nb;
  return SYNC_OK;
}

int sync_bucket_pack(sync_ctx* x, const uint8_t* d_enc, uint8_t* d_buckets, uint64_t buckets_cap,
                     uint32_t* n_buckets, uint64_t* h_offsets, uint64_t* h_sizes, uint32_t max_buckets,
                     sync_stream_t stream) {
  ApiRange nvtx_range("sync_bucket_pack");
  if (!x || !n_buckets || !x->plan_valid || !d_enc) return SYNC_ERR_ARG;
  if (!aligned16(d_buckets) || !aligned16(d_enc)) return SYNC_ERR_ALIGNMENT;
  *n_buckets = 0;
  int st = enqueue_pack(x, nullptr, nullptr, nullptr, d_enc, d_buckets, buckets_cap, max_buckets,
                        (cudaStream_t)stream);
  if (st) return st;
  return sync_pack_result(x, n_buckets, h_offsets, h_sizes, max_buckets, nullptr);
}

int sync_compress_pack_async(sync_ctx* x, const uint32_t* d_I, const uint16_t* d_V, const uint64_t* d_counts,
                             uint8_t* d_buckets, uint64_t buckets_cap, uint32_t max_buckets, sync_stream_t stream) {
  ApiRange nvtx_range("sync_compress_pack_async");
  if (!x || (x->d.T && !d_counts)) return SYNC_ERR_ARG;
  if (x->plan.route && !x->plan.cur) return SYNC_ERR_ARG;   // SYNC_FLAG_ROUTE needs sync_set_current
  if (!aligned16(d_buckets)) return SYNC_ERR_ALIGNMENT;
  if (!aligned16(d_I) || !aligned16(d_V)) return SYNC_ERR_ALIGNMENT;   // the header's I / V contract
  cudaStream_t s = (cudaStream_t)stream;
  // plan (record sizes) exactly as sync_compress, without the encode
  x->plan.enc_cap = ~0ull;
  x->plan.rec_dst = x->plan.enc_off;
  launch_plan_scan(x->plan, d_counts, s);
  if (x->cfg.codec == SYNC_CODEC_COMPRESSED)
    launch_chunk_stats(x->plan, d_I, d_V, d_counts, clamp_ctas(2 * x->grid), s);
  launch_plan_sizes(x->plan, d_counts, s);
  CK(cudaGetLastError());
  x->plan_counts = d_counts;
  x->plan_valid = true;
  return enqueue_pack(x, d_I, d_V, d_counts, nullptr, d_buckets, buckets_cap, max_buckets, s);
}

int sync_compress_pack(sync_ctx* x, const uint32_t* d_I, const uint16_t* d_V, const uint64_t* d_counts,
                       uint8_t* d_buckets, uint64_t buckets_cap, uint32_t* n_buckets, uint64_t* h_offsets,
                       uint64_t* h_sizes, uint32_t max_buckets, uint64_t* h_need, sync_stream_t stream) {
  ApiRange nvtx_range("sync_compress_pack");
  if (!n_buckets) return SYNC_ERR_ARG;
  *n_buckets = 0;
  if (h_need) *h_need = 0;
  int st = sync_compress_pack_async(x, d_I, d_V, d_counts, d_buckets, buckets_cap, max_buckets, stream);
  if (st) return st;
  // the host waits for the plan table only: the encode / pack kernels queued behind it keep the GPU busy
  return sync_pack_result(x, n_buckets, h_offsets, h_sizes, max_buckets, h_need);
}

// ------------------------------------------------------------------------ receive
// CRC checks (flag on) of n <= 32 buckets: bad flags in crc scratch [0, 32), segment CRCs after them.
constexpr u32 kCrcFlagSlots = 32;
static int maybe_crc_check(sync_ctx* x, const uint8_t* const* d_buckets, const uint64_t* bytes, u32 n,
                           cudaStream_t s, const u32** bad) {
  *bad = nullptr;
  if (!(x->cfg.flags & SYNC_FLAG_CRC)) return SYNC_OK;
  for (u32 i = 0; i < n; ++i)
    if (crc_slots(bytes[i]) > x->d.crc_n) return SYNC_ERR_CAPACITY;   // crc_slots includes the flags
  u32* scratch = reinterpret_cast<u32*>(x->ws + x->L.crc);
  CK(cudaMemsetAsync(scratch, 0, 4 * kCrcFlagSlots, s));
  for (u32 i = 0; i < n; ++i)
    launch_crc_check(d_buckets[i], bytes[i], scratch + kCrcFlagSlots, scratch + i, x->plan.status, s);
  *bad = scratch;
  return SYNC_OK;
}

int sync_bucket_unpack(sync_ctx* x, const uint8_t* d_bucket, uint64_t bytes, sync_record_view* d_views,
                       uint32_t max_views, uint32_t* d_n_records, sync_stream_t stream) {
  ApiRange nvtx_range("sync_bucket_unpack");
  if (!x || !d_bucket || !d_views || !d_n_records) return SYNC_ERR_ARG;
  if (!aligned16(d_bucket)) return SYNC_ERR_ALIGNMENT;
  cudaStream_t s = (cudaStream_t)stream;
  const u32* bad;
  int st = maybe_crc_check(x, &d_bucket, &bytes, 1, s, &bad);
  if (st) return st;
  launch_unpack(d_bucket, bytes, x->d.T, x->plan.numel, d_views, max_views, d_n_records, x->plan.status,
                x->plan.dtype, s);
  CK(cudaGetLastError());
  return SYNC_OK;
}

int sync_decompress(sync_ctx* x, const uint8_t* d_bucket, uint64_t bytes, uint32_t* d_I, uint16_t* d_V,
                    uint64_t d_cap, sync_stream_t stream) {
  ApiRange nvtx_range("sync_decompress");
  if (!x || !d_bucket) return SYNC_ERR_ARG;
  if (!aligned16(d_bucket)) return SYNC_ERR_ALIGNMENT;
  if (!aligned16(d_I) || !aligned16(d_V)) return SYNC_ERR_ALIGNMENT;   // the header's I / V contract
  cudaStream_t s = (cudaStream_t)stream;
  const u32* bad;
  int st = maybe_crc_check(x, &d_bucket, &bytes, 1, s, &bad);
  if (st) return st;
  sync_record_view* views = reinterpret_cast<sync_record_view*>(x->ws + x->L.views);
  u32* nv = reinterpret_cast<u32*>(x->ws + x->L.nviews);
  launch_unpack(d_bucket, bytes, x->d.T, x->plan.numel, views, x->d.T, nv, x->plan.status, x->plan.dtype, s);
  launch_decode(&d_bucket, &bytes, 1, x->d.T, x->plan.numel, nullptr, views, d_I, d_V, d_cap, x->plan.status, bad,
                x->plan.dtype, clamp_ctas(x->grid), decode_is_dense(&bytes, 1, x->total_elems), s);
  CK(cudaGetLastError());
  return SYNC_OK;
}

int sync_decompress_apply(sync_ctx* x, const uint8_t* d_bucket, uint64_t bytes, uint16_t* const* d_weight_ptrs,
                          sync_stream_t stream) {
  ApiRange nvtx_range("sync_decompress_apply");
  if (!x || !d_bucket || !d_weight_ptrs) return SYNC_ERR_ARG;
  if (!aligned16(d_bucket)) return SYNC_ERR_ALIGNMENT;
  cudaStream_t s = (cudaStream_t)stream;
  const u32* bad;
  int st = maybe_crc_check(x, &d_bucket, &bytes, 1, s, &bad);
  if (st) return st;
  launch_decode(&d_bucket, &bytes, 1, x->d.T, x->plan.numel, d_weight_ptrs, nullptr, nullptr, nullptr, 0,
                x->plan.status, bad, x->plan.dtype, clamp_ctas(x->grid), decode_is_dense(&bytes, 1, x->total_elems), s);
  CK(cudaGetLastError());
  return SYNC_OK;
}

int sync_decompress_apply_batched(sync_ctx* x, const uint8_t* const* h_buckets, const uint64_t* h_bytes,
                                  uint32_t n_buckets, uint16_t* const* d_weight_ptrs, sync_stream_t stream) {
  ApiRange nvtx_range("sync_decompress_apply_batched");
  if (!x || !d_weight_ptrs || (n_buckets && (!h_buckets || !h_bytes))) return SYNC_ERR_ARG;
  for (u32 i = 0; i < n_buckets; ++i)
    if (!h_buckets[i] || !aligned16(h_buckets[i])) return h_buckets[i] ? SYNC_ERR_ALIGNMENT : SYNC_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const bool dense = decode_is_dense(h_bytes, n_buckets, x->total_elems);
  for (u32 b0 = 0; b0 < n_buckets; b0 += kCrcFlagSlots) {
    const u32 n = n_buckets - b0 < kCrcFlagSlots ? n_buckets - b0 : kCrcFlagSlots;
    const u32* bad;
    int st = maybe_crc_check(x, h_buckets + b0, h_bytes + b0, n, s, &bad);
    if (st) return st;
    launch_decode(h_buckets + b0, h_bytes + b0, n, x->d.T, x->plan.numel, d_weight_ptrs, nullptr, nullptr,
                  nullptr, 0, x->plan.status, bad, x->plan.dtype, clamp_ctas(x->grid), dense, s);
  }
  CK(cudaGetLastError());
  return SYNC_OK;
}

int sync_pack_table(sync_ctx* x, const uint64_t** d_hdr, const uint64_t** d_off, const uint64_t** d_size,
                    uint32_t* stride) {
  if (!x || !d_hdr || !d_off || !d_size || !stride) return SYNC_ERR_ARG;
  // the plan's device-resident copy (workspace): the count in the totals, the bucket descriptors' base / bytes
  // (the mapped host table would cost every decode CTA a round trip to host memory)
  const BucketDesc* bks = reinterpret_cast<const BucketDesc*>(x->ws + x->L.bks);
  *d_hdr = x->plan.totals + kTotBuckets;
  *d_off = &bks[0].base;
  *d_size = &bks[0].bytes;
  *stride = sizeof(BucketDesc) / 8;
  return SYNC_OK;
}

int sync_decompress_apply_table(sync_ctx* x, const uint8_t* d_base, const uint64_t* d_hdr, const uint64_t* d_off,
                                const uint64_t* d_size, uint32_t stride, uint32_t max_buckets,
                                uint16_t* const* d_weight_ptrs, uint32_t flags, sync_stream_t stream) {
  ApiRange nvtx_range("sync_decompress_apply_table");
  if (!x || !d_base || !d_hdr || !d_off || !d_size || !d_weight_ptrs || !stride) return SYNC_ERR_ARG;
  if (x->cfg.flags & SYNC_FLAG_CRC) return SYNC_ERR_ARG;   // table mode has no host sizes for the CRC pass
  if (!aligned16(d_base)) return SYNC_ERR_ALIGNMENT;
  launch_decode_table(d_hdr, d_off, d_size, stride, d_base, max_buckets, x->d.T, x->plan.numel, d_weight_ptrs,
                      x->plan.status, x->plan.dtype, clamp_ctas(x->grid), (flags & 1u) != 0,
                      (cudaStream_t)stream);
  CK(cudaGetLastError());
  return SYNC_OK;
}

// ------------------------------------------------------------------------ apply / commit
int sync_apply(uint16_t* d_W, const uint32_t* d_I, const uint16_t* d_V, uint64_t count, uint64_t numel,
               uint32_t* d_status, sync_stream_t stream) {
  ApiRange nvtx_range("sync_apply");
  if (count && (!d_W || !d_I || !d_V)) return SYNC_ERR_ARG;
  if (numel >= (1ull << 31)) return SYNC_ERR_ARG;
  if (!aligned16(d_W) || !aligned16(d_I) || !aligned16(d_V)) return SYNC_ERR_ALIGNMENT;
  launch_apply(d_W, d_I, d_V, count, numel, d_status, (cudaStream_t)stream);
  CK(cudaGetLastError());
  return SYNC_OK;
}

int sync_commit_snapshot(uint16_t* d_snapshot, const uint32_t* d_I, const uint16_t* d_V, uint64_t count,
                         uint64_t numel, uint32_t* d_status, sync_stream_t stream) {
  ApiRange nvtx_range("sync_commit_snapshot");
  return sync_apply(d_snapshot, d_I, d_V, count, numel, d_status, stream);
}

int sync_commit_snapshot_batched(sync_ctx* x, uint16_t* const* d_snapshot_ptrs, const uint32_t* d_I,
                                 const uint16_t* d_V, const uint64_t* d_counts, sync_stream_t stream) {
  ApiRange nvtx_range("sync_commit_snapshot_batched");
  if (!x || (x->d.T && (!d_snapshot_ptrs || !d_counts))) return SYNC_ERR_ARG;
  if (!aligned16(d_I) || !aligned16(d_V)) return SYNC_ERR_ALIGNMENT;   // the header's I / V contract
  if (x->d.T == 0) return SYNC_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (!(x->plan_valid && x->plan_counts == d_counts)) {
    launch_plan_scan(x->plan, d_counts, s);
    x->plan_valid = false;
  }
  launch_commit_batched(x->plan, d_snapshot_ptrs, d_I, d_V, clamp_ctas(x->grid), s);
  CK(cudaGetLastError());
  return SYNC_OK;
}

// ------------------------------------------------------------------------ status
int sync_status(sync_ctx* x, sync_stream_t stream) {
  if (!x) return SYNC_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  u32 v = 0;
  CK(cudaStreamSynchronize(s));
  CK(cudaMemcpy(&v, x->misc + 1, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemset(x->misc + 1, 0, 4));
  return -(int)v;
}

int sync_ctx_stats(sync_ctx* x, sync_stats* out, sync_stream_t stream) {
  if (!x || !out) return SYNC_ERR_ARG;
  u64 t[16];
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  CK(cudaMemcpy(t, x->plan.totals, sizeof(t), cudaMemcpyDeviceToHost));
  out->nnz = t[kTotNnz];
  out->n_records = t[kTotRecords];
  out->n_delta16 = t[kTotDelta16];
  out->n_abs32 = t[kTotAbs32];
  out->n_chunks = t[kTotChunks];
  out->n_chunks_rans = t[kTotRansChunks];
  out->enc_bytes = t[kTotEnc];
  out->index_bytes = t[kTotIndexBytes];
  out->value_bytes = t[kTotValueBytes];
  out->n_full = t[kTotFull];
  out->n_delta16e = t[kTotDelta16E];
  return SYNC_OK;
}

const char* sync_strerror(int status) {
  switch (status) {
    case SYNC_OK: return "ok";
    case SYNC_ERR_ARG: return "bad argument";
    case SYNC_ERR_ALIGNMENT: return "device pointer not 16-byte aligned";
    case SYNC_ERR_DTYPE: return "unsupported dtype (BF16 only)";
    case SYNC_ERR_WORKSPACE: return "workspace too small";
    case SYNC_ERR_CUDA: return "CUDA runtime error";
    case SYNC_ERR_INDEX_RANGE: return "index out of range";
    case SYNC_ERR_CAPACITY: return "output capacity exceeded";
    case SYNC_ERR_CORRUPT: return "corrupt record or rANS stream";
    case SYNC_ERR_BAD_MAGIC: return "bad bucket magic";
    case SYNC_ERR_VERSION: return "unsupported bucket version";
    case SYNC_ERR_TRUNCATED: return "truncated bucket";
    case SYNC_ERR_CRC: return "CRC-32 mismatch";
    default: return "unknown status";
  }
}

uint64_t sync_launch_count(void) { return g_launches.load(); }

int sync_set_max_ctas(int max_ctas) {
  if (max_ctas < 0) return SYNC_ERR_ARG;
  g_max_ctas.store(max_ctas, std::memory_order_relaxed);
  return SYNC_OK;
}

}  // extern "C"
