/*
 * oracle/sparsesync_oracle.c — plain, slow, obviously-correct CPU oracle of the
 * SparseRL-Sync hot path (arxiv 2605.07330).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this file's library. It shares
 * no code, header, table or constant generator with the CUDA path
 * (paper_2605_07330_b200/csrc) and neither side includes the other.
 *
 * Every function follows a passage of PAPER.md (P:n = line n) or the wire
 * format of DESIGN.md §3, step by step, with scalar loops and no blocking,
 * fusion or reordering.
 *
 * Pins (tests/test_oracle_*.py): SPEC examples, hand-derived rANS golden
 * vectors (tests/golden/), CRC-32 check value and zlib, round-trip identities,
 * exact Eq. (1) payload identity, entropy bounds.
 * Parity status: extract/apply, index codec (incl. f4 escapes), bucketing, f1 cast
 * tracking, f3 FULL routing and the f2 FP16/FP8 tags and layouts are pinned; the exact
 * rANS byte string is pinned only by FORMAT + hand golden vectors
 * (the paper fixes no coder).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_C 16384u           /* values per chunk */
#define OR_M 4096u            /* rANS total frequency, 12 bits */
#define OR_LOW 65536u         /* rANS lower bound 2^16 */
#define OR_LANES 32u

#define OR_OK 0
#define OR_ERR_INDEX_RANGE -6
#define OR_ERR_CAPACITY -7
#define OR_ERR_CORRUPT -8
#define OR_ERR_BAD_MAGIC -9
#define OR_ERR_VERSION -10
#define OR_ERR_TRUNCATED -11
#define OR_ERR_CRC -12
#define OR_ERR_ARG -1

enum { OR_DELTA16 = 0, OR_ABS32 = 1 };
enum { OR_CODEC_RAW = 0, OR_CODEC_COMPRESSED = 1 };
enum { OR_CHUNK_RAW = 0, OR_CHUNK_RANS = 1 };
/* record dtype byte (f2): the 16-bit element types share every encoding; only the tag differs */
enum { OR_DTYPE_BF16 = 1, OR_DTYPE_FP16 = 2, OR_DTYPE_FP8 = 3 };
/* FP8 E4M3 (f2): 8-bit elements. V arrays stay u16 with the byte in the low half;
 * a record has one value plane (the byte itself, rANS-coded per chunk, no lo plane); RAW records carry
 * u8 values; FULL records one byte per element. */
static int is8(int dtype) { return dtype == OR_DTYPE_FP8; }

static uint64_t pad_to(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

static void put16(uint8_t* p, uint16_t v) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); }
static void put32(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24);
}
static void put64(uint8_t* p, uint64_t v) { put32(p, (uint32_t)v); put32(p + 4, (uint32_t)(v >> 32)); }
static uint16_t get16(const uint8_t* p) { return (uint16_t)(p[0] | (p[1] << 8)); }
static uint32_t get32(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
static uint64_t get64(const uint8_t* p) { return (uint64_t)get32(p) | ((uint64_t)get32(p + 4) << 32); }

/* ---------------------------------------------------------------------------
 * a1 extract — Alg. 1 l.6: I_t = { i | W^(i) != W_prev^(i) }, compared
 * bitwise (DESIGN C1); Alg. 2 l.5: V = U[I]. Ascending i ("sorted").
 * I or V may be NULL to only count.
 * ------------------------------------------------------------------------- */
uint64_t or_extract(const uint16_t* old_bits, const uint16_t* new_bits, uint64_t n,
                    uint32_t* I, uint16_t* V) {
  uint64_t count = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (old_bits[i] != new_bits[i]) {
      if (I) I[count] = (uint32_t)i;
      if (V) V[count] = new_bits[i];
      ++count;
    }
  }
  return count;
}

/* ---------------------------------------------------------------------------
 * f1 cast-fused tracking — Alg. 1, the paper's own hook.
 *
 * or_bf16_rne: round_BF16 of CastAndCopy (Alg. 1 l.5) on the fp32 bit
 * pattern: round to nearest, ties to even, by adding 0x7FFF + lsb and keeping
 * the top 16 bits; NaN -> 0x7FC0 (DESIGN C18: the cast the PyTorch/Megatron
 * training stack performs). Overflow rounds to +-Inf by the same addition.
 * ------------------------------------------------------------------------- */
uint16_t or_bf16_rne(uint32_t f) {
  if (((f >> 23) & 0xFFu) == 0xFFu && (f & 0x7FFFFFu) != 0) return 0x7FC0;
  uint32_t lsb = (f >> 16) & 1u;
  return (uint16_t)((f + 0x7FFFu + lsb) >> 16);
}

void or_bf16_rne_array(const uint32_t* f, uint16_t* out, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) out[i] = or_bf16_rne(f[i]);
}

/* One optimizer-step epilogue for one tensor (Alg. 1 l.4-7):
 *   W_prev <- W; W <- round_BF16(W_main); I_t = { i | W^(i) != W_prev^(i) } (bitwise, C1);
 *   cumulative set: tracked[i] |= [i in I_t]   (tracked: one byte per element, 0/1).
 * Returns |I_t|.                                                            */
uint64_t or_cast_track(const uint32_t* master_bits, uint16_t* W, uint8_t* tracked, uint64_t n) {
  uint64_t changed = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint16_t w_prev = W[i];
    uint16_t w = or_bf16_rne(master_bits[i]);
    W[i] = w;
    if (w != w_prev) {
      tracked[i] = 1;
      ++changed;
    }
  }
  return changed;
}

/* Sync point on the tracked set (Alg. 2 l.4-5): I = ascending { i | tracked[i] },
 * V = W[I] (the current values, so a superset still reconstructs W bit-exactly); the set is
 * cleared for the next interval (Alg. 1 l.1, I_0 = {} ). Returns |I|; I/V may be NULL to only count. */
uint64_t or_extract_tracked(const uint16_t* W, uint8_t* tracked, uint64_t n, uint32_t* I, uint16_t* V) {
  uint64_t count = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (tracked[i]) {
      if (I) I[count] = (uint32_t)i;
      if (V) V[count] = W[i];
      ++count;
      tracked[i] = 0;
    }
  }
  return count;
}

/* 8-bit elements (FP8, f2): the same definitions on bytes; V holds the byte in the low half. */
uint64_t or_extract8(const uint8_t* old_bits, const uint8_t* new_bits, uint64_t n, uint32_t* I, uint16_t* V) {
  uint64_t count = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (old_bits[i] != new_bits[i]) {
      if (I) I[count] = (uint32_t)i;
      if (V) V[count] = new_bits[i];
      ++count;
    }
  }
  return count;
}

int or_apply8(uint8_t* W, uint64_t numel, const uint32_t* I, const uint16_t* V, uint64_t count) {
  int status = OR_OK;
  for (uint64_t k = 0; k < count; ++k) {
    if ((uint64_t)I[k] >= numel) { status = OR_ERR_INDEX_RANGE; continue; }
    W[I[k]] = (uint8_t)V[k];
  }
  return status;
}

/* ---------------------------------------------------------------------------
 * a8/a9 apply / commit — Alg. 3 l.6: W[I] <- V. Indices >= numel are
 * skipped and reported (S:327 IndexOutOfRange); all valid ones are written.
 * ------------------------------------------------------------------------- */
int or_apply(uint16_t* W, uint64_t numel, const uint32_t* I, const uint16_t* V, uint64_t count) {
  int status = OR_OK;
  for (uint64_t k = 0; k < count; ++k) {
    if ((uint64_t)I[k] >= numel) { status = OR_ERR_INDEX_RANGE; continue; }
    W[I[k]] = V[k];
  }
  return status;
}

/* ---------------------------------------------------------------------------
 * a2/a3 index mode — §3.3: first differences with a prepended zero;
 * DELTA16 iff every difference (incl. the first, = I_0) fits in int16, i.e.
 * <= 32767 (DESIGN C3/C4); else ABS32.
 * ------------------------------------------------------------------------- */
int or_index_mode(const uint32_t* I, uint64_t nnz) {
  uint32_t prev = 0;
  for (uint64_t k = 0; k < nnz; ++k) {
    uint32_t delta = I[k] - prev;
    if (delta > 32767u) return OR_ABS32;
    prev = I[k];
  }
  return OR_DELTA16;
}

/* Writes the index stream (unpadded); returns its byte length. */
uint64_t or_encode_indices(const uint32_t* I, uint64_t nnz, int mode, uint8_t* out) {
  if (mode == OR_DELTA16) {
    uint32_t prev = 0;
    for (uint64_t k = 0; k < nnz; ++k) {
      put16(out + 2 * k, (uint16_t)(I[k] - prev));
      prev = I[k];
    }
    return 2 * nnz;
  }
  for (uint64_t k = 0; k < nnz; ++k) put32(out + 4 * k, I[k]);
  return 4 * nnz;
}

/* ---------------------------------------------------------------------------
 * f4 escape-coded DELTA16 (P:360 keeps int32 whenever a gap
 * does not fit — for clustered masks that is every record). DELTA16E (idx_mode 3,
 * DESIGN §3.6): per element one u16 word Δ_k when Δ_k <= 32767, else two words
 * (0x8000 | Δ_k >> 16), (Δ_k & 0xFFFF) — an escape. Δ_0 = I_0 as in DELTA16.
 * ------------------------------------------------------------------------- */
enum { OR_DELTA16E = 3 };

uint64_t or_count_escapes(const uint32_t* I, uint64_t nnz) {
  uint64_t e = 0;
  uint32_t prev = 0;
  for (uint64_t k = 0; k < nnz; ++k) {
    if (I[k] - prev > 32767u) ++e;
    prev = I[k];
  }
  return e;
}

/* Mode with the escape option (flags bit 2): DELTA16 if no gap escapes; else DELTA16E when its stream
 * (2 (nnz + escapes) bytes) is smaller than ABS32's (4 nnz), i.e. escapes < nnz; else ABS32. */
int or_index_mode_escape(const uint32_t* I, uint64_t nnz) {
  uint64_t e = or_count_escapes(I, nnz);
  if (e == 0) return OR_DELTA16;
  return e < nnz ? OR_DELTA16E : OR_ABS32;
}

uint64_t or_encode_indices_escape(const uint32_t* I, uint64_t nnz, uint8_t* out) {
  uint64_t w = 0;
  uint32_t prev = 0;
  for (uint64_t k = 0; k < nnz; ++k) {
    uint32_t d = I[k] - prev;
    prev = I[k];
    if (d <= 32767u) {
      put16(out + 2 * w++, (uint16_t)d);
    } else {
      put16(out + 2 * w++, (uint16_t)(0x8000u | (d >> 16)));
      put16(out + 2 * w++, (uint16_t)(d & 0xFFFFu));
    }
  }
  return 2 * w;
}

/* Inverse of or_encode_indices_escape; returns the words consumed, or UINT64_MAX if the stream (words
 * available) ends inside an element. */
uint64_t or_decode_indices_escape(const uint8_t* in, uint64_t words, uint64_t nnz, uint32_t* I) {
  uint64_t w = 0;
  uint32_t acc = 0;
  for (uint64_t k = 0; k < nnz; ++k) {
    if (w >= words) return UINT64_MAX;
    uint16_t a = get16(in + 2 * w++);
    uint32_t d = a;
    if (a & 0x8000u) {
      if (w >= words) return UINT64_MAX;
      d = ((uint32_t)(a & 0x7FFFu) << 16) | get16(in + 2 * w++);
    }
    acc += d;
    I[k] = acc;
  }
  return w;
}

/* Inverse: DELTA16 running sum from 0; ABS32 copy. */
void or_decode_indices(const uint8_t* in, uint64_t nnz, int mode, uint32_t* I) {
  if (mode == OR_DELTA16) {
    uint32_t acc = 0;
    for (uint64_t k = 0; k < nnz; ++k) {
      acc += get16(in + 2 * k);
      I[k] = acc;
    }
    return;
  }
  for (uint64_t k = 0; k < nnz; ++k) I[k] = get32(in + 4 * k);
}

/* ---------------------------------------------------------------------------
 * a4 value entropy coding — §3.3 "Value entropy coding"; coder fixed by
 * DESIGN C6 / §3.3: frequency normalisation to M = 4096.
 * ------------------------------------------------------------------------- */
void or_normalize_freqs(const uint32_t counts[256], uint32_t n, uint32_t freq[256]) {
  uint32_t sum = 0;
  for (int s = 0; s < 256; ++s) {
    if (counts[s] == 0) {
      freq[s] = 0;
    } else {
      uint64_t f = (uint64_t)counts[s] * OR_M / n;
      freq[s] = f < 1 ? 1u : (uint32_t)f;
    }
    sum += freq[s];
  }
  if (sum < OR_M) {
    int best = -1;
    for (int s = 0; s < 256; ++s)
      if (counts[s] > 0 && (best < 0 || counts[s] > counts[best])) best = s;
    freq[best] += OR_M - sum;
    sum = OR_M;
  }
  while (sum > OR_M) {
    int best = -1;
    for (int s = 0; s < 256; ++s)
      if (freq[s] > 1 && (best < 0 || freq[s] > freq[best])) best = s;
    freq[best] -= 1;
    sum -= 1;
  }
}

/* Encodes n (1..C) hi bytes as a RANS block. Writes the block
 * (unpadded) to out and returns hi_bytes = 136 + 4*nsym + 2*nwords.
 * out must hold 136 + 1024 + 2*n bytes. */
uint32_t or_rans_encode(const uint8_t* hi, uint32_t n, uint8_t* out) {
  uint32_t counts[256] = {0}, freq[256], cum[256];
  for (uint32_t p = 0; p < n; ++p) counts[hi[p]]++;
  or_normalize_freqs(counts, n, freq);
  uint32_t c = 0;
  for (int s = 0; s < 256; ++s) { cum[s] = c; c += freq[s]; }

  uint32_t x[OR_LANES];
  for (uint32_t j = 0; j < OR_LANES; ++j) x[j] = OR_LOW;
  uint16_t* words = (uint16_t*)malloc(sizeof(uint16_t) * (n + 1));
  uint32_t nwords = 0;
  uint32_t G = (n + OR_LANES - 1) / OR_LANES;
  for (int64_t g = (int64_t)G - 1; g >= 0; --g) {
    for (uint32_t j = 0; j < OR_LANES; ++j) {
      uint64_t p = (uint64_t)g * OR_LANES + j;
      if (p >= n) continue;
      uint32_t s = hi[p];
      if ((uint64_t)x[j] >= ((uint64_t)freq[s] << 20)) {
        words[nwords++] = (uint16_t)(x[j] & 0xFFFFu);
        x[j] >>= 16;
      }
      x[j] = (x[j] / freq[s]) * OR_M + (x[j] % freq[s]) + cum[s];
    }
  }
  uint32_t nsym = 0;
  for (int s = 0; s < 256; ++s) nsym += freq[s] ? 1u : 0u;

  uint8_t* o = out;
  for (uint32_t j = 0; j < OR_LANES; ++j) put32(o + 4 * j, x[j]);
  o += 4 * OR_LANES;
  put32(o, nwords); o += 4;
  put16(o, (uint16_t)nsym); put16(o + 2, 0); o += 4;
  for (int s = 0; s < 256; ++s) {
    if (!freq[s]) continue;
    put32(o, (uint32_t)s | (freq[s] << 16));
    o += 4;
  }
  for (uint32_t k = 0; k < nwords; ++k) put16(o + 2 * k, words[nwords - 1 - k]);
  free(words);
  return 136u + 4u * nsym + 2u * nwords;
}

/* Decodes a RANS block of hi_bytes bytes into n hi bytes. */
int or_rans_decode(const uint8_t* in, uint32_t hi_bytes, uint32_t n, uint8_t* hi) {
  if (hi_bytes < 136) return OR_ERR_CORRUPT;
  uint32_t x[OR_LANES];
  for (uint32_t j = 0; j < OR_LANES; ++j) x[j] = get32(in + 4 * j);
  uint32_t nwords = get32(in + 128);
  uint32_t nsym = get16(in + 132);
  if (nsym < 1 || nsym > 256) return OR_ERR_CORRUPT;
  if ((uint64_t)136 + 4ull * nsym + 2ull * nwords != hi_bytes) return OR_ERR_CORRUPT;
  uint32_t freq[256] = {0}, cum[256];
  int prev_sym = -1;
  uint32_t total = 0;
  for (uint32_t k = 0; k < nsym; ++k) {
    uint32_t e = get32(in + 136 + 4 * k);
    int s = (int)(e & 0xFFFFu);
    uint32_t f = e >> 16;
    if (s > 255 || s <= prev_sym || f == 0) return OR_ERR_CORRUPT;
    freq[s] = f;
    prev_sym = s;
    total += f;
  }
  if (total != OR_M) return OR_ERR_CORRUPT;
  uint32_t c = 0;
  for (int s = 0; s < 256; ++s) { cum[s] = c; c += freq[s]; }
  const uint8_t* wp = in + 136 + 4 * nsym;

  for (uint32_t j = 0; j < OR_LANES; ++j)
    if (x[j] < OR_LOW) return OR_ERR_CORRUPT;
  uint32_t ptr = 0;
  uint32_t G = (n + OR_LANES - 1) / OR_LANES;
  for (uint32_t g = 0; g < G; ++g) {
    for (uint32_t j = 0; j < OR_LANES; ++j) {
      uint64_t p = (uint64_t)g * OR_LANES + j;
      if (p >= n) continue;
      uint32_t slot = x[j] & (OR_M - 1);
      int s = 0;
      while (!(cum[s] <= slot && slot < cum[s] + freq[s])) ++s;   /* the unique s */
      hi[p] = (uint8_t)s;
      x[j] = freq[s] * (x[j] >> 12) + slot - cum[s];
    }
    for (int j = (int)OR_LANES - 1; j >= 0; --j) {
      uint64_t p = (uint64_t)g * OR_LANES + (uint32_t)j;
      if (p >= n) continue;
      if (x[j] < OR_LOW) {
        if (ptr >= nwords) return OR_ERR_CORRUPT;
        x[j] = (x[j] << 16) | get16(wp + 2 * ptr);
        ++ptr;
      }
    }
  }
  for (uint32_t j = 0; j < OR_LANES; ++j)
    if (x[j] != OR_LOW) return OR_ERR_CORRUPT;
  if (ptr != nwords) return OR_ERR_CORRUPT;
  return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Records (DESIGN §3.1/§3.2) — Alg. 2 l.6-8: per parameter,
 * OptionalEncode then (name, dtype, shape) metadata (name/shape via tensor_id).
 * ------------------------------------------------------------------------- */

/* Upper bound of one record's size (for buffer sizing). */
uint64_t or_record_bound(uint64_t nnz) {
  uint64_t chunks = (nnz + OR_C - 1) / OR_C;
  return 64 + 8 * nnz + chunks * (16 + 136 + 1024 + 16);
}

/* Encodes one record; returns record_bytes (multiple of 16). nnz >= 1. */
uint64_t or_encode_record_ex(uint32_t tensor_id, const uint32_t* I, const uint16_t* V, uint64_t nnz,
                             int codec, uint8_t* out, int dtype, int escape);
uint64_t or_encode_record(uint32_t tensor_id, const uint32_t* I, const uint16_t* V, uint64_t nnz,
                          int codec, uint8_t* out, int dtype) {
  return or_encode_record_ex(tensor_id, I, V, nnz, codec, out, dtype, 0);
}

/* escape != 0: the f4 DELTA16E option (flags bit 2). A DELTA16E record carries, between its header and its
 * index stream, (n_chunks + 1) x u32: the word offset of each chunk's first index word (so chunks decode
 * independently) and the stream's total word count (so the planes after it can be located). */
uint64_t or_encode_record_ex(uint32_t tensor_id, const uint32_t* I, const uint16_t* V, uint64_t nnz,
                             int codec, uint8_t* out, int dtype, int escape) {
  uint8_t* rec = out;
  uint64_t off = 16;
  if (codec == OR_CODEC_RAW) {
    for (uint64_t k = 0; k < nnz; ++k) put32(rec + off + 4 * k, I[k]);
    off += 4 * nnz;
    if (is8(dtype)) {
      for (uint64_t k = 0; k < nnz; ++k) rec[off + k] = (uint8_t)V[k];
      off += nnz;
    } else {
      for (uint64_t k = 0; k < nnz; ++k) put16(rec + off + 2 * k, V[k]);
      off += 2 * nnz;
    }
    uint64_t total = pad_to(off, 16);
    memset(rec + off, 0, total - off);
    put32(rec + 0, tensor_id);
    put32(rec + 4, (uint32_t)nnz);
    put32(rec + 8, (uint32_t)total);
    rec[12] = OR_ABS32; rec[13] = (uint8_t)dtype; rec[14] = OR_CODEC_RAW; rec[15] = 0;
    return total;
  }
  int mode = escape ? or_index_mode_escape(I, nnz) : or_index_mode(I, nnz);
  uint64_t n_chunks = (nnz + OR_C - 1) / OR_C;
  if (mode == OR_DELTA16E) {   /* word offset of each chunk's first index word, then the total */
    uint64_t w = 0;
    uint32_t prev = 0;
    for (uint64_t k = 0; k < nnz; ++k) {
      if (k % OR_C == 0) put32(rec + off + 4 * (k / OR_C), (uint32_t)w);
      w += (I[k] - prev > 32767u) ? 2 : 1;
      prev = I[k];
    }
    put32(rec + off + 4 * n_chunks, (uint32_t)w);
    off += 4 * (n_chunks + 1);
  }
  uint64_t ib = mode == OR_DELTA16E ? or_encode_indices_escape(I, nnz, rec + off)
                                    : or_encode_indices(I, nnz, mode, rec + off);
  memset(rec + off + ib, 0, pad_to(ib, 4) - ib);
  off += pad_to(ib, 4);
  if (!is8(dtype)) {   /* lo plane (16-bit elements only) */
    for (uint64_t k = 0; k < nnz; ++k) rec[off + k] = (uint8_t)(V[k] & 0xFFu);
    memset(rec + off + nnz, 0, pad_to(nnz, 4) - nnz);
    off += pad_to(nnz, 4);
  }
  uint64_t dir = off;
  off += 16 * n_chunks;
  uint8_t* hi = (uint8_t*)malloc(OR_C);
  for (uint64_t k = 0; k < n_chunks; ++k) {
    uint64_t p0 = k * OR_C;
    uint32_t nk = (uint32_t)((nnz - p0) < OR_C ? (nnz - p0) : OR_C);
    for (uint32_t p = 0; p < nk; ++p) hi[p] = is8(dtype) ? (uint8_t)V[p0 + p] : (uint8_t)(V[p0 + p] >> 8);
    uint32_t hb = or_rans_encode(hi, nk, rec + off);
    uint32_t chunk_mode = OR_CHUNK_RANS;
    if (hb >= nk) {                       /* never-expand */
      memcpy(rec + off, hi, nk);
      hb = nk;
      chunk_mode = OR_CHUNK_RAW;
    }
    uint32_t base = ((mode == OR_DELTA16 || mode == OR_DELTA16E) && k > 0) ? I[p0 - 1] : 0u;
    put32(rec + dir + 16 * k + 0, (uint32_t)off);
    put32(rec + dir + 16 * k + 4, hb);
    put32(rec + dir + 16 * k + 8, chunk_mode);
    put32(rec + dir + 16 * k + 12, base);
    memset(rec + off + hb, 0, pad_to(hb, 4) - hb);
    off += pad_to(hb, 4);
  }
  free(hi);
  uint64_t total = pad_to(off, 16);
  memset(rec + off, 0, total - off);
  put32(rec + 0, tensor_id);
  put32(rec + 4, (uint32_t)nnz);
  put32(rec + 8, (uint32_t)total);
  rec[12] = (uint8_t)mode; rec[13] = (uint8_t)dtype; rec[14] = OR_CODEC_COMPRESSED; rec[15] = 0;
  return total;
}

/* ---------------------------------------------------------------------------
 * f3 per-parameter routing — WeightUpdater: "parameters that change on
 * nearly every element each step are transmitted via a full-weight copy".
 * FULL record (idx_mode 2): header {tensor_id, nnz field = numel,
 * record_bytes, mode 2, dtype 1, codec} || numel x u16 LE current values || zero
 * pad to 16. Routing rule (DESIGN C19): a record goes FULL iff its FULL size is
 * strictly smaller than its sparse (I, V) record.
 * ------------------------------------------------------------------------- */
enum { OR_FULL = 2 };

uint64_t or_full_record_bytes(uint64_t numel) { return pad_to(16 + 2 * numel, 16); }
uint64_t or_full_record_bytes_dt(uint64_t numel, int dtype) {
  return pad_to(16 + (is8(dtype) ? 1 : 2) * numel, 16);
}

/* W: the tensor's current elements (u16, or u8 for FP8). */
uint64_t or_encode_full_record(uint32_t tensor_id, const void* Wv, uint64_t numel, int codec, uint8_t* out,
                               int dtype) {
  uint64_t total = or_full_record_bytes_dt(numel, dtype);
  uint64_t eb = is8(dtype) ? 1 : 2;
  if (is8(dtype)) memcpy(out + 16, Wv, numel);
  else for (uint64_t i = 0; i < numel; ++i) put16(out + 16 + 2 * i, ((const uint16_t*)Wv)[i]);
  memset(out + 16 + eb * numel, 0, total - 16 - eb * numel);
  put32(out + 0, tensor_id);
  put32(out + 4, (uint32_t)numel);
  put32(out + 8, (uint32_t)total);
  out[12] = OR_FULL; out[13] = (uint8_t)dtype; out[14] = (uint8_t)codec; out[15] = 0;
  return total;
}

/* Decodes one record (exact inverse, Alg. 3 l.5) into I, V
 * (nnz entries). Returns 0 or an error; *tensor_id and *nnz filled. */
int or_decode_record(const uint8_t* rec, uint64_t avail, uint32_t* tensor_id, uint64_t* nnz_out,
                     uint32_t* I, uint16_t* V, uint64_t cap) {
  if (avail < 16) return OR_ERR_TRUNCATED;
  uint32_t tid = get32(rec), nnz = get32(rec + 4), rb = get32(rec + 8);
  uint8_t mode = rec[12], dtype = rec[13], codec = rec[14];
  if (rb > avail || rb < 16 || (rb % 16) != 0) return OR_ERR_TRUNCATED;
  if ((dtype != OR_DTYPE_BF16 && dtype != OR_DTYPE_FP16 && dtype != OR_DTYPE_FP8) || mode > 3 || codec > 1 ||
      nnz == 0)
    return OR_ERR_CORRUPT;
  const uint64_t eb = is8(dtype) ? 1 : 2;
  *tensor_id = tid;
  *nnz_out = nnz;
  if (nnz > cap) return OR_ERR_CAPACITY;
  if (mode == OR_FULL) {                /* every element, in order */
    if (16 + eb * nnz > rb) return OR_ERR_CORRUPT;
    for (uint64_t k = 0; k < nnz; ++k) {
      I[k] = (uint32_t)k;
      V[k] = eb == 1 ? rec[16 + k] : get16(rec + 16 + 2 * k);
    }
    return OR_OK;
  }
  if (codec == OR_CODEC_RAW) {
    if (mode != OR_ABS32 || 16 + (4 + eb) * nnz > rb) return OR_ERR_CORRUPT;
    for (uint64_t k = 0; k < nnz; ++k) I[k] = get32(rec + 16 + 4 * k);
    for (uint64_t k = 0; k < nnz; ++k)
      V[k] = eb == 1 ? rec[16 + 4ull * nnz + k] : get16(rec + 16 + 4ull * nnz + 2 * k);
    return OR_OK;
  }
  uint64_t off = 16;
  uint64_t n_chunks = (nnz + OR_C - 1) / OR_C;
  uint64_t ib;
  const uint8_t* table = NULL;
  if (mode == OR_DELTA16E) {
    if (off + 4 * (n_chunks + 1) > rb) return OR_ERR_CORRUPT;
    table = rec + off;
    off += 4 * (n_chunks + 1);
    uint64_t total = get32(table + 4 * n_chunks);
    if (total < nnz || total > 2ull * nnz || off + 2 * total > rb) return OR_ERR_CORRUPT;
    if (or_decode_indices_escape(rec + off, total, nnz, I) != total) return OR_ERR_CORRUPT;
    ib = 2 * total;
  } else {
    ib = (mode == OR_DELTA16 ? 2ull : 4ull) * nnz;
  }
  const uint64_t lo_bytes = eb == 1 ? 0 : pad_to(nnz, 4);   /* no lo plane for 8-bit elements */
  if (off + pad_to(ib, 4) + lo_bytes + 16 * n_chunks > rb) return OR_ERR_CORRUPT;
  if (mode != OR_DELTA16E) or_decode_indices(rec + off, nnz, mode, I);
  if (table) {   /* the chunk word offsets must match the stream */
    uint64_t w = 0;
    uint32_t prev = 0;
    for (uint64_t k = 0; k < nnz; ++k) {
      if (k % OR_C == 0 && get32(table + 4 * (k / OR_C)) != w) return OR_ERR_CORRUPT;
      w += (I[k] - prev > 32767u) ? 2 : 1;
      prev = I[k];
    }
  }
  off += pad_to(ib, 4);
  const uint8_t* lo = rec + off;
  off += lo_bytes;
  const uint8_t* dir = rec + off;
  uint8_t* hi = (uint8_t*)malloc(OR_C);
  int st = OR_OK;
  for (uint64_t k = 0; k < n_chunks && st == OR_OK; ++k) {
    uint64_t p0 = k * OR_C;
    uint32_t nk = (uint32_t)((nnz - p0) < OR_C ? (nnz - p0) : OR_C);
    uint32_t ho = get32(dir + 16 * k), hb = get32(dir + 16 * k + 4), cm = get32(dir + 16 * k + 8);
    uint32_t base = get32(dir + 16 * k + 12);
    uint32_t expect_base = ((mode == OR_DELTA16 || mode == OR_DELTA16E) && k > 0) ? I[p0 - 1] : 0u;
    if (base != expect_base || (uint64_t)ho + hb > rb) { st = OR_ERR_CORRUPT; break; }
    if (cm == OR_CHUNK_RAW) {
      if (hb != nk) { st = OR_ERR_CORRUPT; break; }
      memcpy(hi, rec + ho, nk);
    } else if (cm == OR_CHUNK_RANS) {
      st = or_rans_decode(rec + ho, hb, nk, hi);
    } else {
      st = OR_ERR_CORRUPT;
    }
    for (uint32_t p = 0; p < nk && st == OR_OK; ++p)
      V[p0 + p] = eb == 1 ? hi[p] : (uint16_t)(((uint16_t)hi[p] << 8) | lo[p0 + p]);
  }
  free(hi);
  return st;
}

/* ---------------------------------------------------------------------------
 * CRC-32/IEEE (reflected 0xEDB88320, init/xorout 0xFFFFFFFF), bitwise.
 * ------------------------------------------------------------------------- */
uint32_t or_crc32(const uint8_t* data, uint64_t n) {
  uint32_t crc = 0xFFFFFFFFu;
  for (uint64_t i = 0; i < n; ++i) {
    crc ^= data[i];
    for (int b = 0; b < 8; ++b) crc = (crc >> 1) ^ (0xEDB88320u & (0u - (crc & 1u)));
  }
  return crc ^ 0xFFFFFFFFu;
}

/* ---------------------------------------------------------------------------
 * a5 bucketing (DESIGN C11): greedy over record sizes.
 * bucket_of[r] receives the bucket index; returns the number of buckets.
 * ------------------------------------------------------------------------- */
static uint64_t bucket_size(uint64_t n_rec, uint64_t rec_bytes_sum) {
  return 32 + pad_to(8 * n_rec, 16) + rec_bytes_sum;
}

uint32_t or_bucketize(const uint64_t* rec_bytes, uint64_t n_records, uint64_t limit, uint32_t* bucket_of) {
  uint32_t b = 0;
  uint64_t n_in = 0, sum = 0;
  for (uint64_t r = 0; r < n_records; ++r) {
    if (n_in > 0 && bucket_size(n_in + 1, sum + rec_bytes[r]) > limit) {
      ++b;
      n_in = 0;
      sum = 0;
    }
    bucket_of[r] = b;
    ++n_in;
    sum += rec_bytes[r];
  }
  return n_records ? b + 1 : 0;
}

/* ---------------------------------------------------------------------------
 * Whole sender path: Alg. 2 over a manifest, with extract (Alg. 1
 * l.6) per tensor, in manifest order. Writes buckets into out (bucket b at
 * offsets[b], 256-aligned), sizes[b]. Returns n_buckets or a negative error.
 * stats (may be NULL): [0] total nnz, [1] n_records, [2] delta16 records,
 * [3] abs32 records, [4] payload bytes (Σ bucket bytes), [5] value-stream bytes,
 * [6] FULL records (flags bit 1 = routing, f3), [7] DELTA16E records (flags bit 2 = escapes, f4).
 * ------------------------------------------------------------------------- */
int64_t or_sync_pack(uint32_t n_tensors, const uint64_t* numel, const void* const* old_ptrs,
                     const void* const* new_ptrs, int codec, uint64_t limit, uint32_t flags,
                     uint8_t* out, uint64_t out_cap, uint64_t* offsets, uint64_t* sizes,
                     uint32_t max_buckets, uint64_t* stats, int dtype) {
  uint64_t st[8] = {0};
  /* 1. per tensor records into a scratch stream */
  uint64_t cap_total = 0;
  for (uint32_t t = 0; t < n_tensors; ++t) cap_total += or_record_bound(numel[t] ? numel[t] : 1);
  uint8_t* stream = (uint8_t*)malloc(cap_total ? cap_total : 16);
  uint64_t* rec_bytes = (uint64_t*)malloc(sizeof(uint64_t) * (n_tensors + 1));
  uint64_t* rec_pos = (uint64_t*)malloc(sizeof(uint64_t) * (n_tensors + 1));
  uint32_t* rec_chunks = (uint32_t*)malloc(sizeof(uint32_t) * (n_tensors + 1));
  uint64_t n_records = 0, pos = 0;
  for (uint32_t t = 0; t < n_tensors; ++t) {
    uint64_t n = numel[t];
    uint32_t* I = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    uint16_t* V = (uint16_t*)malloc(sizeof(uint16_t) * (n ? n : 1));
    uint64_t nnz = is8(dtype) ? or_extract8((const uint8_t*)old_ptrs[t], (const uint8_t*)new_ptrs[t], n, I, V)
                              : or_extract((const uint16_t*)old_ptrs[t], (const uint16_t*)new_ptrs[t], n, I, V);
    if (nnz > 0) {
      uint64_t rb = or_encode_record_ex(t, I, V, nnz, codec, stream + pos, dtype, (flags & 4u) != 0);
      int full = (flags & 2u) && or_full_record_bytes_dt(n, dtype) < rb;   /* routing, DESIGN C19 */
      if (full) rb = or_encode_full_record(t, new_ptrs[t], n, codec, stream + pos, dtype);
      rec_bytes[n_records] = rb;
      rec_pos[n_records] = pos;
      rec_chunks[n_records] = (uint32_t)(((full ? n : nnz) + OR_C - 1) / OR_C);
      ++n_records;
      pos += rb;
      st[0] += nnz;
      if (full) {
        st[6] += 1;
        st[5] += rb - 16;
      } else if (codec == OR_CODEC_COMPRESSED) {
        int mode = stream[pos - rb + 12];
        uint64_t ib = (mode == OR_ABS32 ? 4 : 2) * nnz;
        if (mode == OR_DELTA16E) {
          uint64_t e = 0;
          uint32_t prev = 0;
          for (uint64_t k = 0; k < nnz; ++k) { e += (I[k] - prev > 32767u); prev = I[k]; }
          ib = 2 * (nnz + e);
          st[7] += 1;
        } else {
          st[mode == OR_DELTA16 ? 2 : 3] += 1;
        }
        st[5] += rb - 16 - pad_to(ib, 4);
      } else {
        st[3] += 1;
        st[5] += (is8(dtype) ? 1 : 2) * nnz;
      }
    }
    free(I);
    free(V);
  }
  st[1] = n_records;
  /* 2. greedy bucketing */
  uint32_t* bucket_of = (uint32_t*)malloc(sizeof(uint32_t) * (n_records + 1));
  uint32_t nb = or_bucketize(rec_bytes, n_records, limit, bucket_of);
  int64_t ret = nb;
  if (nb > max_buckets) { ret = OR_ERR_CAPACITY; goto done; }
  /* 3. assemble buckets */
  {
    uint64_t r = 0, base = 0;
    for (uint32_t b = 0; b < nb; ++b) {
      uint64_t r0 = r, sum = 0, nch = 0;
      while (r < n_records && bucket_of[r] == b) { sum += rec_bytes[r]; nch += rec_chunks[r]; ++r; }
      uint64_t nr = r - r0;
      uint64_t bytes = bucket_size(nr, sum);
      base = pad_to(base, 256);
      if (base + bytes > out_cap) { ret = OR_ERR_CAPACITY; goto done; }
      uint8_t* bk = out + base;
      memset(bk, 0, 32 + pad_to(8 * nr, 16));
      uint64_t ro = 32 + pad_to(8 * nr, 16);
      uint32_t first_chunk = 0;
      for (uint64_t q = 0; q < nr; ++q) {
        put32(bk + 32 + 8 * q, (uint32_t)ro);
        put32(bk + 32 + 8 * q + 4, first_chunk);
        memcpy(bk + ro, stream + rec_pos[r0 + q], rec_bytes[r0 + q]);
        ro += rec_bytes[r0 + q];
        first_chunk += rec_chunks[r0 + q];
      }
      put32(bk + 0, 0x424C5253u);
      put16(bk + 4, 1);
      put16(bk + 6, (uint16_t)(flags & 1u));
      put32(bk + 8, b);
      put32(bk + 12, (uint32_t)nr);
      put32(bk + 16, (uint32_t)nch);
      put64(bk + 24, bytes);
      put32(bk + 20, (flags & 1u) ? or_crc32(bk + 32, bytes - 32) : 0u);
      offsets[b] = base;
      sizes[b] = bytes;
      st[4] += bytes;
      base += bytes;
    }
  }
done:
  if (stats) memcpy(stats, st, sizeof(st));
  free(stream); free(rec_bytes); free(rec_pos); free(rec_chunks); free(bucket_of);
  return ret;
}

/* ---------------------------------------------------------------------------
 * Receiver: Alg. 3 for one bucket — validate header (and CRC),
 * decode every record, scatter into weights[tensor_id]. Returns 0 or error.
 * ------------------------------------------------------------------------- */
/* weights: per-tensor element arrays (u16; u8 for records tagged FP8). */
int or_bucket_apply(const uint8_t* bk, uint64_t avail, uint32_t n_tensors, const uint64_t* numel,
                    void* const* weights) {
  if (avail < 32) return OR_ERR_TRUNCATED;
  if (get32(bk) != 0x424C5253u) return OR_ERR_BAD_MAGIC;
  if (get16(bk + 4) != 1) return OR_ERR_VERSION;
  uint16_t flags = get16(bk + 6);
  uint32_t nr = get32(bk + 12);
  uint64_t bytes = get64(bk + 24);
  if (bytes > avail || bytes < 32 + pad_to(8ull * nr, 16)) return OR_ERR_TRUNCATED;
  if ((flags & 1u) && or_crc32(bk + 32, bytes - 32) != get32(bk + 20)) return OR_ERR_CRC;
  int status = OR_OK;
  for (uint32_t q = 0; q < nr; ++q) {
    uint32_t ro = get32(bk + 32 + 8 * q);
    if (ro >= bytes) return OR_ERR_CORRUPT;
    uint32_t nnz_hdr = (bytes - ro >= 16) ? get32(bk + ro + 4) : 0;
    uint32_t* I = (uint32_t*)malloc(sizeof(uint32_t) * (nnz_hdr ? nnz_hdr : 1));
    uint16_t* V = (uint16_t*)malloc(sizeof(uint16_t) * (nnz_hdr ? nnz_hdr : 1));
    uint32_t tid;
    uint64_t nnz;
    int st = or_decode_record(bk + ro, bytes - ro, &tid, &nnz, I, V, nnz_hdr);
    if (st == OR_OK) {
      if (tid >= n_tensors) st = OR_ERR_CORRUPT;
      else if (bk[ro + 13] == OR_DTYPE_FP8) st = or_apply8((uint8_t*)weights[tid], numel[tid], I, V, nnz);
      else st = or_apply((uint16_t*)weights[tid], numel[tid], I, V, nnz);
    }
    free(I);
    free(V);
    if (st != OR_OK) status = st;
  }
  return status;
}

/* Receiver debug path: decode every record of a bucket into I/V arrays in
 * record order; rec_info[3*q] = tensor_id, [3*q+1] = nnz, [3*q+2] = out offset. */
int or_bucket_decode(const uint8_t* bk, uint64_t avail, uint32_t* I, uint16_t* V, uint64_t cap,
                     uint64_t* rec_info, uint32_t max_records, uint32_t* n_records) {
  if (avail < 32) return OR_ERR_TRUNCATED;
  if (get32(bk) != 0x424C5253u) return OR_ERR_BAD_MAGIC;
  if (get16(bk + 4) != 1) return OR_ERR_VERSION;
  uint16_t flags = get16(bk + 6);
  uint32_t nr = get32(bk + 12);
  uint64_t bytes = get64(bk + 24);
  if (bytes > avail || bytes < 32 + pad_to(8ull * nr, 16)) return OR_ERR_TRUNCATED;
  if ((flags & 1u) && or_crc32(bk + 32, bytes - 32) != get32(bk + 20)) return OR_ERR_CRC;
  if (nr > max_records) return OR_ERR_CAPACITY;
  uint64_t out = 0;
  for (uint32_t q = 0; q < nr; ++q) {
    uint32_t ro = get32(bk + 32 + 8 * q);
    if (ro >= bytes) return OR_ERR_CORRUPT;
    uint32_t tid;
    uint64_t nnz;
    int st = or_decode_record(bk + ro, bytes - ro, &tid, &nnz, I + out, V + out, cap - out);
    if (st != OR_OK) return st;
    rec_info[3 * q] = tid;
    rec_info[3 * q + 1] = nnz;
    rec_info[3 * q + 2] = out;
    out += nnz;
  }
  *n_records = nr;
  return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Cost model, Eq. (1)-(4): raw and compressed payload sizes and ratios.
 * ------------------------------------------------------------------------- */
double or_eq1_sparse_bytes(double rho, double N, double b_v, double b_i, double s_meta) {
  return rho * N * (b_v + b_i) + s_meta;                  /* Eq. (1) */
}
double or_eq2_ratio(double rho, double b_v, double b_i) {
  return b_v / (rho * (b_v + b_i));                        /* Eq. (2) */
}
double or_eq3_compressed_bytes(double rho, double N, double b_v, double b_i, double alpha) {
  return rho * N * (b_i + alpha * b_v);                    /* Eq. (3) */
}
double or_eq4_ratio(double rho, double b_v, double b_i, double alpha) {
  return b_v / (rho * (b_i + alpha * b_v));                /* Eq. (4) */
}
