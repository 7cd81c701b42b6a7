"""CPU oracle of the SparseRL-Sync hot path (arxiv 2605.07330).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package. The product path (``paper_2605_07330_b200``) never imports it and
shares no code with it.

Thin ctypes wrapper over ``oracle/sparsesync_oracle.c`` (plain scalar C, see its
header for the passage each function follows). Arrays are numpy.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sparsesync_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK = 0
ERR_INDEX_RANGE = -6
ERR_CAPACITY = -7
ERR_CORRUPT = -8
ERR_BAD_MAGIC = -9
ERR_VERSION = -10
ERR_TRUNCATED = -11
ERR_CRC = -12

DELTA16, ABS32 = 0, 1
DTYPE_BF16, DTYPE_FP16, DTYPE_FP8 = 1, 2, 3
DELTA16E = 3
CODEC_RAW, CODEC_COMPRESSED = 0, 1
CHUNK = 16384


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 (no tuning, no SIMD intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", _SRC, "-o", _LIB])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        u64, u32, i32, i64 = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_int64
        sig = {
            "or_extract": (u64, [P, P, u64, P, P]),
            "or_full_record_bytes": (u64, [u64]),
            "or_full_record_bytes_dt": (u64, [u64, i32]),
            "or_extract8": (u64, [P, P, u64, P, P]),
            "or_apply8": (i32, [P, u64, P, P, u64]),
            "or_encode_full_record": (u64, [u32, P, u64, i32, P, i32]),
            "or_bf16_rne": (ctypes.c_uint16, [u32]),
            "or_bf16_rne_array": (None, [P, P, u64]),
            "or_cast_track": (u64, [P, P, P, u64]),
            "or_extract_tracked": (u64, [P, P, u64, P, P]),
            "or_apply": (i32, [P, u64, P, P, u64]),
            "or_index_mode": (i32, [P, u64]),
            "or_encode_indices": (u64, [P, u64, i32, P]),
            "or_decode_indices": (None, [P, u64, i32, P]),
            "or_normalize_freqs": (None, [P, u32, P]),
            "or_rans_encode": (u32, [P, u32, P]),
            "or_rans_decode": (i32, [P, u32, u32, P]),
            "or_record_bound": (u64, [u64]),
            "or_encode_record": (u64, [u32, P, P, u64, i32, P, i32]),
            "or_encode_record_ex": (u64, [u32, P, P, u64, i32, P, i32, i32]),
            "or_count_escapes": (u64, [P, u64]),
            "or_index_mode_escape": (i32, [P, u64]),
            "or_encode_indices_escape": (u64, [P, u64, P]),
            "or_decode_indices_escape": (u64, [P, u64, u64, P]),
            "or_decode_record": (i32, [P, u64, P, P, P, P, u64]),
            "or_crc32": (u32, [P, u64]),
            "or_bucketize": (u32, [P, u64, u64, P]),
            "or_sync_pack": (i64, [u32, P, P, P, i32, u64, u32, P, u64, P, P, u32, P, i32]),
            "or_bucket_apply": (i32, [P, u64, u32, P, P]),
            "or_bucket_decode": (i32, [P, u64, P, P, u64, P, u32, P]),
            "or_eq1_sparse_bytes": (ctypes.c_double, [ctypes.c_double] * 5),
            "or_eq2_ratio": (ctypes.c_double, [ctypes.c_double] * 3),
            "or_eq3_compressed_bytes": (ctypes.c_double, [ctypes.c_double] * 5),
            "or_eq4_ratio": (ctypes.c_double, [ctypes.c_double] * 4),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a.size else None


def _u8(a) -> np.ndarray:
    a = np.asarray(a)
    return np.ascontiguousarray(a.view(np.uint8) if a.dtype != np.uint8 else a)


def _u16(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a).view(np.uint16) if np.asarray(a).dtype != np.uint16
                                else np.asarray(a))


# ----------------------------------------------------------------------------- a1
def extract(old: np.ndarray, new: np.ndarray):
    """Alg. 1 l.6 + Alg. 2 l.5: (I, V) of bitwise-changed elements."""
    old, new = _u16(old), _u16(new)
    assert old.shape == new.shape
    n = old.size
    I = np.empty(max(n, 1), np.uint32)
    V = np.empty(max(n, 1), np.uint16)
    c = lib().or_extract(_p(old), _p(new), n, _p(I), _p(V))
    return I[:c].copy(), V[:c].copy()


# ----------------------------------------------------------------------------- f1 cast-fused tracking
def bf16_rne(master: np.ndarray) -> np.ndarray:
    """Alg. 1 l.5 round_BF16 of fp32 masters (float32 array) -> uint16 bf16 bit patterns."""
    m = np.ascontiguousarray(np.ascontiguousarray(master, np.float32).view(np.uint32).reshape(-1))
    out = np.empty(m.size, np.uint16)
    lib().or_bf16_rne_array(_p(m), _p(out), m.size)
    return out


def cast_track(master: np.ndarray, W: np.ndarray, tracked: np.ndarray) -> int:
    """Alg. 1 l.4-7 on one tensor: W <- round_BF16(master) in place, tracked |= (W changed).
    master float32, W uint16 bits, tracked uint8 (0/1). Returns |I_t|."""
    m = np.ascontiguousarray(master, np.float32).view(np.uint32)
    assert W.dtype == np.uint16 and W.flags.c_contiguous and tracked.dtype == np.uint8
    assert m.size == W.size == tracked.size
    return int(lib().or_cast_track(_p(m), _p(W), _p(tracked), W.size))


def extract_tracked(W: np.ndarray, tracked: np.ndarray):
    """Alg. 2 l.4-5 on the tracked set: (I ascending, V = W[I]); clears tracked."""
    n = W.size
    I = np.empty(max(n, 1), np.uint32)
    V = np.empty(max(n, 1), np.uint16)
    c = lib().or_extract_tracked(_p(W), _p(tracked), n, _p(I), _p(V))
    return I[:c].copy(), V[:c].copy()


def extract8(old: np.ndarray, new: np.ndarray):
    """FP8 (f2): Alg. 1 l.6 + Alg. 2 l.5 on 8-bit elements: (I, V as uint16 holding the byte)."""
    old, new = _u8(old).ravel(), _u8(new).ravel()
    n = old.size
    I = np.empty(max(n, 1), np.uint32)
    V = np.empty(max(n, 1), np.uint16)
    c = lib().or_extract8(_p(old), _p(new), n, _p(I), _p(V))
    return I[:c].copy(), V[:c].copy()


# ----------------------------------------------------------------------------- a8/a9
def apply(W: np.ndarray, I: np.ndarray, V: np.ndarray) -> int:
    """Alg. 3 l.6: W[I] <- V in place (W uint16 bits). Returns status."""
    assert W.dtype == np.uint16 and W.flags.c_contiguous
    I = np.ascontiguousarray(I, np.uint32)
    V = np.ascontiguousarray(V, np.uint16)
    return lib().or_apply(_p(W), W.size, _p(I), _p(V), I.size)


# ----------------------------------------------------------------------------- a2/a3
def index_mode(I) -> int:
    I = np.ascontiguousarray(I, np.uint32)
    return lib().or_index_mode(_p(I), I.size)


def encode_indices(I, mode: int) -> bytes:
    I = np.ascontiguousarray(I, np.uint32)
    out = np.zeros(4 * I.size + 4, np.uint8)
    n = lib().or_encode_indices(_p(I), I.size, mode, _p(out))
    return out[:n].tobytes()


def decode_indices(b: bytes, nnz: int, mode: int) -> np.ndarray:
    buf = np.frombuffer(b, np.uint8).copy() if b else np.zeros(1, np.uint8)
    I = np.empty(max(nnz, 1), np.uint32)
    lib().or_decode_indices(_p(buf), nnz, mode, _p(I))
    return I[:nnz].copy()


# ----------------------------------------------------------------------------- a4
def normalize_freqs(counts) -> np.ndarray:
    counts = np.ascontiguousarray(counts, np.uint32)
    assert counts.size == 256
    f = np.zeros(256, np.uint32)
    lib().or_normalize_freqs(_p(counts), int(counts.sum()), _p(f))
    return f


def rans_encode(hi) -> bytes:
    hi = np.ascontiguousarray(hi, np.uint8)
    assert 1 <= hi.size <= CHUNK
    out = np.zeros(136 + 1024 + 2 * hi.size + 8, np.uint8)
    n = lib().or_rans_encode(_p(hi), hi.size, _p(out))
    return out[:n].tobytes()


def rans_decode(block: bytes, n: int):
    buf = np.frombuffer(block, np.uint8).copy()
    hi = np.zeros(n, np.uint8)
    st = lib().or_rans_decode(_p(buf), len(block), n, _p(hi))
    return st, hi


# ----------------------------------------------------------------------------- records
def encode_full_record(tensor_id: int, W, codec: int = CODEC_COMPRESSED, dtype: int = 1) -> bytes:
    """f3 FULL record: the whole tensor's current values (uint8 for FP8)."""
    W = (_u8(W) if dtype == DTYPE_FP8 else _u16(W)).ravel()
    out = np.zeros(int(lib().or_full_record_bytes_dt(W.size, dtype)), np.uint8)
    n = lib().or_encode_full_record(tensor_id, _p(W), W.size, codec, _p(out), dtype)
    return out[:n].tobytes()


def encode_indices_escape(I) -> bytes:
    """f4 DELTA16E index stream."""
    I = np.ascontiguousarray(I, np.uint32)
    out = np.zeros(4 * max(I.size, 1), np.uint8)
    n = lib().or_encode_indices_escape(_p(I), I.size, _p(out))
    return out[:n].tobytes()


def decode_indices_escape(stream: bytes, nnz: int):
    """Inverse; returns (I, words consumed) or (None, None) on a truncated stream."""
    buf = np.frombuffer(stream, np.uint8).copy()
    I = np.zeros(max(nnz, 1), np.uint32)
    w = lib().or_decode_indices_escape(_p(buf), len(stream) // 2, nnz, _p(I))
    if w == (1 << 64) - 1:
        return None, None
    return I[:nnz].copy(), int(w)


def encode_record(tensor_id: int, I, V, codec: int = CODEC_COMPRESSED, dtype: int = 1,
                  escape: bool = False) -> bytes:
    I = np.ascontiguousarray(I, np.uint32)
    V = np.ascontiguousarray(V, np.uint16)
    assert I.size == V.size and I.size > 0
    out = np.zeros(lib().or_record_bound(I.size), np.uint8)
    n = lib().or_encode_record_ex(tensor_id, _p(I), _p(V), I.size, codec, _p(out), dtype, 1 if escape else 0)
    return out[:n].tobytes()


def decode_record(rec: bytes):
    buf = np.frombuffer(rec, np.uint8).copy()
    cap = max(1, (len(rec) - 16))
    I = np.empty(cap, np.uint32)
    V = np.empty(cap, np.uint16)
    tid = ctypes.c_uint32()
    nnz = ctypes.c_uint64()
    st = lib().or_decode_record(_p(buf), len(rec), ctypes.byref(tid), ctypes.byref(nnz), _p(I), _p(V), cap)
    k = nnz.value if st == OK else 0
    return st, tid.value, I[:k].copy(), V[:k].copy()


def crc32(data: bytes) -> int:
    buf = np.frombuffer(data, np.uint8).copy() if data else np.zeros(1, np.uint8)
    return lib().or_crc32(_p(buf), len(data))


def bucketize(rec_bytes, limit: int):
    rb = np.ascontiguousarray(rec_bytes, np.uint64)
    out = np.zeros(max(rb.size, 1), np.uint32)
    nb = lib().or_bucketize(_p(rb), rb.size, limit, _p(out))
    return nb, out[: rb.size].copy()


# ----------------------------------------------------------------------------- whole path
class PackResult:
    def __init__(self, buf, offsets, sizes, stats):
        self.buf = buf
        self.offsets = offsets
        self.sizes = sizes
        self.stats = dict(zip(["nnz", "n_records", "delta16", "abs32", "payload_bytes", "value_bytes", "full",
                               "delta16e"],
                              [int(s) for s in stats]))

    @property
    def n_buckets(self):
        return len(self.sizes)

    def bucket(self, b: int) -> bytes:
        o, s = int(self.offsets[b]), int(self.sizes[b])
        return self.buf[o:o + s].tobytes()


def sync_pack(olds, news, codec: int = CODEC_COMPRESSED, limit: int = 256 << 20, crc: bool = False,
              max_buckets: int = 1 << 16, route: bool = False, dtype: int = 1,
              escape: bool = False) -> PackResult:
    """Sender path (Alg. 2) over a manifest of (old, new) uint16 arrays.
    route: per-parameter routing (f3) — a record goes FULL when that is smaller (DESIGN C19).
    escape: escape-coded DELTA16 (f4) for records with gaps > 32767."""
    conv = _u8 if dtype == DTYPE_FP8 else _u16   # FP8 (f2): 8-bit elements
    olds = [conv(o).ravel() for o in olds]
    news = [conv(n).ravel() for n in news]
    T = len(olds)
    numel = np.array([o.size for o in olds], np.uint64)
    keep = [np.zeros(1, o.dtype) if o.size == 0 else o for o in olds] + \
           [np.zeros(1, n.dtype) if n.size == 0 else n for n in news]
    op = (ctypes.c_void_p * max(T, 1))(*[k.ctypes.data for k in keep[:T]])
    np_ = (ctypes.c_void_p * max(T, 1))(*[k.ctypes.data for k in keep[T:]])
    L = lib()
    bound = sum(int(L.or_record_bound(max(int(n), 1))) for n in numel)
    cap = bound + 512 * (T + 2) + 4096
    buf = np.zeros(cap, np.uint8)
    offs = np.zeros(max_buckets, np.uint64)
    sizes = np.zeros(max_buckets, np.uint64)
    stats = np.zeros(8, np.uint64)
    flags = (1 if crc else 0) | (2 if route else 0) | (4 if escape else 0)
    nb = L.or_sync_pack(T, _p(numel), ctypes.cast(op, ctypes.c_void_p), ctypes.cast(np_, ctypes.c_void_p),
                        codec, limit, flags, _p(buf), cap, _p(offs), _p(sizes), max_buckets,
                        _p(stats), dtype)
    if nb < 0:
        raise RuntimeError(f"or_sync_pack failed: {nb}")
    return PackResult(buf, offs[:nb].copy(), sizes[:nb].copy(), stats)


def bucket_apply(bucket: bytes, weights) -> int:
    """Receiver path (Alg. 3): decode + scatter into weights (list of uint16 arrays; uint8 for
    FP8-tagged records)."""
    buf = np.frombuffer(bucket, np.uint8).copy()
    T = len(weights)
    numel = np.array([w.size for w in weights], np.uint64)
    for w in weights:
        assert w.dtype in (np.uint16, np.uint8) and w.flags.c_contiguous
    keep = [w if w.size else np.zeros(1, w.dtype) for w in weights]
    wp = (ctypes.c_void_p * max(T, 1))(*[k.ctypes.data for k in keep])
    return lib().or_bucket_apply(_p(buf), len(bucket), T, _p(numel), ctypes.cast(wp, ctypes.c_void_p))


def bucket_decode(bucket: bytes, cap: int, max_records: int = 1 << 20):
    """Receiver debug path: (status, [(tensor_id, I, V), ...])."""
    buf = np.frombuffer(bucket, np.uint8).copy()
    I = np.empty(max(cap, 1), np.uint32)
    V = np.empty(max(cap, 1), np.uint16)
    info = np.zeros(3 * max_records, np.uint64)
    nr = ctypes.c_uint32()
    st = lib().or_bucket_decode(_p(buf), len(bucket), _p(I), _p(V), cap, _p(info), max_records,
                                ctypes.byref(nr))
    recs = []
    if st == OK:
        for q in range(nr.value):
            tid, nnz, off = (int(v) for v in info[3 * q:3 * q + 3])
            recs.append((tid, I[off:off + nnz].copy(), V[off:off + nnz].copy()))
    return st, recs


# ----------------------------------------------------------------------------- cost model
def eq1_sparse_bytes(rho, N, b_v=2.0, b_i=4.0, s_meta=0.0):
    return lib().or_eq1_sparse_bytes(rho, N, b_v, b_i, s_meta)


def eq2_ratio(rho, b_v=2.0, b_i=4.0):
    return lib().or_eq2_ratio(rho, b_v, b_i)


def eq3_compressed_bytes(rho, N, b_v=2.0, b_i=2.0, alpha=0.6):
    return lib().or_eq3_compressed_bytes(rho, N, b_v, b_i, alpha)


def eq4_ratio(rho, b_v=2.0, b_i=2.0, alpha=0.6):
    return lib().or_eq4_ratio(rho, b_v, b_i, alpha)
