"""B200-native SparseRL-Sync hot path (arxiv 2605.07330) — Python binding.

Thin ctypes binding over ``libsparsesync.so`` (hand-written sm_100a CUDA behind
the C ABI of ``include/sparsesync.h``). Functions keep the C names; this module
only marshals torch tensors into pointers, sizes and the current CUDA stream.
Every step of the method runs in the library's kernels. There is no CPU
fallback: if the library is missing or no CUDA device is present, calls raise.

Higher-level helpers: :class:`SyncContext` (one manifest, sender and/or
receiver), :class:`SparseSyncSender` / :class:`SparseSyncReceiver` (buffers +
the whole path), :mod:`.transport` (bucket exchange over torch.distributed).
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# SS_LIB: another build of the same library (dev A/B runs on one box); the default is the in-tree build
LIB_PATH = os.environ.get("SS_LIB") or os.path.join(_HERE, "libsparsesync.so")

SYNC_OK = 0
SYNC_ERR_ARG = -1
SYNC_ERR_ALIGNMENT = -2
SYNC_ERR_DTYPE = -3
SYNC_ERR_WORKSPACE = -4
SYNC_ERR_CUDA = -5
SYNC_ERR_INDEX_RANGE = -6
SYNC_ERR_CAPACITY = -7
SYNC_ERR_CORRUPT = -8
SYNC_ERR_BAD_MAGIC = -9
SYNC_ERR_VERSION = -10
SYNC_ERR_TRUNCATED = -11
SYNC_ERR_CRC = -12

SYNC_CODEC_RAW = 0
SYNC_CODEC_COMPRESSED = 1
SYNC_FLAG_CRC = 1
SYNC_FLAG_ROUTE = 2
SYNC_FLAG_ESCAPE = 4
SYNC_DTYPE_BF16 = 1
SYNC_DTYPE_FP16 = 2
SYNC_DTYPE_FP8 = 3
SYNC_CHUNK = 16384

EXPORTS = [
    "sync_workspace_size", "sync_ctx_create", "sync_ctx_destroy", "sync_extract_workspace_size", "sync_extract",
    "sync_extract_status", "sync_extract_batched", "sync_enc_bound", "sync_compress", "sync_bucket_pack",
    "sync_buckets_bound", "sync_compress_pack", "sync_bucket_unpack", "sync_decompress", "sync_decompress_apply", "sync_decompress_apply_batched", "sync_apply",
    "sync_commit_snapshot", "sync_commit_snapshot_batched", "sync_status", "sync_ctx_stats", "sync_strerror",
    "sync_launch_count", "sync_bitmap_words", "sync_cast_track_batched", "sync_extract_tracked",
    "sync_set_current", "sync_set_max_ctas", "sync_compress_pack_async", "sync_pack_result",
    "sync_pack_table", "sync_decompress_apply_table",
]
# NVLink peer-memory plumbing (include/sparsesync_peer.h)
PEER_EXPORTS = [
    "sync_peer_mem_export", "sync_peer_mem_open", "sync_peer_mem_close", "sync_peer_event_create",
    "sync_peer_event_open", "sync_peer_event_record", "sync_peer_stream_wait", "sync_peer_event_destroy",
    "sync_peer_copy",
]


class SyncError(RuntimeError):
    def __init__(self, code: int, where: str = ""):
        self.code = code
        super().__init__(f"{where}: {strerror(code)} ({code})" if where else f"{strerror(code)} ({code})")


class _Manifest(ctypes.Structure):
    _fields_ = [("n_tensors", ctypes.c_uint32), ("numel", ctypes.POINTER(ctypes.c_uint64))]


class _Config(ctypes.Structure):
    _fields_ = [("bucket_limit", ctypes.c_uint64), ("max_changed", ctypes.c_uint64),
                ("codec", ctypes.c_uint32), ("flags", ctypes.c_uint32), ("dtype", ctypes.c_uint32)]


class _Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in ["nnz", "n_records", "n_delta16", "n_abs32", "n_chunks",
                                                "n_chunks_rans", "enc_bytes", "index_bytes", "value_bytes",
                                                "n_full", "n_delta16e"]]


RECORD_VIEW_BYTES = 32

_lib = None


def lib() -> ctypes.CDLL:
    """Load libsparsesync.so (build it with ``python -m paper_2605_07330_b200.build``). Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        P, u64, u32, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
        PP = ctypes.POINTER
        sig = {
            "sync_workspace_size": [P, P, P],
            "sync_ctx_create": [P, P, P, P, ctypes.c_size_t, P],
            "sync_ctx_destroy": [P],
            "sync_extract_workspace_size": [u64, P],
            "sync_extract": [P, P, u64, P, P, u64, P, P, ctypes.c_size_t, P],
            "sync_extract_status": [P, P],
            "sync_extract_batched": [P, P, P, P, P, P, P],
            "sync_enc_bound": [P, P, P],
            "sync_compress": [P, P, P, P, P, u64, P],
            "sync_bucket_pack": [P, P, P, u64, P, P, P, u32, P],
            "sync_buckets_bound": [P, P, P],
            "sync_compress_pack": [P, P, P, P, P, u64, P, P, P, u32, P, P],
            "sync_compress_pack_async": [P, P, P, P, P, u64, u32, P],
            "sync_pack_result": [P, P, P, P, u32, P],
            "sync_pack_table": [P, P, P, P, P],
            "sync_decompress_apply_table": [P, P, P, P, P, u32, u32, P, u32, P],
            "sync_bucket_unpack": [P, P, u64, P, u32, P, P],
            "sync_decompress": [P, P, u64, P, P, u64, P],
            "sync_decompress_apply": [P, P, u64, P, P],
            "sync_decompress_apply_batched": [P, P, P, u32, P, P],
            "sync_apply": [P, P, P, u64, u64, P, P],
            "sync_commit_snapshot": [P, P, P, u64, u64, P, P],
            "sync_commit_snapshot_batched": [P, P, P, P, P, P],
            "sync_status": [P, P],
            "sync_ctx_stats": [P, P, P],
            "sync_bitmap_words": [P, P],
            "sync_set_current": [P, P],
            "sync_cast_track_batched": [P, P, P, P, P],
            "sync_extract_tracked": [P, P, P, P, P, P, i32, P],
            "sync_peer_mem_export": [P, P, P, P],
            "sync_peer_mem_open": [P, P],
            "sync_peer_mem_close": [P],
            "sync_peer_event_create": [P, P],
            "sync_peer_event_open": [P, P],
            "sync_peer_event_record": [P, P],
            "sync_peer_stream_wait": [P, P],
            "sync_peer_event_destroy": [P],
            "sync_peer_copy": [P, P, u64, P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = i32
        L.sync_strerror.argtypes = [i32]
        L.sync_strerror.restype = ctypes.c_char_p
        L.sync_launch_count.argtypes = []
        L.sync_launch_count.restype = u64
        L.sync_set_max_ctas.argtypes = [i32]
        L.sync_set_max_ctas.restype = i32
        _lib = L
    return _lib


def strerror(code: int) -> str:
    try:
        return lib().sync_strerror(code).decode()
    except ImportError:
        return f"status {code}"


def _ck(code: int, where: str):
    if code != SYNC_OK:
        raise SyncError(code, where)


def _stream(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor | None) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() if t is not None and t.numel() > 0 else 0)


def _dev_ptr(t: torch.Tensor) -> ctypes.c_void_p:
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor (no CPU path exists)")
    return _ptr(t)


def _bits(t: torch.Tensor) -> torch.Tensor:
    """bf16 / fp16 / int16 / uint16 tensor -> its 16-bit patterns; fp8 / uint8 / int8 -> its bytes (views)."""
    if t.dtype in (torch.bfloat16, torch.float16):
        return t.view(torch.int16)
    if t.dtype in (torch.int16, torch.uint16, torch.uint8):
        return t
    if t.dtype in (torch.float8_e4m3fn, torch.int8):
        return t.view(torch.uint8)
    raise SyncError(SYNC_ERR_DTYPE, f"dtype {t.dtype} (16-bit element types only)")


def ptr_table(tensors, device) -> torch.Tensor:
    """Device int64 array of data pointers (the C ABI's `const uint16_t* const*`)."""
    return torch.tensor([t.data_ptr() for t in tensors], dtype=torch.int64).to(device)


def launch_count() -> int:
    return int(lib().sync_launch_count())


def set_max_ctas(max_ctas: int) -> None:
    """Cap the CTAs of every library kernel launched from now on (0 = no cap); see sync_set_max_ctas."""
    _ck(lib().sync_set_max_ctas(int(max_ctas)), "sync_set_max_ctas")


# ----------------------------------------------------------------------------- single-tensor calls
def sync_extract(old: torch.Tensor, new: torch.Tensor, I: torch.Tensor | None = None, V: torch.Tensor | None = None,
                 count: torch.Tensor | None = None, workspace: torch.Tensor | None = None, stream=None):
    """Alg. 1 l.6 + Alg. 2 l.5 on one tensor: returns (I int32, V int16 bits, count int64[1]), all on device.

    I/V default to capacity numel (every element could change). The count is the true count even when
    it exceeds the capacity (then SYNC_ERR_CAPACITY is latched; see :func:`sync_extract_status`).
    """
    o, n = _bits(old).reshape(-1), _bits(new).reshape(-1)
    if o.shape != n.shape:
        raise SyncError(SYNC_ERR_ARG, "sync_extract: shape mismatch")
    N = o.numel()
    dev = o.device
    I = torch.empty(max(N, 1), dtype=torch.int32, device=dev) if I is None else I
    V = torch.empty(max(N, 1), dtype=torch.int16, device=dev) if V is None else V
    count = torch.empty(1, dtype=torch.int64, device=dev) if count is None else count
    if workspace is None:
        need = ctypes.c_size_t()
        _ck(lib().sync_extract_workspace_size(N, ctypes.byref(need)), "sync_extract_workspace_size")
        workspace = torch.zeros(need.value, dtype=torch.uint8, device=dev)
    _ck(lib().sync_extract(_dev_ptr(o), _dev_ptr(n), N, _dev_ptr(I), _dev_ptr(V), I.numel(), _dev_ptr(count),
                           _dev_ptr(workspace), workspace.numel(), _stream(stream)), "sync_extract")
    return I, V, count, workspace


def sync_extract_status(workspace: torch.Tensor, stream=None) -> int:
    return lib().sync_extract_status(_dev_ptr(workspace), _stream(stream))


def sync_apply(W: torch.Tensor, I: torch.Tensor, V: torch.Tensor, count: int | None = None,
               status: torch.Tensor | None = None, stream=None):
    """Alg. 3 l.6: W[I] <- V in place (bit copy). Out-of-range indices latch SYNC_ERR_INDEX_RANGE in status."""
    w = _bits(W).reshape(-1)
    count = I.numel() if count is None else count
    _ck(lib().sync_apply(_dev_ptr(w), _ptr(I), _ptr(V), count, w.numel(), _ptr(status), _stream(stream)),
        "sync_apply")


def sync_commit_snapshot(snapshot: torch.Tensor, I: torch.Tensor, V: torch.Tensor, count: int | None = None,
                         status: torch.Tensor | None = None, stream=None):
    """Same as sync_apply on the Trainer's snapshot; call after the transfer completed (DESIGN C13)."""
    w = _bits(snapshot).reshape(-1)
    count = I.numel() if count is None else count
    _ck(lib().sync_commit_snapshot(_dev_ptr(w), _ptr(I), _ptr(V), count, w.numel(), _ptr(status),
                                   _stream(stream)), "sync_commit_snapshot")


# ----------------------------------------------------------------------------- context
class SyncContext:
    """A manifest (ordered tensor sizes) + config + device workspace, for sender and receiver calls."""

    def __init__(self, numel, bucket_limit: int = 256 << 20, max_changed: int | None = None,
                 codec: int = SYNC_CODEC_COMPRESSED, crc: bool = False, device=None, route: bool = False,
                 dtype: int = SYNC_DTYPE_BF16, escape: bool = False, workspace: torch.Tensor | None = None):
        """workspace: optional caller-owned uint8 device tensor of >= workspace_size bytes (else allocated)."""
        self.numel = [int(n) for n in numel]
        self.device = torch.device(device or "cuda")
        self.T = len(self.numel)
        self.max_changed = int(max_changed if max_changed is not None else sum(self.numel))
        self._numel_arr = (ctypes.c_uint64 * max(self.T, 1))(*self.numel)
        self._m = _Manifest(self.T, self._numel_arr)
        self._c = _Config(int(bucket_limit), self.max_changed, int(codec),
                          (SYNC_FLAG_CRC if crc else 0) | (SYNC_FLAG_ROUTE if route else 0) |
                          (SYNC_FLAG_ESCAPE if escape else 0), int(dtype))
        self.codec, self.crc, self.bucket_limit, self.route = codec, crc, bucket_limit, route
        need = ctypes.c_size_t()
        _ck(lib().sync_workspace_size(ctypes.byref(self._m), ctypes.byref(self._c), ctypes.byref(need)),
            "sync_workspace_size")
        if workspace is not None:
            if workspace.dtype != torch.uint8 or workspace.numel() < need.value:
                raise SyncError(SYNC_ERR_WORKSPACE if workspace.numel() < need.value else -1, "workspace")
            self.workspace = workspace
        else:
            self.workspace = torch.zeros(need.value, dtype=torch.uint8, device=self.device)
        eb = ctypes.c_uint64()
        _ck(lib().sync_enc_bound(ctypes.byref(self._m), ctypes.byref(self._c), ctypes.byref(eb)), "sync_enc_bound")
        self.enc_bound = eb.value
        h = ctypes.c_void_p()
        _ck(lib().sync_ctx_create(ctypes.byref(h), ctypes.byref(self._m), ctypes.byref(self._c),
                                  _dev_ptr(self.workspace), self.workspace.numel(), _stream()), "sync_ctx_create")
        self._h = h
        self._max_buckets = max(self.T, 1)
        self._h_off = (ctypes.c_uint64 * self._max_buckets)()
        self._h_size = (ctypes.c_uint64 * self._max_buckets)()

    def close(self):
        if getattr(self, "_h", None):
            lib().sync_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- sender ---------------------------------------------------------------
    def sync_extract_batched(self, old_ptrs: torch.Tensor, new_ptrs: torch.Tensor, I: torch.Tensor,
                             V: torch.Tensor, counts: torch.Tensor, stream=None):
        _ck(lib().sync_extract_batched(self._h, _dev_ptr(old_ptrs), _dev_ptr(new_ptrs), _dev_ptr(I), _dev_ptr(V),
                                       _dev_ptr(counts), _stream(stream)), "sync_extract_batched")

    def sync_compress(self, I: torch.Tensor, V: torch.Tensor, counts: torch.Tensor, enc: torch.Tensor, stream=None):
        _ck(lib().sync_compress(self._h, _ptr(I), _ptr(V), _dev_ptr(counts), _dev_ptr(enc), enc.numel(),
                                _stream(stream)), "sync_compress")

    def sync_buckets_bound(self, stream=None) -> int:
        b = ctypes.c_uint64()
        _ck(lib().sync_buckets_bound(self._h, ctypes.byref(b), _stream(stream)), "sync_buckets_bound")
        return b.value

    def sync_bucket_pack(self, enc: torch.Tensor, buckets: torch.Tensor, stream=None):
        """Blocking. Returns [(offset, size)] of each bucket inside `buckets` (uint8)."""
        nb = ctypes.c_uint32()
        _ck(lib().sync_bucket_pack(self._h, _dev_ptr(enc), _dev_ptr(buckets), buckets.numel(), ctypes.byref(nb),
                                   self._h_off, self._h_size, self._max_buckets, _stream(stream)),
            "sync_bucket_pack")
        return [(int(self._h_off[b]), int(self._h_size[b])) for b in range(nb.value)]

    def sync_compress_pack(self, I: torch.Tensor, V: torch.Tensor, counts: torch.Tensor, buckets: torch.Tensor,
                           stream=None):
        """Blocking fused compress + pack. Returns ([(offset, size)], needed_bytes); raises SyncError
        (SYNC_ERR_CAPACITY) with .need set when `buckets` is too small."""
        nb = ctypes.c_uint32()
        need = ctypes.c_uint64()
        code = lib().sync_compress_pack(self._h, _ptr(I), _ptr(V), _dev_ptr(counts), _dev_ptr(buckets),
                                        buckets.numel(), ctypes.byref(nb), self._h_off, self._h_size,
                                        self._max_buckets, ctypes.byref(need), _stream(stream))
        if code != SYNC_OK:
            err = SyncError(code, "sync_compress_pack")
            err.need = need.value
            raise err
        return [(int(self._h_off[b]), int(self._h_size[b])) for b in range(nb.value)]

    def sync_compress_pack_async(self, I: torch.Tensor, V: torch.Tensor, counts: torch.Tensor,
                                 buckets: torch.Tensor, stream=None):
        """Enqueue-only fused compress + pack (CUDA-graph capturable); read the plan with sync_pack_result."""
        _ck(lib().sync_compress_pack_async(self._h, _ptr(I), _ptr(V), _dev_ptr(counts), _dev_ptr(buckets),
                                           buckets.numel(), self._max_buckets, _stream(stream)),
            "sync_compress_pack_async")

    def sync_pack_result(self):
        """Blocks until the last enqueued bucket plan is on the host; [(offset, size)] or SyncError (.need)."""
        nb = ctypes.c_uint32()
        need = ctypes.c_uint64()
        code = lib().sync_pack_result(self._h, ctypes.byref(nb), self._h_off, self._h_size, self._max_buckets,
                                      ctypes.byref(need))
        if code != SYNC_OK:
            err = SyncError(code, "sync_pack_result")
            err.need = need.value
            raise err
        return [(int(self._h_off[b]), int(self._h_size[b])) for b in range(nb.value)]

    def sync_pack_table(self):
        """Device pointers (hdr, offsets, sizes) of this context's bucket table (see include/sparsesync.h)."""
        h, o, z = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        st = ctypes.c_uint32()
        _ck(lib().sync_pack_table(self._h, ctypes.byref(h), ctypes.byref(o), ctypes.byref(z), ctypes.byref(st)),
            "sync_pack_table")
        return h.value, o.value, z.value, st.value

    def sync_decompress_apply_table(self, buckets: torch.Tensor, table, max_buckets: int, weight_ptrs: torch.Tensor,
                                    dense: bool = False, stream=None):
        """K5 over a sender's device bucket table (graph-capturable; no host knowledge of the bucket count)."""
        h, o, z, st = table
        _ck(lib().sync_decompress_apply_table(self._h, _dev_ptr(buckets), ctypes.c_void_p(h), ctypes.c_void_p(o),
                                              ctypes.c_void_p(z), int(st), int(max_buckets), _dev_ptr(weight_ptrs),
                                              1 if dense else 0, _stream(stream)), "sync_decompress_apply_table")

    def sync_commit_snapshot_batched(self, snap_ptrs: torch.Tensor, I: torch.Tensor, V: torch.Tensor,
                                     counts: torch.Tensor, stream=None):
        _ck(lib().sync_commit_snapshot_batched(self._h, _dev_ptr(snap_ptrs), _ptr(I), _ptr(V), _dev_ptr(counts),
                                               _stream(stream)), "sync_commit_snapshot_batched")

    def sync_set_current(self, new_ptrs: torch.Tensor):
        """f3: the current-weight pointer table FULL records copy from (kept alive by this object)."""
        self._cur = new_ptrs
        _ck(lib().sync_set_current(self._h, _dev_ptr(new_ptrs)), "sync_set_current")

    # -- f1 cast-fused tracking (Alg. 1) ---------------------------------------
    def bitmap_words(self) -> int:
        w = ctypes.c_uint64()
        _ck(lib().sync_bitmap_words(self._h, ctypes.byref(w)), "sync_bitmap_words")
        return w.value

    def sync_cast_track_batched(self, master_ptrs: torch.Tensor, weight_ptrs: torch.Tensor, bitmap: torch.Tensor,
                                stream=None):
        _ck(lib().sync_cast_track_batched(self._h, _dev_ptr(master_ptrs), _dev_ptr(weight_ptrs), _dev_ptr(bitmap),
                                          _stream(stream)), "sync_cast_track_batched")

    def sync_extract_tracked(self, weight_ptrs: torch.Tensor, bitmap: torch.Tensor, I: torch.Tensor,
                             V: torch.Tensor, counts: torch.Tensor, clear: bool = True, stream=None):
        _ck(lib().sync_extract_tracked(self._h, _dev_ptr(weight_ptrs), _dev_ptr(bitmap), _dev_ptr(I), _dev_ptr(V),
                                       _dev_ptr(counts), 1 if clear else 0, _stream(stream)), "sync_extract_tracked")

    # -- receiver -------------------------------------------------------------
    def sync_bucket_unpack(self, bucket: torch.Tensor, nbytes: int, views: torch.Tensor, n_records: torch.Tensor,
                           stream=None):
        _ck(lib().sync_bucket_unpack(self._h, _dev_ptr(bucket), nbytes, _dev_ptr(views),
                                     views.numel() // RECORD_VIEW_BYTES, _dev_ptr(n_records), _stream(stream)),
            "sync_bucket_unpack")

    def sync_decompress(self, bucket: torch.Tensor, nbytes: int, I: torch.Tensor, V: torch.Tensor, stream=None):
        _ck(lib().sync_decompress(self._h, _dev_ptr(bucket), nbytes, _dev_ptr(I), _dev_ptr(V), I.numel(),
                                  _stream(stream)), "sync_decompress")

    def sync_decompress_apply(self, bucket: torch.Tensor, nbytes: int, weight_ptrs: torch.Tensor, stream=None):
        _ck(lib().sync_decompress_apply(self._h, _dev_ptr(bucket), nbytes, _dev_ptr(weight_ptrs), _stream(stream)),
            "sync_decompress_apply")

    def sync_decompress_apply_batched(self, buckets, weight_ptrs: torch.Tensor, stream=None):
        """buckets: [(device address, nbytes)]; one kernel per 32 buckets."""
        n = len(buckets)
        if n == 0:
            return
        ptrs = (ctypes.c_void_p * n)(*[b[0] for b in buckets])
        sizes = (ctypes.c_uint64 * n)(*[b[1] for b in buckets])
        _ck(lib().sync_decompress_apply_batched(self._h, ptrs, sizes, n, _dev_ptr(weight_ptrs), _stream(stream)),
            "sync_decompress_apply_batched")

    def sync_decompress_apply_ptr(self, bucket_ptr: int, nbytes: int, weight_ptrs: torch.Tensor, stream=None):
        """Same, for a raw device address (e.g. a bucket inside a peer GPU's mapped buffer)."""
        _ck(lib().sync_decompress_apply(self._h, ctypes.c_void_p(bucket_ptr), nbytes, _dev_ptr(weight_ptrs),
                                        _stream(stream)), "sync_decompress_apply")

    # -- status ---------------------------------------------------------------
    def sync_status(self, stream=None) -> int:
        return lib().sync_status(self._h, _stream(stream))

    def check(self, where: str = "sync", stream=None):
        _ck(self.sync_status(stream), where)

    def stats(self, stream=None) -> dict:
        s = _Stats()
        _ck(lib().sync_ctx_stats(self._h, ctypes.byref(s), _stream(stream)), "sync_ctx_stats")
        return {n: int(getattr(s, n)) for n, _ in _Stats._fields_}


from .sync import SparseSyncReceiver, SparseSyncSender, TrackedSender  # noqa: E402,F401
