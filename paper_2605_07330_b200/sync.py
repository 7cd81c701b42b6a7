"""Sender / receiver objects over one manifest: buffers + the whole hot path.

Sender (Trainer rank; Alg. 1 l.6 + Alg. 2):
    extract (K1) -> compress (K2/K3) -> pack (K4) ... transfer ... -> commit (K6)
Receiver (Rollout rank; Alg. 3):
    per bucket: decompress + scatter-apply (K5)

Every step is one or a few C-ABI calls into libsparsesync; this module only
owns the torch buffers (grown on demand from the library's size reports).
"""
from __future__ import annotations

import torch

from . import (SYNC_CODEC_COMPRESSED, SYNC_ERR_CAPACITY, SyncContext, SyncError, _bits, ptr_table)


def _flat_bits(ts):
    return [_bits(t).reshape(-1) for t in ts]


class SparseSyncSender:
    """Trainer side. `snapshot` = last-synced copy (W_prev), `current` = new weights W."""

    def __init__(self, snapshot, current, bucket_limit: int = 256 << 20, max_changed: int | None = None,
                 codec: int = SYNC_CODEC_COMPRESSED, crc: bool = False, expected_density: float = 0.02,
                 route: bool = False, dtype: int = 1, escape: bool = False):
        """route: per-parameter routing (f3): a record whose FULL copy is smaller goes FULL.
        dtype: SYNC_DTYPE_BF16 / SYNC_DTYPE_FP16 (f2): the record tag; the work is the same.
        escape: escape-coded DELTA16 (f4) for records with index gaps > 32767."""
        self.snapshot = _flat_bits(snapshot)
        self.current = _flat_bits(current)
        assert len(self.snapshot) == len(self.current)
        for a, b in zip(self.snapshot, self.current):
            if a.numel() != b.numel():
                raise SyncError(-1, "snapshot/current shape mismatch")
        self.device = self.current[0].device if self.current else torch.device("cuda")
        self.numel = [t.numel() for t in self.current]
        total = sum(self.numel)
        cap = int(max_changed if max_changed is not None else min(total, int(total * expected_density) + 65536))
        self._cfg = dict(bucket_limit=bucket_limit, codec=codec, crc=crc, route=route, dtype=dtype, escape=escape)
        self.old_ptrs = ptr_table(self.snapshot, self.device)
        self.new_ptrs = ptr_table(self.current, self.device)
        self.counts = torch.zeros(max(len(self.numel), 1), dtype=torch.int64, device=self.device)
        self.buckets = torch.empty(0, dtype=torch.uint8, device=self.device)
        self.bucket_list: list[tuple[int, int]] = []
        self._alloc(cap)

    def _alloc(self, cap: int):
        """(Re)size the changed-element capacity: context workspace, I/V and the encoded stream."""
        self.ctx = SyncContext(self.numel, max_changed=cap, device=self.device, **self._cfg)
        if self._cfg.get("route"):
            self.ctx.sync_set_current(self.new_ptrs)
        self.cap = cap
        self.I = torch.empty(max(cap, 1), dtype=torch.int32, device=self.device)
        self.V = torch.empty(max(cap, 1), dtype=torch.int16, device=self.device)
        self.enc = torch.empty(0, dtype=torch.uint8, device=self.device)  # only the unfused path uses it

    # K1 + K2/K3 (unfused path: contiguous encoded stream, then sync_bucket_pack copies it)
    def extract_compress(self, stream=None):
        if self.enc.numel() == 0:
            enc0 = min(self.ctx.enc_bound, int(3.6 * self.cap) + 64 * len(self.numel) + 4096)
            self.enc = torch.empty(enc0, dtype=torch.uint8, device=self.device)
        self.ctx.sync_extract_batched(self.old_ptrs, self.new_ptrs, self.I, self.V, self.counts, stream)
        self.ctx.sync_compress(self.I, self.V, self.counts, self.enc, stream)

    # K4 (blocking: the greedy bucket plan needs the record sizes on the host)
    def pack(self, stream=None):
        try:
            self.bucket_list = self._pack_once(stream)
        except SyncError as e:
            if e.code != SYNC_ERR_CAPACITY:
                raise
            self.ctx.sync_status(stream)           # clear the latched capacity error
            stats = self.ctx.stats(stream)
            if stats["nnz"] > self.cap:            # more changes than I/V can hold: grow, extract again
                self._alloc(min(sum(self.numel), int(stats["nnz"] * 1.1) + 65536))
                self.extract_compress(stream)
                stats = self.ctx.stats(stream)
            if stats["enc_bytes"] > self.enc.numel():
                self.enc = torch.empty(stats["enc_bytes"] + 4096, dtype=torch.uint8, device=self.device)
                self.ctx.sync_compress(self.I, self.V, self.counts, self.enc, stream)
            self.bucket_list = self._pack_once(stream)
        return self.bucket_list

    def _pack_once(self, stream):
        need = self.ctx.sync_buckets_bound(stream)
        if self.buckets.numel() < need:
            self.buckets = torch.empty(int(need * 1.05) + 4096, dtype=torch.uint8, device=self.device)
        return self.ctx.sync_bucket_pack(self.enc, self.buckets, stream)

    def bucket(self, b: int) -> torch.Tensor:
        off, size = self.bucket_list[b]
        return self.buckets[off:off + size]

    # K6: after the transfer completed (DESIGN C13)
    def commit(self, stream=None, mode: str = "scatter"):
        """Advance the snapshot to the synced weights.

        mode "scatter": snapshot[I] <- V in place (sync_commit_snapshot_batched, row a9).
        mode "swap": for a trainer that double-buffers its working copy, the current buffers become the
        snapshot by exchanging the two pointer tables (no bytes move); the next CastAndCopy / optimizer
        step then writes into the former snapshot buffers (W_prev is a per-step clone).
        """
        if mode == "swap":
            self.snapshot, self.current = self.current, self.snapshot
            self.old_ptrs, self.new_ptrs = self.new_ptrs, self.old_ptrs
            if self._cfg.get("route"):
                self.ctx.sync_set_current(self.new_ptrs)
            return
        self.ctx.sync_commit_snapshot_batched(self.old_ptrs, self.I, self.V, self.counts, stream)

    def compress_pack(self, stream=None):
        """Fused K2-K4 (sync_compress_pack): records encoded straight into their bucket positions."""
        if self.buckets.numel() == 0:
            self.buckets = torch.empty(int(3.5 * self.cap) + 64 * len(self.numel) + 4096, dtype=torch.uint8,
                                       device=self.device)
        for _ in range(3):
            try:
                self.bucket_list = self.ctx.sync_compress_pack(self.I, self.V, self.counts, self.buckets, stream)
                return self.bucket_list
            except SyncError as e:
                if e.code != SYNC_ERR_CAPACITY:
                    raise
                self.ctx.sync_status(stream)  # clear the latched error
                stats = self.ctx.stats(stream)
                if stats["nnz"] > self.cap:   # more changes than I/V can hold: grow, extract again
                    self._alloc(min(sum(self.numel), int(stats["nnz"] * 1.1) + 65536))
                    self.ctx.sync_extract_batched(self.old_ptrs, self.new_ptrs, self.I, self.V, self.counts, stream)
                elif getattr(e, "need", 0) > self.buckets.numel():
                    self.buckets = torch.empty(int(e.need * 1.05) + 4096, dtype=torch.uint8, device=self.device)
        raise SyncError(SYNC_ERR_CAPACITY, "sync_compress_pack: could not size the buffers")

    def compress_pack_async(self, stream=None):
        """Enqueue-only fused K2-K4 (sync_compress_pack_async: the bucket plan runs on the device, the host does
        not wait); collect the bucket list with pack_result(). Lets a caller enqueue several groups' syncs back
        to back and read their plans afterwards."""
        if self.buckets.numel() == 0:
            self.buckets = torch.empty(int(3.5 * self.cap) + 64 * len(self.numel) + 4096, dtype=torch.uint8,
                                       device=self.device)
        self.ctx.sync_compress_pack_async(self.I, self.V, self.counts, self.buckets, stream)

    def pack_result(self, stream=None):
        """The bucket list of the last compress_pack_async (blocks until its plan is on the host). On a capacity
        error the buffers are grown and the group is re-done synchronously (compress_pack), so the returned
        list is always complete; .redone tells the caller that the buckets were rewritten after the enqueue."""
        self.redone = False
        try:
            self.bucket_list = self.ctx.sync_pack_result()
            return self.bucket_list
        except SyncError as e:
            if e.code != SYNC_ERR_CAPACITY:
                raise
            self.ctx.sync_status(stream)
            stats = self.ctx.stats(stream)
            if stats["nnz"] > self.cap:
                self._alloc(min(sum(self.numel), int(stats["nnz"] * 1.1) + 65536))
                self._reextract(stream)
            elif getattr(e, "need", 0) > self.buckets.numel():
                self.buckets = torch.empty(int(e.need * 1.05) + 4096, dtype=torch.uint8, device=self.device)
            self.redone = True
            return self.compress_pack(stream)

    def _reextract(self, stream=None):
        self.ctx.sync_extract_batched(self.old_ptrs, self.new_ptrs, self.I, self.V, self.counts, stream)

    def sync(self, stream=None, fused: bool = True):
        """extract + compress + pack; returns the bucket list. Call commit() once the buckets were delivered."""
        if fused:
            self.ctx.sync_extract_batched(self.old_ptrs, self.new_ptrs, self.I, self.V, self.counts, stream)
            return self.compress_pack(stream)
        self.extract_compress(stream)
        return self.pack(stream)

    def check(self, stream=None):
        self.ctx.check("sender", stream)

    def stats(self, stream=None) -> dict:
        return self.ctx.stats(stream)


class TrackedSender(SparseSyncSender):
    """Trainer side with the paper's own hook (f1; Alg. 1): no snapshot. `cast_track()` is the
    optimizer-step epilogue (CastAndCopy W <- round_BF16(W_main) that also ORs the changed elements into the
    cumulative set); `sync()` extracts I from the set with V = W[I] (Alg. 2 l.4-5) and packs the buckets.

    master: fp32 master weights (one tensor per manifest entry); weights: the bf16 model weights W."""

    def __init__(self, master, weights, **kw):
        w = _flat_bits(weights)
        super().__init__(w, w, **kw)            # snapshot == current: the extract path is never used
        self.master = [m.reshape(-1) for m in master]
        for m, x in zip(self.master, w):
            if m.dtype != torch.float32 or m.numel() != x.numel():
                raise SyncError(-1, "master must be fp32 and match the weights")
        self.master_ptrs = ptr_table(self.master, self.device)
        self.weight_ptrs = self.new_ptrs
        self.bitmap = torch.zeros(max(self.ctx.bitmap_words(), 4), dtype=torch.int32, device=self.device)

    def cast_track(self, stream=None):
        """Alg. 1 l.5-7: W <- round_BF16(master); changed elements join the cumulative set."""
        self.ctx.sync_cast_track_batched(self.master_ptrs, self.weight_ptrs, self.bitmap, stream)

    def extract(self, stream=None, clear: bool = True):
        self.ctx.sync_extract_tracked(self.weight_ptrs, self.bitmap, self.I, self.V, self.counts, clear, stream)

    def _reextract(self, stream=None):
        self.extract(stream)   # on overflow the set was kept (nothing cleared)

    def compress_pack(self, stream=None):
        if self.buckets.numel() == 0:
            self.buckets = torch.empty(int(3.5 * self.cap) + 64 * len(self.numel) + 4096, dtype=torch.uint8,
                                       device=self.device)
        for _ in range(3):
            try:
                self.bucket_list = self.ctx.sync_compress_pack(self.I, self.V, self.counts, self.buckets, stream)
                return self.bucket_list
            except SyncError as e:
                if e.code != SYNC_ERR_CAPACITY:
                    raise
                self.ctx.sync_status(stream)
                stats = self.ctx.stats(stream)
                if stats["nnz"] > self.cap:   # the set was kept (nothing cleared): grow and extract again
                    self._alloc(min(sum(self.numel), int(stats["nnz"] * 1.1) + 65536))
                    self.extract(stream)
                if getattr(e, "need", 0) > self.buckets.numel():
                    self.buckets = torch.empty(int(e.need * 1.05) + 4096, dtype=torch.uint8, device=self.device)
        raise SyncError(SYNC_ERR_CAPACITY, "sync_compress_pack: could not size the buffers")

    def sync(self, stream=None, fused: bool = True):
        self.extract(stream)
        return self.compress_pack(stream)

    def commit(self, stream=None, mode: str = "none"):
        """Nothing to commit: the cumulative set was cleared by the extract (Alg. 1 l.1 of the next interval)."""
        return


class SparseSyncReceiver:
    """Rollout side: holds the weights and applies buckets in place (bit-exact)."""

    def __init__(self, weights, bucket_limit: int = 256 << 20, codec: int = SYNC_CODEC_COMPRESSED,
                 crc: bool = False, dtype: int = 1):
        self.weights = _flat_bits(weights)
        self.device = self.weights[0].device if self.weights else torch.device("cuda")
        numel = [t.numel() for t in self.weights]
        # a receiver never extracts or encodes: no changed-element capacity needed
        self.ctx = SyncContext(numel, bucket_limit=bucket_limit, max_changed=0, codec=codec, crc=crc,
                               device=self.device, dtype=dtype)
        self.weight_ptrs = ptr_table(self.weights, self.device)

    def apply(self, bucket, nbytes: int | None = None, stream=None):
        """bucket: a uint8 device tensor, or (device address, nbytes) — e.g. a bucket read in place from a
        peer GPU's mapped buffer (transport.PeerLink mode "direct")."""
        if isinstance(bucket, tuple):
            self.ctx.sync_decompress_apply_ptr(bucket[0], bucket[1], self.weight_ptrs, stream)
            return
        self.ctx.sync_decompress_apply(bucket, bucket.numel() if nbytes is None else nbytes, self.weight_ptrs,
                                       stream)

    def apply_many(self, buckets, stream=None):
        """Several buckets in one batched decode (sync_decompress_apply_batched); each a uint8 device tensor
        or (device address, nbytes)."""
        self.ctx.sync_decompress_apply_batched(
            [b if isinstance(b, tuple) else (b.data_ptr(), b.numel()) for b in buckets], self.weight_ptrs, stream)

    def check(self, stream=None):
        self.ctx.check("receiver", stream)


class GroupedSender:
    """A Trainer's tensors split into G contiguous groups (transport.shard_ranges), each a SparseSyncSender with
    its own context and buffers, so group g's buckets can be on the wire and applied while group g+1 is still
    being extracted (bucket pipelining, P:61 / P:275). Records carry group-local tensor ids; the receiving
    side uses a GroupedReceiver built from the same tensor list and G."""

    def __init__(self, snapshot, current, groups: int = 1, max_changed: int | None = None,
                 expected_density: float = 0.02, master=None, **kw):
        """master: fp32 master weights -> every group is a TrackedSender (f1, Alg. 1) over (master, current);
        `snapshot` is then unused."""
        from .transport import shard_ranges
        cur = list(current)
        snap = list(snapshot) if master is None else cur
        numel = [t.numel() for t in cur]
        self.ranges = shard_ranges(numel, max(1, min(groups, len(numel))))
        total = max(sum(numel), 1)
        self.parts = []
        for lo, hi in self.ranges:
            n = sum(numel[lo:hi])
            cap = None if max_changed is None else min(n, int(max_changed * n / total) + (1 << 16))
            if master is None:
                self.parts.append(SparseSyncSender(snap[lo:hi], cur[lo:hi], max_changed=cap,
                                                   expected_density=expected_density, **kw))
            else:
                self.parts.append(TrackedSender(list(master)[lo:hi], cur[lo:hi], max_changed=cap,
                                                expected_density=expected_density, **kw))

    def commit(self, stream=None, mode: str = "scatter"):
        for p in self.parts:
            p.commit(stream, mode)

    def stats(self, stream=None) -> dict:
        out = {}
        for p in self.parts:
            for k, v in p.stats(stream).items():
                out[k] = out.get(k, 0) + v
        return out

    def bucket_lists(self):
        return [p.bucket_list for p in self.parts]


class GroupedReceiver:
    """Receiving side of a GroupedSender: one SparseSyncReceiver per group of the same tensor list."""

    def __init__(self, weights, groups: int = 1, **kw):
        from .transport import shard_ranges
        w = list(weights)
        self.ranges = shard_ranges([t.numel() for t in w], max(1, min(groups, len(w))))
        self.parts = [SparseSyncReceiver(w[lo:hi], **kw) for lo, hi in self.ranges]
