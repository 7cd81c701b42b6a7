"""Bucket transfer between ranks (row a6; Alg. 2 l.10 SendToRollout / Alg. 3 l.2 RecvFromUpdater).

The paper moves buckets with "the same PyTorch process groups (NCCL) as before"
 and triggers them over a separate control plane (Ray). Here:
  * control plane: a gloo group carries the per-sync bucket manifest
    (count, offsets, sizes) — a few bytes on the host, like the paper's Ray call;
  * data plane: one NCCL P2P batch per bucket index (send bucket b to every
    destination, receive bucket b from every source), so bucket b+1 is on the
    wire while the receiver's decode+apply kernel (K5) works on bucket b.

Topologies:
  RingLink   rank r = Trainer of its model + Rollout replica of rank r-1's (weak scaling);
  PairLink   Trainer t -> Rollout t + T (1T->1R pairs; with sharded trainers this is
             the paper's "sharded Rollout" layout);
  FanoutLink T Trainers each own a shard; every Rollout holds the whole model and
             receives every Trainer's buckets ("forwards the aggregated M·K buckets
             to every rank").
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def _manifest_exchange(blist, dsts, srcs, ctrl):
    """Send our bucket list to every dst, receive every src's over the control group.
    Returns {src: [(offset, size)]}."""
    n_out = torch.tensor([len(blist)], dtype=torch.int64)
    n_in = {s: torch.zeros(1, dtype=torch.int64) for s in srcs}
    reqs = [dist.isend(n_out, d, group=ctrl) for d in dsts] + [dist.irecv(n_in[s], s, group=ctrl) for s in srcs]
    for q in reqs:
        q.wait()
    m_out = torch.tensor([x for o, s in blist for x in (o, s)] or [0], dtype=torch.int64)
    m_in = {s: torch.zeros(max(2 * int(n_in[s].item()), 1), dtype=torch.int64) for s in srcs}
    reqs = [dist.isend(m_out, d, group=ctrl) for d in dsts if len(blist)]
    reqs += [dist.irecv(m_in[s], s, group=ctrl) for s in srcs if int(n_in[s].item())]
    for q in reqs:
        q.wait()
    return {s: [(int(m_in[s][2 * i]), int(m_in[s][2 * i + 1])) for i in range(int(n_in[s].item()))] for s in srcs}


class _Link:
    def __init__(self, rank: int, world: int, device, ctrl=None, group=None, recv_buf: torch.Tensor | None = None,
                 slots: int = 2):
        """recv_buf: optional uint8 device tensor to receive into (e.g. memory the caller no longer needs
        during the transfer; used for the first source, and then single-buffered); otherwise `slots`
        private receive buffers per source rotate across syncs, so the receive of sync k+1 does not wait
        for the decode+apply of sync k."""
        self.rank, self.world, self.device = rank, world, torch.device(device)
        self.ctrl = ctrl
        self.group = group
        self._given = recv_buf
        self.slots = max(1, slots)
        self.recv: dict[tuple, torch.Tensor] = {}
        self.free: dict[tuple, object] = {}     # CUDA event: the applies that read this buffer are done
        self.seq: dict[int, int] = {}           # per tag: syncs run so far
        self.pending_sends: dict[int, list] = {}
        self.last_in: dict[int, list] = {}
        self.cuda = self.device.type == "cuda"
        self.comm = torch.cuda.Stream(device=self.device) if self.cuda else None

    def _buf(self, src: int, tag: int, first: bool, need: int, given=None):
        given = given if given is not None else (self._given if tag == 0 else None)
        slot = 0 if (first and given is not None) else self.seq.get(tag, 0) % self.slots
        key = (src, tag, slot)
        b = self.recv.get(key)
        if b is None and first and given is not None:
            b = given
        if b is None or b.numel() < need:
            b = torch.empty(int(need * 1.1) + 4096, dtype=torch.uint8, device=self.device)
        self.recv[key] = b
        return key, b

    def fence(self, tag: int = 0):
        """Make the current stream wait until the previous sync's sends of `tag` have left the send buffer
        (call before overwriting it, i.e. before the next compress_pack of that buffer)."""
        for w in self.pending_sends.pop(tag, []):
            w.wait()

    def _run(self, send_buf, blist, dsts, srcs, apply_fns, tag: int = 0, recv_buf=None):
        """Send blist's buckets to every rank in dsts; receive every src's buckets and call apply_fns[src]
        on each as it lands (stream-ordered after that bucket's receive only). NCCL work is posted on a
        dedicated communication stream that waits for the producer (this stream) and, for a receive slot,
        for the applies that last read it; sends are only fenced before the send buffer is rewritten."""
        incoming = _manifest_exchange(blist, dsts, srcs, self.ctrl)
        self.last_in = incoming
        self.fence(tag)
        bufs, keys = {}, {}
        for i, s in enumerate(srcs):
            keys[s], bufs[s] = self._buf(s, tag, i == 0, max((o + z for o, z in incoming[s]), default=0), recv_buf)
        n_out = len(blist) if dsts else 0
        nb = max([n_out] + [len(v) for v in incoming.values()])
        cur = torch.cuda.current_stream(self.device) if self.cuda else None
        if self.cuda:
            self.comm.wait_stream(cur)
            for s in srcs:
                ev = self.free.get(keys[s])
                if ev is not None:
                    self.comm.wait_event(ev)
        works = []
        ctx = torch.cuda.stream(self.comm) if self.cuda else _Null()
        with ctx:
            for b in range(nb):
                ops = []
                if b < n_out:
                    o, z = blist[b]
                    ops += [dist.P2POp(dist.isend, send_buf[o:o + z], d, group=self.group) for d in dsts]
                n_send = len(ops)
                for s in srcs:
                    if b < len(incoming[s]):
                        o, z = incoming[s][b]
                        ops.append(dist.P2POp(dist.irecv, bufs[s][o:o + z], s, group=self.group))
                ws = dist.batch_isend_irecv(ops) if ops else []
                works.append((ws, n_send))
        for b in range(nb):
            ws, n_send = works[b]
            if srcs or not self.cuda:
                for w in ws:
                    w.wait()                  # NCCL: stream-ordered, no host block (gloo: blocks)
            else:
                self.pending_sends.setdefault(tag, []).extend(ws)   # fenced before the buffer is rewritten
            for s in srcs:
                if b < len(incoming[s]) and apply_fns.get(s) is not None:
                    o, z = incoming[s][b]
                    apply_fns[s](bufs[s][o:o + z])
        if self.cuda:
            for s in srcs:
                ev = torch.cuda.Event()
                ev.record(cur)
                self.free[keys[s]] = ev
        self.seq[tag] = self.seq.get(tag, 0) + 1
        return incoming


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class RingLink(_Link):
    """Buckets go r -> r+1; the buckets from r-1 are applied as they land."""

    def exchange(self, send_buf: torch.Tensor, blist, apply_fn, tag: int = 0, recv_buf=None):
        src = (self.rank - 1) % self.world
        return self._run(send_buf, blist, [(self.rank + 1) % self.world], [src], {src: apply_fn}, tag,
                         recv_buf)[src]


class PairLink(_Link):
    """Trainer rank `trainer` -> Rollout rank `rollout` (1T->1R; replica fan-out is FanoutLink)."""

    def __init__(self, rank, world, device, trainer: int, rollout: int, ctrl=None, group=None, recv_buf=None):
        super().__init__(rank, world, device, ctrl, group, recv_buf)
        self.trainer, self.rollout = trainer, rollout

    def send(self, send_buf, blist, tag: int = 0):
        return self._run(send_buf, blist, [self.rollout], [], {}, tag)

    def receive(self, apply_fn, tag: int = 0):
        return self._run(None, [], [], [self.trainer], {self.trainer: apply_fn}, tag)[self.trainer]


class FanoutLink(_Link):
    """T Trainers (shards) -> R Rollouts (full replicas): every Trainer sends each bucket to every Rollout;
    a Rollout applies Trainer t's buckets with the receiver of t's shard.

    mode "p2p": one NCCL send per (bucket, Rollout) — R copies leave the Trainer.
    mode "broadcast": one NCCL broadcast per bucket in the group {t} + Rollouts (NCCL pipelines it through
    the group, or multicasts it over NVSwitch with NVLS), so each bucket leaves the Trainer once. The groups
    are created here: every rank must construct the link (torch.distributed.new_group is collective)."""

    def __init__(self, rank, world, device, trainers: list[int], rollouts: list[int], ctrl=None, group=None,
                 mode: str = "p2p"):
        super().__init__(rank, world, device, ctrl, group)
        self.trainers, self.rollouts = list(trainers), list(rollouts)
        if mode not in ("p2p", "broadcast"):
            raise ValueError(f"FanoutLink mode {mode!r}")
        self.mode = mode
        self.bgroups = {}
        if mode == "broadcast":
            for t in self.trainers:
                self.bgroups[t] = dist.new_group(sorted([t] + self.rollouts))

    def send(self, send_buf, blist, tag: int = 0):
        if self.mode == "broadcast":
            return self._bcast(send_buf, blist, {}, tag)
        return self._run(send_buf, blist, self.rollouts, [], {}, tag)

    def receive(self, apply_fns: dict, tag: int = 0):
        """apply_fns: {trainer rank: fn(bucket)}."""
        if self.mode == "broadcast":
            return self._bcast(None, [], apply_fns, tag)
        return self._run(None, [], [], self.trainers, apply_fns, tag)

    def _bcast(self, send_buf, blist, apply_fns, tag: int = 0):
        trainer = self.rank in self.trainers
        dsts = self.rollouts if trainer else []
        srcs = [] if trainer else self.trainers
        incoming = _manifest_exchange(blist, dsts, srcs, self.ctrl)
        self.last_in = incoming
        self.fence(tag)
        bufs, keys = {}, {}
        for i, s in enumerate(srcs):
            keys[s], bufs[s] = self._buf(s, tag, i == 0, max((o + z for o, z in incoming[s]), default=0))
        cur = torch.cuda.current_stream(self.device) if self.cuda else None
        if self.cuda:
            self.comm.wait_stream(cur)
            for s in srcs:
                ev = self.free.get(keys[s])
                if ev is not None:
                    self.comm.wait_event(ev)
        # every group member walks (bucket b, trainer t) in the same order
        order = []
        nb = len(blist) if trainer else max([len(v) for v in incoming.values()] or [0])
        for b in range(nb):
            for t in self.trainers:
                if trainer and t == self.rank:
                    order.append((t, b, send_buf[blist[b][0]:blist[b][0] + blist[b][1]]))
                elif not trainer and b < len(incoming[t]):
                    o, z = incoming[t][b]
                    order.append((t, b, bufs[t][o:o + z]))
        ctx = torch.cuda.stream(self.comm) if self.cuda else _Null()
        works = []
        with ctx:
            for t, b, view in order:
                works.append(dist.broadcast(view, src=t, group=self.bgroups[t], async_op=True))
        for (t, b, view), w in zip(order, works):
            if trainer and self.cuda:
                self.pending_sends.setdefault(tag, []).append(w)
                continue
            w.wait()
            if not trainer and apply_fns.get(t) is not None:
                apply_fns[t](view)
        if self.cuda:
            for s in srcs:
                ev = torch.cuda.Event()
                ev.record(cur)
                self.free[keys[s]] = ev
        self.seq[tag] = self.seq.get(tag, 0) + 1
        return incoming


def shard_ranges(numel: list[int], parts: int) -> list[tuple[int, int]]:
    """Split a manifest (tensor sizes in record order) into `parts` contiguous tensor ranges of about equal
    element count ("T contiguous, element-balanced ranges", PP-stage-like). Range k ends
    at the first tensor boundary at or past k/parts of the elements, so every range is non-empty when there
    are at least `parts` tensors."""
    n = len(numel)
    if parts < 1 or n < parts:
        raise ValueError(f"cannot split {n} tensors into {parts} shards")
    total = sum(numel)
    cuts, acc, k = [0], 0, 1
    for i, x in enumerate(numel):
        acc += x
        while k < parts and acc * parts >= k * total and i + 1 > cuts[-1] and n - (i + 1) >= parts - k:
            cuts.append(i + 1)
            k += 1
    while len(cuts) < parts:   # degenerate tails: one tensor per remaining shard
        cuts.append(n - (parts - len(cuts)))
    cuts.append(n)
    return [(cuts[j], cuts[j + 1]) for j in range(parts)]


# ============================================================================ NVLink peer-memory transport
def _plib():
    from . import lib
    return lib()


def _pck(code, where):
    if code != 0:
        from . import SyncError
        raise SyncError(code, where)


def _h2t(h: bytes) -> torch.Tensor:
    return torch.frombuffer(bytearray(h), dtype=torch.int64).clone()


def _t2h(t: torch.Tensor) -> bytes:
    return t.numpy().tobytes()


class _PeerEvent:
    """An interprocess CUDA event of this process (created here, exported as a 64-byte handle)."""

    def __init__(self):
        import ctypes
        self.ev = ctypes.c_void_p()
        self.handle = ctypes.create_string_buffer(64)
        _pck(_plib().sync_peer_event_create(ctypes.byref(self.ev), self.handle), "sync_peer_event_create")

    def record(self, stream):
        _pck(_plib().sync_peer_event_record(self.ev, stream), "sync_peer_event_record")


def _open_event(handle: bytes):
    import ctypes
    ev = ctypes.c_void_p()
    _pck(_plib().sync_peer_event_open(ctypes.create_string_buffer(handle, 64), ctypes.byref(ev)),
         "sync_peer_event_open")
    return ev


def _wait(stream, ev):
    _pck(_plib().sync_peer_stream_wait(stream, ev), "sync_peer_stream_wait")


_HDR = 21   # [seq, n, gen, base_offset, reserved] + mem handle (8 x i64) + ready-event handle (8 x i64)
_ACK = 9    # [seq] + consumed-event handle (8 x i64)


class PeerLink:
    """Bucket transfer over NVLink peer memory instead of NCCL (same roles and call pattern as the NCCL
    links; `dsts` = ranks this rank sends to, `srcs` = ranks it receives from).

    The Trainer exports its bucket buffer once (CUDA IPC) and, per sync and tag, records an interprocess
    "ready" event after the encode and sends the bucket manifest over the gloo control group. The Rollout
    maps the buffer, makes its stream wait for "ready", and then either pulls each bucket into a local
    buffer with the copy engines (mode "copy": no SMs spent on the transfer, bucket b+1 copies while bucket
    b is decoded) or lets the decode kernel read it in place over NVLink (mode "direct": one fused
    transfer+decompress+apply kernel, no staging copy). After its applies it records "consumed" and sends
    an ack; the Trainer waits for both before it rewrites that buffer (fence). The control messages order
    every record before the matching wait."""

    def __init__(self, rank: int, world: int, device, dsts, srcs, ctrl=None, mode: str = "copy"):
        assert mode in ("copy", "direct")
        self.rank, self.world, self.device = rank, world, torch.device(device)
        self.dsts, self.srcs, self.ctrl, self.mode = list(dsts), list(srcs), ctrl, mode
        self.seq: dict[int, int] = {}               # per tag: syncs sent
        self.rseq: dict[int, int] = {}              # per tag: syncs received
        # sender state
        self.exported: dict[int, tuple] = {}        # tag -> (ptr, numel, gen, handle bytes, offset)
        self.ready: dict[int, _PeerEvent] = {}
        self.pending: dict[int, list] = {}          # tag -> [(dst, ack work, ack tensor, send works)]
        self.peer_consumed: dict[tuple, object] = {}
        # receiver state
        self.maps: dict[tuple, tuple] = {}          # (src, tag) -> (gen, base ptr)
        self.peer_ready: dict[tuple, object] = {}
        self.consumed: dict[int, _PeerEvent] = {}
        self.local: dict[tuple, torch.Tensor] = {}  # copy mode: (src, tag) -> local bucket buffer
        self.local_free: dict[tuple, object] = {}
        self.ack_works = []
        self.copy_stream = torch.cuda.Stream(device=self.device) if mode == "copy" else None
        self.span_bytes = 64 << 20
        self._events, self._ev_i = [], 0
        self.last_in: dict[int, list] = {}

    def _event(self):
        """A reusable CUDA event (a ring of 64: far more than the spans in flight between two host syncs)."""
        if len(self._events) < 64:
            self._events.append(torch.cuda.Event())
            return self._events[-1]
        self._ev_i = (self._ev_i + 1) % len(self._events)
        return self._events[self._ev_i]

    @staticmethod
    def _tag(kind: int, tag: int) -> int:
        return 1000 * kind + tag + 1

    def _stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    # ------------------------------------------------------------------ sender
    def fence(self, tag: int = 0):
        """Before rewriting tag's send buffer: every destination has acknowledged the previous sync's buckets
        and this stream waits for their "consumed" events."""
        for dst, ack_w, ack_t, send_ws, _keep in self.pending.pop(tag, []):
            ack_w.wait()
            for w in send_ws:
                w.wait()
            key = (dst, tag)
            if key not in self.peer_consumed:
                self.peer_consumed[key] = _open_event(_t2h(ack_t[1:9]))
            _wait(self._stream(), self.peer_consumed[key])

    def mark_ready(self, tag: int = 0):
        """Record group `tag`'s "ready" event on the stream now (right after its encode was enqueued), for a
        caller that enqueues several groups before it sends their manifests (send(..., marked=True))."""
        if tag not in self.ready:
            self.ready[tag] = _PeerEvent()
        self.ready[tag].record(self._stream())

    def send(self, send_buf: torch.Tensor, blist, tag: int = 0, marked: bool = False):
        import ctypes
        self.fence(tag)   # normally already done by the caller before it rewrote the buffer
        seq = self.seq.get(tag, 0)
        ex = self.exported.get(tag)
        if ex is None or ex[0] != send_buf.data_ptr() or ex[1] != send_buf.numel():
            h = ctypes.create_string_buffer(64)
            off = ctypes.c_uint64()
            _pck(_plib().sync_peer_mem_export(ctypes.c_void_p(send_buf.data_ptr()), h, ctypes.byref(off), None),
                 "sync_peer_mem_export")
            ex = (send_buf.data_ptr(), send_buf.numel(), (ex[2] + 1) if ex else 1, h.raw, off.value)
            self.exported[tag] = ex
        if not marked:
            self.mark_ready(tag)
        hdr = torch.zeros(_HDR, dtype=torch.int64)
        hdr[0], hdr[1], hdr[2], hdr[3] = seq, len(blist), ex[2], ex[4]
        hdr[5:13] = _h2t(ex[3])
        hdr[13:21] = _h2t(self.ready[tag].handle.raw)
        body = torch.tensor([x for o, s in blist for x in (o, s)] or [0], dtype=torch.int64)
        for dst in self.dsts:
            ws = [dist.isend(hdr, dst, group=self.ctrl, tag=self._tag(1, tag))]
            if blist:
                ws.append(dist.isend(body, dst, group=self.ctrl, tag=self._tag(2, tag)))
            ack = torch.zeros(_ACK, dtype=torch.int64)
            aw = dist.irecv(ack, dst, group=self.ctrl, tag=self._tag(3, tag))
            self.pending.setdefault(tag, []).append((dst, aw, ack, ws, (hdr, body)))
        self.seq[tag] = seq + 1
        return blist

    # ------------------------------------------------------------------ receiver
    def receive(self, apply_fns: dict, tag: int = 0):
        """apply_fns: {src rank: fn([(device address, nbytes), ...])} — a batch of buckets per call (e.g.
        SparseSyncReceiver.apply_many): one copy span (copy mode) or all of src's buckets (direct mode)."""
        import ctypes
        cur = torch.cuda.current_stream(self.device)
        incoming = {}
        for w in self.ack_works:
            w.wait()
        self.ack_works = []
        for src in self.srcs:
            hdr = torch.zeros(_HDR, dtype=torch.int64)
            dist.recv(hdr, src, group=self.ctrl, tag=self._tag(1, tag))
            n, gen, off = int(hdr[1]), int(hdr[2]), int(hdr[3])
            blist = []
            if n:
                body = torch.zeros(2 * n, dtype=torch.int64)
                dist.recv(body, src, group=self.ctrl, tag=self._tag(2, tag))
                blist = [(int(body[2 * i]), int(body[2 * i + 1])) for i in range(n)]
            incoming[src] = blist
            key = (src, tag)
            m = self.maps.get(key)
            if m is None or m[0] != gen:
                if m is not None:
                    torch.cuda.synchronize(self.device)
                    _plib().sync_peer_mem_close(ctypes.c_void_p(m[1]))
                base = ctypes.c_void_p()
                _pck(_plib().sync_peer_mem_open(ctypes.create_string_buffer(_t2h(hdr[5:13]), 64), ctypes.byref(base)),
                     "sync_peer_mem_open")
                m = (gen, base.value)
                self.maps[key] = m
            if key not in self.peer_ready:
                self.peer_ready[key] = _open_event(_t2h(hdr[13:21]))
            remote = m[1] + off
            if not blist or apply_fns.get(src) is None:
                continue
            if self.mode == "direct":
                _wait(cur.cuda_stream, self.peer_ready[key])
                apply_fns[src]([(remote + o, z) for o, z in blist])
                continue
            need = max(o + z for o, z in blist)
            buf = self.local.get(key)
            if buf is None or buf.numel() < need:
                buf = torch.empty(int(need * 1.1) + 4096, dtype=torch.uint8, device=self.device)
                self.local[key] = buf
            cs = self.copy_stream
            cs.wait_stream(cur)                            # the previous decode from this buffer was enqueued
            _wait(cs.cuda_stream, self.peer_ready[key])    # the Trainer's encode of this sync is done
            # consecutive buckets are pulled in spans of >= span_bytes (one copy + one event per span), so small
            # buckets do not pay a copy launch and an event each; bucket b is decoded as soon as its span landed
            i = 0
            while i < len(blist):
                j, lo = i, blist[i][0]
                while j + 1 < len(blist) and blist[j][0] + blist[j][1] - lo < self.span_bytes:
                    j += 1
                hi = blist[j][0] + blist[j][1]
                _pck(_plib().sync_peer_copy(ctypes.c_void_p(buf.data_ptr() + lo), ctypes.c_void_p(remote + lo),
                                            hi - lo, ctypes.c_void_p(cs.cuda_stream)), "sync_peer_copy")
                ev = self._event()
                ev.record(cs)
                cur.wait_event(ev)
                apply_fns[src]([(buf.data_ptr() + o, z) for o, z in blist[i:j + 1]])   # one batched decode
                i = j + 1
        if tag not in self.consumed:
            self.consumed[tag] = _PeerEvent()
        self.consumed[tag].record(cur.cuda_stream)
        ack = torch.zeros(_ACK, dtype=torch.int64)
        ack[0] = self.rseq.get(tag, 0)
        ack[1:9] = _h2t(self.consumed[tag].handle.raw)
        for src in self.srcs:
            self.ack_works.append(dist.isend(ack, src, group=self.ctrl, tag=self._tag(3, tag)))
        self._ack_keep = ack
        self.rseq[tag] = self.rseq.get(tag, 0) + 1
        self.last_in = incoming
        return incoming

    def exchange(self, send_buf, blist, apply_fn, tag: int = 0, recv_buf=None):
        """Ring step: announce our buckets to the next rank, then receive and apply the previous rank's
        (apply_fn takes a batch, as in receive)."""
        self.send(send_buf, blist, tag)
        src = self.srcs[0]
        if recv_buf is not None and self.mode == "copy" and (src, tag) not in self.local:
            self.local[(src, tag)] = recv_buf
        return self.receive({src: apply_fn}, tag)[src]
