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
        self.recv: dict[tuple[int, int], torch.Tensor] = {}
        self.free: dict[tuple[int, int], object] = {}     # CUDA event: applies that read this slot are done
        self.seq = 0
        self.pending_sends = []
        self.last_in: dict[int, list] = {}
        self.cuda = self.device.type == "cuda"
        self.comm = torch.cuda.Stream(device=self.device) if self.cuda else None

    def _buf(self, src: int, first: bool, need: int):
        slot = 0 if (first and self._given is not None) else self.seq % self.slots
        key = (src, slot)
        b = self.recv.get(key)
        if b is None and first and self._given is not None:
            b = self._given
        if b is None or b.numel() < need:
            b = torch.empty(int(need * 1.1) + 4096, dtype=torch.uint8, device=self.device)
        self.recv[key] = b
        return key, b

    def fence(self):
        """Make the current stream wait until the previous sync's sends have left the send buffer (call before
        overwriting it, i.e. before the next compress_pack)."""
        for w in self.pending_sends:
            w.wait()
        self.pending_sends = []

    def _run(self, send_buf, blist, dsts, srcs, apply_fns):
        """Send blist's buckets to every rank in dsts; receive every src's buckets and call apply_fns[src]
        on each as it lands (stream-ordered after that bucket's receive only). NCCL work is posted on a
        dedicated communication stream that waits for the producer (this stream) and, for a receive slot,
        for the applies that last read it; sends are only fenced before the send buffer is rewritten."""
        incoming = _manifest_exchange(blist, dsts, srcs, self.ctrl)
        self.last_in = incoming
        self.fence()
        bufs, keys = {}, {}
        for i, s in enumerate(srcs):
            keys[s], bufs[s] = self._buf(s, i == 0, max((o + z for o, z in incoming[s]), default=0))
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
                self.pending_sends += list(ws)   # send-only: fenced before the send buffer is rewritten
            for s in srcs:
                if b < len(incoming[s]) and apply_fns.get(s) is not None:
                    o, z = incoming[s][b]
                    apply_fns[s](bufs[s][o:o + z])
        if self.cuda:
            for s in srcs:
                ev = torch.cuda.Event()
                ev.record(cur)
                self.free[keys[s]] = ev
        self.seq += 1
        return incoming


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class RingLink(_Link):
    """Buckets go r -> r+1; the buckets from r-1 are applied as they land."""

    def exchange(self, send_buf: torch.Tensor, blist, apply_fn):
        src = (self.rank - 1) % self.world
        return self._run(send_buf, blist, [(self.rank + 1) % self.world], [src], {src: apply_fn})[src]


class PairLink(_Link):
    """Trainer rank `trainer` -> Rollout rank `rollout` (1T->1R; replica fan-out is FanoutLink)."""

    def __init__(self, rank, world, device, trainer: int, rollout: int, ctrl=None, group=None, recv_buf=None):
        super().__init__(rank, world, device, ctrl, group, recv_buf)
        self.trainer, self.rollout = trainer, rollout

    def send(self, send_buf, blist):
        return self._run(send_buf, blist, [self.rollout], [], {})

    def receive(self, apply_fn):
        return self._run(None, [], [], [self.trainer], {self.trainer: apply_fn})[self.trainer]


class FanoutLink(_Link):
    """T Trainers (shards) -> R Rollouts (full replicas): every Trainer sends each bucket to every Rollout;
    a Rollout applies Trainer t's buckets with the receiver of t's shard."""

    def __init__(self, rank, world, device, trainers: list[int], rollouts: list[int], ctrl=None, group=None):
        super().__init__(rank, world, device, ctrl, group)
        self.trainers, self.rollouts = list(trainers), list(rollouts)

    def send(self, send_buf, blist):
        return self._run(send_buf, blist, self.rollouts, [], {})

    def receive(self, apply_fns: dict):
        """apply_fns: {trainer rank: fn(bucket)}."""
        return self._run(None, [], [], self.trainers, apply_fns)


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
