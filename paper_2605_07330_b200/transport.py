"""Bucket transfer between ranks (row a6; Alg. 2 l.10 SendToRollout / Alg. 3 l.2 RecvFromUpdater).

The paper moves buckets with "the same PyTorch process groups (NCCL) as before"
 and triggers them over a separate control plane (Ray). Here:
  * control plane: a gloo group carries the per-sync bucket manifest
    (count, offsets, sizes) — a few bytes on the host, like the paper's Ray call;
  * data plane: one NCCL P2P batch per bucket (send to the next rank, receive
    from the previous one), so bucket b+1 is on the wire while the receiver's
    decode+apply kernel (K5) works on bucket b.

RingLink implements the ring used by bench.py (rank r = Trainer of its model and
Rollout replica of rank r-1's model); PairLink a plain Trainer -> Rollout pair.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def _manifest_exchange(blist, dst, src, ctrl):
    """Send our bucket list to dst and receive src's over the control group. Returns [(offset, size)]."""
    n_out = torch.tensor([len(blist)], dtype=torch.int64)
    n_in = torch.zeros(1, dtype=torch.int64)
    reqs = []
    if dst is not None:
        reqs.append(dist.isend(n_out, dst, group=ctrl))
    if src is not None:
        reqs.append(dist.irecv(n_in, src, group=ctrl))
    for q in reqs:
        q.wait()
    m_out = torch.tensor([x for o, s in blist for x in (o, s)] or [0], dtype=torch.int64)
    m_in = torch.zeros(max(2 * int(n_in.item()), 1), dtype=torch.int64)
    reqs = []
    if dst is not None and len(blist):
        reqs.append(dist.isend(m_out, dst, group=ctrl))
    if src is not None and int(n_in.item()):
        reqs.append(dist.irecv(m_in, src, group=ctrl))
    for q in reqs:
        q.wait()
    k = int(n_in.item())
    return [(int(m_in[2 * i]), int(m_in[2 * i + 1])) for i in range(k)]


class _Link:
    def __init__(self, rank: int, world: int, device, ctrl=None, group=None, recv_buf: torch.Tensor | None = None):
        """recv_buf: optional uint8 device tensor to receive into (e.g. memory the caller no longer needs
        during the transfer); a private buffer is allocated if it is absent or too small."""
        self.rank, self.world, self.device = rank, world, torch.device(device)
        self.ctrl = ctrl
        self.group = group
        self.recv = recv_buf if recv_buf is not None else torch.empty(0, dtype=torch.uint8, device=self.device)
        self.last_in = []

    def _ensure(self, need: int):
        if self.recv.numel() < need:
            self.recv = torch.empty(int(need * 1.1) + 4096, dtype=torch.uint8, device=self.device)

    def _run(self, send_buf, blist, dst, src, apply_fn):
        incoming = _manifest_exchange(blist, dst, src, self.ctrl)
        self.last_in = incoming
        self._ensure(max((o + s for o, s in incoming), default=0))
        n_out = len(blist) if dst is not None else 0
        n_in = len(incoming)
        works = []
        for b in range(max(n_out, n_in)):
            ops = []
            if b < n_out:
                o, s = blist[b]
                ops.append(dist.P2POp(dist.isend, send_buf[o:o + s], dst, group=self.group))
            if b < n_in:
                o, s = incoming[b]
                ops.append(dist.P2POp(dist.irecv, self.recv[o:o + s], src, group=self.group))
            works.append(dist.batch_isend_irecv(ops))
        for b in range(max(n_out, n_in)):
            for w in works[b]:
                w.wait()                      # stream-ordered for NCCL: no host block
            if b < n_in and apply_fn is not None:
                o, s = incoming[b]
                apply_fn(self.recv[o:o + s])
        return incoming


class RingLink(_Link):
    """Buckets go r -> r+1; the buckets from r-1 are applied as they land."""

    def exchange(self, send_buf: torch.Tensor, blist, apply_fn):
        return self._run(send_buf, blist, (self.rank + 1) % self.world, (self.rank - 1) % self.world, apply_fn)


class PairLink(_Link):
    """Trainer rank `trainer` -> Rollout rank `rollout` (1T->1R; replica fan-out is several pairs)."""

    def __init__(self, rank, world, device, trainer: int, rollout: int, ctrl=None, group=None, recv_buf=None):
        super().__init__(rank, world, device, ctrl, group, recv_buf)
        self.trainer, self.rollout = trainer, rollout

    def send(self, send_buf, blist):
        return self._run(send_buf, blist, self.rollout, None, None)

    def receive(self, apply_fn):
        return self._run(None, [], None, self.trainer, apply_fn)
