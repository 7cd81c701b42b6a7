"""NVLink peer-memory transport (row a6, transport.PeerLink) end to end on the GPU.

Two processes (both on cuda:0 when the box has one GPU, else cuda:0 / cuda:1) form a
world-2 ring over a gloo control group: each is the Trainer of its own synthetic model
and the Rollout replica of the other's. Buckets travel through CUDA IPC (copy-engine
pull, or decoded in place from the peer's buffer); after several syncs each replica
must equal its peer's committed snapshot bit for bit, and the peer's buckets
must be byte-identical to what the oracle packs for the same inputs."""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, mode, groups, q):
    import sys
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        import synth
        import synth.gpu as sg
        from paper_2605_07330_b200 import transport
        from paper_2605_07330_b200.sync import GroupedReceiver, GroupedSender
        m = synth.Manifest("m", [synth.Tensor("a", (512, 700)), synth.Tensor("n", (64,), synth.KIND_NORM),
                                 synth.Tensor("b", (300_000,)), synth.Tensor("c", (96, 1000))])
        X, Xv = sg.arena(m, dev)
        Y, Yv = sg.arena(m, dev)
        R, Rv = sg.arena(m, dev)
        sg.fill_old(Xv, m, 100 + rank)
        sg.fill_new(Xv, Yv, m, 100 + rank, 0.03)
        sg.fill_old(Rv, m, 100 + (1 - rank))
        snd = GroupedSender(Xv, Yv, groups=groups, bucket_limit=64 << 10)
        rcv = GroupedReceiver(Rv, groups=groups, bucket_limit=64 << 10)
        link = transport.PeerLink(rank, 2, dev, [1 - rank], [1 - rank], mode=mode)
        first = {}
        for step in range(3):
            for g, p in enumerate(snd.parts):
                p.ctx.sync_extract_batched(p.old_ptrs, p.new_ptrs, p.I, p.V, p.counts)
                link.fence(g)
                blist = p.compress_pack()
                if step == 0:
                    first[g] = [p.bucket(b).cpu().numpy().tobytes() for b in range(len(blist))]
                link.exchange(p.buckets, blist, rcv.parts[g].apply_many, tag=g)
            snd.commit(mode="swap")   # the two buffers trade roles: the syncs go v0 -> v1 -> v0 -> v1
            X, Y = Y, X
        torch.cuda.synchronize()
        ok = all(p.ctx.sync_status() == 0 for p in snd.parts) and all(p.ctx.sync_status() == 0 for p in rcv.parts)
        # replica == peer's committed snapshot; own buckets == the oracle's for the same inputs
        mine = X.cpu().numpy().tobytes()
        got = R.cpu().numpy().tobytes()
        both = [None, None]
        dist.all_gather_object(both, (mine, got))
        ok = ok and both[1 - rank][0] == got
        import oracle
        import synth.cpu as sc
        olds, news = sc.generate(m, seed=100 + rank, rho=0.03)
        for g, (lo, hi) in enumerate(snd.ranges):
            pk = oracle.sync_pack(olds[lo:hi], news[lo:hi], limit=64 << 10)
            ok = ok and [pk.bucket(b) for b in range(pk.n_buckets)] == first[g]
        q.put((rank, bool(ok), np.uint8(0)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,groups", [("copy", 1), ("direct", 1), ("copy", 3), ("direct", 2)])
def test_peer_ring_world2(mode, groups):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, port, mode, groups, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
    res = {}
    for _ in range(2):
        r, ok, _ = q.get(timeout=30)
        res[r] = ok
    assert res == {0: True, 1: True}
    assert all(p.exitcode == 0 for p in ps)


def _worker_fanout(rank, world, port, q, deferred=False):
    """ranks 0, 1: Trainers of shards 0, 1 of one model (2 groups each); ranks 2, 3: full-replica Rollouts
    (fanout). Every process on cuda:(rank % device count). deferred: the Trainers enqueue each group's
    compress + pack without waiting for its plan (compress_pack_async), mark its buckets ready in stream order
    and send group g-1's manifest once group g is queued (bench.py's sender)."""
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        import synth.gpu as sg
        from paper_2605_07330_b200 import transport
        from paper_2605_07330_b200.sync import GroupedReceiver, GroupedSender
        m = synth.Manifest("m", [synth.Tensor("a", (512, 700)), synth.Tensor("n", (64,), synth.KIND_NORM),
                                 synth.Tensor("b", (300_000,)), synth.Tensor("c", (96, 1000)),
                                 synth.Tensor("d", (20_000,))])
        shards = transport.shard_ranges(m.numel, 2)
        ok = True
        if rank < 2:
            lo, hi = shards[rank]
            ms = m.slice(lo, hi)
            X, Xv = sg.arena(ms, dev)
            Y, Yv = sg.arena(ms, dev)
            sg.fill_old(Xv, ms, 7, tid0=lo)
            sg.fill_new(Xv, Yv, ms, 7, 0.03, tid0=lo)
            snd = GroupedSender(Xv, Yv, groups=2, bucket_limit=32 << 10)
            link = transport.PeerLink(rank, world, dev, [2, 3], [])
            for step in range(3):
                pending = []
                for g, p in enumerate(snd.parts):
                    p.ctx.sync_extract_batched(p.old_ptrs, p.new_ptrs, p.I, p.V, p.counts)
                    link.fence(g)
                    if deferred:
                        p.compress_pack_async()
                        link.mark_ready(g)
                        pending.append(g)
                        if len(pending) > 1:
                            h = pending.pop(0)
                            link.send(snd.parts[h].buckets, snd.parts[h].pack_result(), tag=h,
                                      marked=not snd.parts[h].redone)
                        continue
                    blist = p.compress_pack()
                    link.send(p.buckets, blist, tag=g)
                for h in pending:
                    link.send(snd.parts[h].buckets, snd.parts[h].pack_result(), tag=h,
                              marked=not snd.parts[h].redone)
                snd.commit(mode="swap")
                X, Y = Y, X
            for g in range(2):
                link.fence(g)
            torch.cuda.synchronize()
            both = [None] * world
            dist.all_gather_object(both, X.cpu().numpy().tobytes())
        else:
            R, Rv = sg.arena(m, dev)
            sg.fill_old(Rv, m, 7)
            rcvs = {t: GroupedReceiver(Rv[lo:hi], groups=2, bucket_limit=32 << 10) for t, (lo, hi) in enumerate(shards)}
            link = transport.PeerLink(rank, world, dev, [], [0, 1])
            for step in range(3):
                for g in range(2):
                    link.receive({t: rcvs[t].parts[g].apply_many for t in rcvs}, tag=g)
            torch.cuda.synchronize()
            ok = all(p.ctx.sync_status() == 0 for r in rcvs.values() for p in r.parts)
            both = [None] * world
            dist.all_gather_object(both, None)
            got = R.cpu().numpy().tobytes()
            ok = ok and got == both[0] + both[1]    # the replica = the two Trainers' committed shards
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("deferred", [False, True])
def test_peer_fanout_world4(deferred):
    """Send-only / receive-only PeerLink roles: 2 sharded Trainers fan out to 2 full replicas (3 syncs); with
    deferred manifests (enqueue-only compress + pack) as well."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_fanout, args=(r, 4, port, q, deferred)) for r in range(4)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
    res = dict(q.get(timeout=30) for _ in range(4))
    assert res == {r: True for r in range(4)}
    assert all(p.exitcode == 0 for p in ps)
