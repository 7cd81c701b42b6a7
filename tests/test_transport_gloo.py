"""Multi-process host logic of the transport (row a6) on CPU: world_size 2 with gloo.

The bucket bytes come from the oracle here (no GPU); the GPU path uses the same
RingLink with NCCL. Checks: manifests and bucket bytes arrive intact and in
order in the ring and in a Trainer -> Rollout pair, and the receiving side
reconstructs the sender's weights bit-exactly. World size 4: two sharded
Trainers fan their buckets out to two full-replica Rollouts (FanoutLink), and two
sharded 1T->1R pairs (PairLink)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _model(seed):
    import synth
    m = synth.Manifest("m", [synth.Tensor("a", (64, 300)), synth.Tensor("n", (32,), synth.KIND_NORM),
                             synth.Tensor("b", (50_000,))])
    return synth.generate(m, seed=seed, rho=0.05)


def _worker(rank, world, port, mode, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2605_07330_b200.transport import PairLink, RingLink
        olds, news = _model(seed=rank)
        pk = oracle.sync_pack(olds, news, limit=8 << 10)
        send_buf = torch.from_numpy(pk.buf.copy())
        blist = [(int(o), int(s)) for o, s in zip(pk.offsets, pk.sizes)]
        peer_olds, peer_news = _model(seed=(rank - 1) % world)
        W = [o.copy() for o in peer_olds]
        got = []

        def apply_fn(bk):
            b = bk.numpy().tobytes()
            got.append(b)
            assert oracle.bucket_apply(b, W) == oracle.OK

        if mode == "ring":
            link = RingLink(rank, world, "cpu", ctrl=None)
            link.exchange(send_buf, blist, apply_fn)
            ok = all((w == n).all() for w, n in zip(W, peer_news)) and len(got) > 1
        else:
            link = PairLink(rank, world, "cpu", trainer=0, rollout=1)
            if rank == 0:
                link.send(send_buf, blist)
                ok = True
            else:
                W = [o.copy() for o in _model(seed=0)[0]]
                link.receive(apply_fn)
                ok = all((w == n).all() for w, n in zip(W, _model(seed=0)[1]))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def _model4(seed):
    import synth
    m = synth.Manifest("m4", [synth.Tensor("a", (64, 300)), synth.Tensor("n", (32,), synth.KIND_NORM),
                              synth.Tensor("b", (50_000,)), synth.Tensor("c", (128, 129))])
    return synth.generate(m, seed=seed, rho=0.05)


def _shards(half):
    from paper_2605_07330_b200.transport import shard_ranges
    import synth
    m = synth.Manifest("m4", [synth.Tensor("a", (64, 300)), synth.Tensor("n", (32,), synth.KIND_NORM),
                              synth.Tensor("b", (50_000,)), synth.Tensor("c", (128, 129))])
    return shard_ranges(m.numel, half)


def _worker4(rank, world, port, mode, q):
    """ranks < world/2: Trainers of element-balanced shards of one model; ranks >= world/2: Rollouts (full
    replica for fanout / fanout_bcast, shard rank - world/2 for sharded pairs). World 4: 2T -> 2R; world 8:
    4T -> 4R (configs 4 and 5 of BASELINE.json)."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2605_07330_b200.transport import FanoutLink, PairLink
        half = world // 2
        shards = _shards(half)
        trainers, rollouts = list(range(half)), list(range(half, world))
        olds, news = _model4(seed=7)
        link = None
        if mode in ("fanout", "fanout_bcast"):   # every rank builds the link (broadcast groups are collective)
            link = FanoutLink(rank, world, "cpu", trainers=trainers, rollouts=rollouts,
                              mode="broadcast" if mode == "fanout_bcast" else "p2p")
        if rank < half:
            lo, hi = shards[rank]
            pk = oracle.sync_pack(olds[lo:hi], news[lo:hi], limit=2 << 10)
            send_buf = torch.from_numpy(pk.buf.copy())
            blist = [(int(o), int(s)) for o, s in zip(pk.offsets, pk.sizes)]
            if link is not None:
                link.send(send_buf, blist)
            else:
                PairLink(rank, world, "cpu", trainer=rank, rollout=rank + half).send(send_buf, blist)
            ok = len(blist) >= 1
        else:
            W = [o.copy() for o in olds]

            def fn(t):
                lo, hi = shards[t]
                view = W[lo:hi]   # the shard's records carry shard-local tensor ids

                def apply(bk):
                    assert oracle.bucket_apply(bk.numpy().tobytes(), view) == oracle.OK
                return apply

            if link is not None:
                link.receive({t: fn(t) for t in trainers})
                ok = all((w == n).all() for w, n in zip(W, news))
            else:
                t = rank - half
                PairLink(rank, world, "cpu", trainer=t, rollout=rank).receive(fn(t))
                lo, hi = shards[t]
                ok = all((w == n).all() for w, n in zip(W[lo:hi], news[lo:hi]))
                ok = ok and all((w == o).all() for k, (w, o) in enumerate(zip(W, olds)) if not lo <= k < hi)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [4, 8])
@pytest.mark.parametrize("mode", ["fanout", "fanout_bcast", "sharded_pairs"])
def test_fanout_and_pairs_gloo(world, mode):
    """2T->2R and 4T->4R (the 8-GPU topology of configs 4/5): replica fan-out by per-destination sends and
    by broadcast, and sharded Trainer -> Rollout pairs; every Rollout's weights == the oracle's new weights."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker4, args=(r, world, port, mode, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(240)
    res = dict(q.get(timeout=10) for _ in range(world))
    assert res == {r: True for r in range(world)}
    assert all(p.exitcode == 0 for p in ps)


@pytest.mark.parametrize("mode", ["ring", "pair"])
def test_world2_gloo(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: True, 1: True}
    assert all(p.exitcode == 0 for p in ps)


def test_shard_ranges():
    """Contiguous, non-empty, covering, element-balanced tensor ranges."""
    import random
    import sys
    sys.path.insert(0, ROOT)
    import synth
    from paper_2605_07330_b200.transport import shard_ranges
    for name in ("qwen3-30b-a3b", "qwen3-235b-a22b"):
        m = synth.qwen3_manifest(name)
        for T in (1, 2, 4, 8):
            r = shard_ranges(m.numel, T)
            assert r[0][0] == 0 and r[-1][1] == len(m.numel)
            assert all(a < b for a, b in r) and all(r[i][1] == r[i + 1][0] for i in range(T - 1))
            sizes = [sum(m.numel[a:b]) for a, b in r]
            assert max(sizes) - min(sizes) <= 2 * max(m.numel)
    # config 5: Qwen3-235B in 4 shards, one per Trainer of the 4T -> 4R box: each shard (old + new during the
    # sync) must leave room on a 180 GB B200 for the streamed groups (SURVEY 8(d) memory check)
    m = synth.qwen3_manifest("qwen3-235b-a22b")
    r4 = shard_ranges(m.numel, 4)
    per = [2 * sum(m.numel[a:b]) for a, b in r4]          # bf16 bytes of each shard
    assert all(1.14e11 < x < 1.21e11 for x in per), per   # 117.5 GB each, balanced to ~3%
    rng = random.Random(0)
    for _ in range(300):
        n = rng.randint(1, 12)
        numel = [rng.choice([0, 1, 5, 1000]) for _ in range(n)]
        for T in range(1, n + 1):
            r = shard_ranges(numel, T)
            assert len(r) == T and r[0][0] == 0 and r[-1][1] == n
            assert all(a < b for a, b in r) and all(r[i][1] == r[i + 1][0] for i in range(T - 1))
    with pytest.raises(ValueError):
        shard_ranges([1, 2], 3)
