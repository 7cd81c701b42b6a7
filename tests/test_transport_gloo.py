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


SHARDS = [(0, 2), (2, 4)]


def _worker4(rank, world, port, mode, q):
    """ranks 0, 1: Trainers of shards 0, 1 of one model; ranks 2, 3: Rollouts (full replica for fanout,
    shard rank-2 for sharded pairs)."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2605_07330_b200.transport import FanoutLink, PairLink
        olds, news = _model4(seed=7)
        if rank < 2:
            lo, hi = SHARDS[rank]
            pk = oracle.sync_pack(olds[lo:hi], news[lo:hi], limit=2 << 10)
            send_buf = torch.from_numpy(pk.buf.copy())
            blist = [(int(o), int(s)) for o, s in zip(pk.offsets, pk.sizes)]
            if mode == "fanout":
                FanoutLink(rank, world, "cpu", trainers=[0, 1], rollouts=[2, 3]).send(send_buf, blist)
            else:
                PairLink(rank, world, "cpu", trainer=rank, rollout=rank + 2).send(send_buf, blist)
            ok = len(blist) > 1
        else:
            W = [o.copy() for o in olds]

            def fn(t):
                lo, hi = SHARDS[t]
                view = W[lo:hi]   # the shard's records carry shard-local tensor ids

                def apply(bk):
                    assert oracle.bucket_apply(bk.numpy().tobytes(), view) == oracle.OK
                return apply

            if mode == "fanout":
                FanoutLink(rank, world, "cpu", trainers=[0, 1], rollouts=[2, 3]).receive({0: fn(0), 1: fn(1)})
                ok = all((w == n).all() for w, n in zip(W, news))
            else:
                t = rank - 2
                PairLink(rank, world, "cpu", trainer=t, rollout=rank).receive(fn(t))
                lo, hi = SHARDS[t]
                ok = all((w == n).all() for w, n in zip(W[lo:hi], news[lo:hi]))
                ok = ok and all((w == o).all() for k, (w, o) in enumerate(zip(W, olds)) if not lo <= k < hi)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["fanout", "sharded_pairs"])
def test_world4_gloo(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker4, args=(r, 4, port, mode, q)) for r in range(4)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(180)
    res = dict(q.get(timeout=10) for _ in range(4))
    assert res == {r: True for r in range(4)}
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
    m = synth.qwen3_manifest("qwen3-30b-a3b")
    for T in (1, 2, 4, 8):
        r = shard_ranges(m.numel, T)
        assert r[0][0] == 0 and r[-1][1] == len(m.numel)
        assert all(a < b for a, b in r) and all(r[i][1] == r[i + 1][0] for i in range(T - 1))
        sizes = [sum(m.numel[a:b]) for a, b in r]
        assert max(sizes) - min(sizes) <= 2 * max(m.numel)
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
