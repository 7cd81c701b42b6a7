"""Multi-process host logic of the transport (row a6) on CPU: world_size 2 with gloo.

The bucket bytes come from the oracle here (no GPU); the GPU path uses the same
RingLink with NCCL. Checks: manifests and bucket bytes arrive intact and in
order in the ring and in a Trainer -> Rollout pair, and the receiving side
reconstructs the sender's weights bit-exactly."""
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
