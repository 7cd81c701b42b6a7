"""NCCL data plane of the transport (row a6; "the same PyTorch process groups (NCCL)") on real GPUs.

One process per GPU (skipped unless the box has enough GPUs: run with `gpurun --gpus 2` / `--gpus 4`), an
NCCL group for the buckets and a gloo group for the bucket manifests, as bench.py sets them up:
  * ring (RingLink): every rank is the Trainer of its own model and the Rollout of rank r-1's;
  * pair (PairLink): Trainer t -> Rollout t + N/2, sharded model;
  * fanout (FanoutLink, per-destination sends and broadcast): N/2 sharded Trainers, N/2 full replicas.
The GPU sender's buckets must equal the oracle's bytes for the same seeded inputs, and every Rollout's
weights must equal the Trainer's new weights bit for bit after the sync."""
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


def _manifest():
    import synth
    return synth.Manifest("m", [synth.Tensor("a", (512, 700)), synth.Tensor("n", (64,), synth.KIND_NORM),
                                synth.Tensor("b", (300_000,)), synth.Tensor("c", (96, 1000)),
                                synth.Tensor("d", (2048, 256))])


def _worker(rank, world, port, mode, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    ctrl = dist.new_group(backend="gloo")
    ok = False
    try:
        import oracle
        import synth
        import synth.cpu as sc
        import synth.gpu as sg
        from paper_2605_07330_b200 import transport
        from paper_2605_07330_b200.sync import SparseSyncReceiver, SparseSyncSender
        m = _manifest()
        half = world // 2
        L = 64 << 10
        if mode == "ring":
            src = (rank - 1) % world
            own, peer = m, m
            own_seed, peer_seed, own_t0, peer_t0 = 200 + rank, 200 + src, 0, 0
            is_t, is_r = True, True
        else:
            shards = transport.shard_ranges(m.numel, half)
            is_t, is_r = rank < half, rank >= half
            t = rank if is_t else rank - half
            lo, hi = shards[t]
            own = m.slice(lo, hi)
            own_seed, own_t0 = 300, lo
            peer = m if mode.startswith("fanout") else m.slice(lo, hi)
            peer_seed, peer_t0 = 300, (0 if mode.startswith("fanout") else lo)
        snd = None
        if is_t:
            X, Xv = sg.arena(own, dev)
            Y, Yv = sg.arena(own, dev)
            sg.fill_old(Xv, own, own_seed, tid0=own_t0)
            sg.fill_new(Xv, Yv, own, own_seed, 0.03, tid0=own_t0)
            snd = SparseSyncSender(Xv, Yv, bucket_limit=L)
        rcvs = {}
        if is_r:
            R, Rv = sg.arena(peer, dev)
            sg.fill_old(Rv, peer, peer_seed, tid0=peer_t0)
            if mode == "ring":
                rcvs[src] = SparseSyncReceiver(Rv, bucket_limit=L)
            elif mode.startswith("fanout"):
                for tt in range(half):
                    a, b = shards[tt]
                    rcvs[tt] = SparseSyncReceiver(Rv[a:b], bucket_limit=L)
            else:
                rcvs[rank - half] = SparseSyncReceiver(Rv, bucket_limit=L)
        if mode == "ring":
            link = transport.RingLink(rank, world, dev, ctrl)
        elif mode == "pair":
            link = transport.PairLink(rank, world, dev, trainer=t, rollout=t + half, ctrl=ctrl)
        else:
            link = transport.FanoutLink(rank, world, dev, trainers=list(range(half)), rollouts=list(range(half, world)),
                                        ctrl=ctrl, mode="broadcast" if mode == "fanout_bcast" else "p2p")
        got = None
        if snd is not None:
            bl = snd.sync()
            got = [snd.bucket(b).cpu().numpy().tobytes() for b in range(len(bl))]
        if mode == "ring":
            link.exchange(snd.buckets, bl, rcvs[src].apply)
        elif is_t:
            link.send(snd.buckets, bl)
        elif mode.startswith("fanout"):
            link.receive({tt: rcvs[tt].apply for tt in rcvs})
        else:
            link.receive(rcvs[rank - half].apply)
        torch.cuda.synchronize()
        if snd is not None:
            snd.commit()
            link.fence(0)
        torch.cuda.synchronize()
        ok = True
        if snd is not None:
            snd.check()
            olds, news = sc.generate(own, seed=own_seed, rho=0.03, tid0=own_t0)
            pk = oracle.sync_pack(olds, news, limit=L)
            ok = ok and got == [pk.bucket(b) for b in range(pk.n_buckets)] and len(got) >= 1
        if is_r:
            for r in rcvs.values():
                r.check()
            _, pnews = sc.generate(peer, seed=peer_seed, rho=0.03, tid0=peer_t0)
            ok = ok and all((v.cpu().numpy().view("uint16") == n).all() for v, n in zip(Rv, pnews))
    except Exception as e:   # report, do not hang the other ranks' queue reads
        import traceback
        traceback.print_exc()
        ok = f"{type(e).__name__}: {e}"
    finally:
        q.put((rank, ok))
        try:
            dist.destroy_process_group()
        except Exception:
            pass


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("mode", ["ring", "pair", "fanout", "fanout_bcast"])
def test_nccl_links_bit_exact(world, mode):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (gpurun --gpus {world})")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in ps:
        p.join(60)
    assert res == {r: True for r in range(world)}, res
    assert all(p.exitcode == 0 for p in ps)
