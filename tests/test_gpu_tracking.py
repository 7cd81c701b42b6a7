"""GPU parity of f1 cast-fused tracking (Alg. 1) against the oracle, through the C ABI.

Several optimizer steps of synthetic fp32 masters: after every step the bf16 weights W must equal the
oracle's round_BF16 bit for bit, and at the sync the tracked (I, V, counts) must equal the oracle's cumulative
set; the buckets packed from them must carry the oracle's record bytes, and a Rollout replica that applies
them must equal W. Edge cases: tensor tails (numel not a multiple of 32 / 8), an unaligned
tensor (scalar path), NaN / Inf / ties in the masters, an empty interval, capacity overflow (true counts,
CAPACITY latched, the set kept for the retry)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2605_07330_b200 as ss

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def host16(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16).reshape(-1)


SIZES = [70_000, 1, 31, 32, 33, 4096 * 9 + 5, 64, 0, 32768 * 2 + 40]


def masters(seed, sizes=SIZES):
    rng = np.random.default_rng(seed)
    return [(rng.standard_normal(n) * 0.02).astype(np.float32) for n in sizes]


def perturb(ms, rng, frac=0.02, scale=2e-3):
    out = []
    for m in ms:
        m = m.copy()
        if m.size:
            idx = rng.choice(m.size, max(1, int(frac * m.size)), replace=False)
            m[idx] += (rng.standard_normal(idx.size) * scale).astype(np.float32)
        out.append(m)
    return out


def make_sender(ms, W0, **kw):
    master_d = [torch.from_numpy(m).to(DEV) for m in ms]
    W_d = [torch.from_numpy(w.view(np.int16).copy()).to(DEV) for w in W0]
    snd = ss.TrackedSender(master_d, W_d, **kw)
    return snd, master_d, W_d


@pytest.mark.parametrize("steps", [1, 3])
def test_cast_track_and_extract_match_oracle(steps):
    rng = np.random.default_rng(steps)
    ms = masters(10 + steps)
    W_o = [oracle.bf16_rne(m) for m in ms]          # synced state (Rollout) = W at the last sync
    synced = [w.copy() for w in W_o]
    snd, master_d, W_d = make_sender(ms, W_o, max_changed=sum(m.size for m in ms))
    tracked = [np.zeros(m.size, np.uint8) for m in ms]
    for _ in range(steps):
        ms = perturb(ms, rng)
        for md, m in zip(master_d, ms):
            md.copy_(torch.from_numpy(m))
        snd.cast_track()
        for m, w, tr in zip(ms, W_o, tracked):
            oracle.cast_track(m, w, tr)
        torch.cuda.synchronize()
        for wd, w in zip(W_d, W_o):
            assert (host16(wd) == w).all()            # CastAndCopy bit-exact
    blist = snd.sync()
    torch.cuda.synchronize()
    snd.check()
    counts = snd.counts.cpu().numpy()
    I = snd.I.cpu().numpy().view(np.uint32)
    V = snd.V.cpu().numpy().view(np.uint16)
    off = 0
    recs = {}
    for t, (w, tr) in enumerate(zip(W_o, tracked)):
        Io, Vo = oracle.extract_tracked(w, tr)
        assert counts[t] == Io.size
        assert (I[off:off + Io.size] == Io).all() and (V[off:off + Io.size] == Vo).all()
        off += Io.size
        if Io.size:
            recs[t] = oracle.encode_record(t, Io, Vo)
    assert snd.bitmap.count_nonzero().item() == 0      # cleared for the next interval
    # the records in the buckets are the oracle's, and the replica reconstructs W exactly
    got = {}
    for b in range(len(blist)):
        a = snd.bucket(b).cpu().numpy()
        nrec = int(a[12:16].view(np.uint32)[0])
        dirv = a[32:32 + 8 * nrec].view(np.uint32).reshape(-1, 2)
        for q in range(nrec):
            ro = int(dirv[q, 0])
            tid, _, rb = (int(v) for v in a[ro:ro + 12].view(np.uint32))
            got[tid] = a[ro:ro + rb].tobytes()
    assert got == recs
    R = [torch.from_numpy(s.view(np.int16).copy()).to(DEV) for s in synced]
    rcv = ss.SparseSyncReceiver(R)
    rcv.apply_many([snd.bucket(b) for b in range(len(blist))])
    torch.cuda.synchronize()
    rcv.check()
    for r, w in zip(R, W_o):
        assert (host16(r) == w).all()


def test_special_values_and_unaligned_tensor():
    vals = np.array([np.nan, np.inf, -np.inf, 0.0, -0.0, 1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8,
                     np.finfo(np.float32).max, 1e-40, -1e-40], np.float32)
    base = np.resize(vals, 1001).astype(np.float32)
    W0 = oracle.bf16_rne(np.zeros(1001, np.float32))
    # an unaligned bf16 / fp32 pair: views starting one element into larger buffers
    mbuf = torch.zeros(1002, dtype=torch.float32, device=DEV)
    wbuf = torch.zeros(1002, dtype=torch.int16, device=DEV)
    mview, wview = mbuf[1:], wbuf[1:]
    mview.copy_(torch.from_numpy(base))
    wview.copy_(torch.from_numpy(W0.view(np.int16)))
    snd = ss.TrackedSender([mview], [wview], max_changed=1001)
    snd.cast_track()
    w_o = W0.copy()
    tr = np.zeros(1001, np.uint8)
    oracle.cast_track(base, w_o, tr)
    torch.cuda.synchronize()
    assert (host16(wview) == w_o).all()
    snd.extract()
    torch.cuda.synchronize()
    Io, Vo = oracle.extract_tracked(w_o, tr)
    c = int(snd.counts[0].item())
    assert c == Io.size
    assert (snd.I[:c].cpu().numpy().view(np.uint32) == Io).all()
    assert (snd.V[:c].cpu().numpy().view(np.uint16) == Vo).all()


def test_empty_interval_and_capacity():
    ms = masters(3)
    W_o = [oracle.bf16_rne(m) for m in ms]
    snd, master_d, W_d = make_sender(ms, W_o, max_changed=64)
    snd.cast_track()                  # masters unchanged: nothing enters the set
    snd.extract()
    torch.cuda.synchronize()
    assert int(snd.counts.sum().item()) == 0
    rng = np.random.default_rng(5)
    ms2 = perturb(ms, rng, frac=0.05)
    for md, m in zip(master_d, ms2):
        md.copy_(torch.from_numpy(m))
    snd.cast_track()
    want = sum(int((oracle.bf16_rne(a) != oracle.bf16_rne(b)).sum()) for a, b in zip(ms, ms2))
    assert want > 64
    snd.ctx.sync_extract_tracked(snd.weight_ptrs, snd.bitmap, snd.I, snd.V, snd.counts, True)
    torch.cuda.synchronize()
    assert int(snd.counts.sum().item()) == want                # true counts
    assert snd.ctx.sync_status() == ss.SYNC_ERR_CAPACITY
    assert snd.bitmap.count_nonzero().item() > 0              # the set is kept for the retry
    blist = snd.sync()                                        # grows I/V and extracts again
    torch.cuda.synchronize()
    snd.check()
    assert int(snd.counts.sum().item()) == want and len(blist) >= 1
    assert snd.bitmap.count_nonzero().item() == 0


def test_tracking_is_bf16_only():
    """Alg. 1's cast is round_BF16: an FP16 / FP8 context refuses the tracking calls (SYNC_ERR_DTYPE)."""
    ms = masters(4, sizes=[1000, 64])
    W0 = [oracle.bf16_rne(m) for m in ms]
    for dt in (ss.SYNC_DTYPE_FP16, ss.SYNC_DTYPE_FP8):
        with pytest.raises(ss.SyncError) as e:
            snd, _, _ = make_sender(ms, W0, dtype=dt)
            snd.cast_track()
        assert e.value.code == ss.SYNC_ERR_DTYPE


def test_random_bit_patterns_round_like_the_oracle():
    """Every fp32 class through the vectorised cast (cvt.rn.bf16x2 with the NaN fix-up, TMA-staged aligned tiles):
    uniformly random 32-bit patterns — normals of every exponent, subnormals, Inf, NaN payloads, values that
    round up into the next binade or overflow — must give round_BF16 (DESIGN C18) bit for bit."""
    n = 4 * 1024 * 1024 + 40
    rng = np.random.default_rng(123)
    bits = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    bits[:: 97] |= 0x7F800000          # more Inf / NaN
    bits[1:: 89] &= 0x807FFFFF         # more zeros / subnormals
    bits[2:: 83] |= 0x00007FFF         # ties and near-ties below the rounding bit
    master = bits.view(np.float32)
    W0 = np.zeros(n, np.uint16)
    md = torch.from_numpy(master.copy()).to(DEV)
    wd = torch.from_numpy(W0.view(np.int16).copy()).to(DEV)
    snd = ss.TrackedSender([md], [wd], max_changed=n)
    snd.cast_track()
    torch.cuda.synchronize()
    assert (host16(wd) == oracle.bf16_rne(master)).all()
    tr = np.zeros(n, np.uint8)
    w_o = W0.copy()
    oracle.cast_track(master, w_o, tr)
    snd.extract()
    torch.cuda.synchronize()
    Io, Vo = oracle.extract_tracked(w_o, tr)
    c = int(snd.counts[0].item())
    assert c == Io.size
    assert (snd.I[:c].cpu().numpy().view(np.uint32) == Io).all() and (snd.V[:c].cpu().numpy().view(np.uint16) == Vo).all()
