"""Out-of-bounds write checks with guard bands (compute-sanitizer is closed on this GPU pool).

Every buffer the library writes — I / V, the encoded stream, the bucket buffer, the context workspace, the
Rollout's weights — is allocated inside a larger tensor whose surrounding bytes hold a canary pattern; after a
full sync (extract, compress, pack, decode + apply, commit) at tight capacities the canaries must be intact and
every output must equal the oracle's. Also the single-tensor extract past its capacity and the Rollout
weights of tensors laid out with gaps between them (a scatter outside a tensor would land in a gap)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
ss = pytest.importorskip("paper_2605_07330_b200")
DEV = "cuda:0"
CANARY = 0xA5
PAD = 1 << 16   # guard bytes on each side


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_07330_b200 import build
    build.build()
    torch.cuda.set_device(0)


class Guarded:
    """n elements of `dtype` with PAD canary bytes before and after (the view is 256-byte aligned)."""

    def __init__(self, n, dtype):
        es = torch.empty(0, dtype=dtype).element_size()
        self.raw = torch.full((2 * PAD + n * es,), CANARY, dtype=torch.uint8, device=DEV)
        self.n, self.es = n, es
        self.t = self.raw[PAD:PAD + n * es].view(dtype)

    def intact(self) -> bool:
        head = self.raw[:PAD]
        tail = self.raw[PAD + self.n * self.es:]
        return bool((head == CANARY).all()) and bool((tail == CANARY).all())


def to_dev(a):
    return torch.from_numpy(a.view(np.int16).copy()).to(DEV)


def host16(t):
    return t.cpu().numpy().view(np.uint16)


@pytest.mark.parametrize("codec,crc,escape,route", [(ss.SYNC_CODEC_COMPRESSED, False, False, False),
                                                    (ss.SYNC_CODEC_COMPRESSED, True, True, True),
                                                    (ss.SYNC_CODEC_RAW, True, False, False)])
@pytest.mark.parametrize("fused", [True, False])
def test_sender_receiver_writes_stay_in_bounds(codec, crc, escape, route, fused):
    m = synth.Manifest("g", [synth.Tensor("a", (300, 512)), synth.Tensor("n", (64,), synth.KIND_NORM),
                             synth.Tensor("b", (200_000,)), synth.Tensor("c", (24,)), synth.Tensor("z", (0,)),
                             synth.Tensor("d", (96, 40), layer=0, expert=1)])
    olds, news = synth.generate(m, seed=9, rho=0.05, mask=synth.MASK_R if escape else synth.MASK_U)
    if route:
        news[3] = olds[3] ^ np.uint16(1)
    ref = oracle.sync_pack(olds, news, codec=codec, limit=32 << 10, crc=crc, route=route, escape=escape)
    nnz = ref.stats["nnz"]
    L = 32 << 10
    kw = dict(bucket_limit=L, max_changed=nnz, codec=codec, crc=crc, route=route, escape=escape, device=DEV)
    probe = ss.SyncContext(m.numel, **kw)
    ws = Guarded(probe.workspace.numel(), torch.uint8)   # the context workspace inside a guard band
    probe.close()
    ctx2 = ss.SyncContext(m.numel, workspace=ws.t, **kw)
    old_d = [to_dev(o) for o in olds]
    new_d = [to_dev(n) for n in news]
    old_ptrs = ss.ptr_table(old_d, DEV)
    new_ptrs = ss.ptr_table(new_d, DEV)
    if route:
        ctx2.sync_set_current(new_ptrs)
    gI = Guarded(nnz, torch.int32)
    gV = Guarded(nnz, torch.int16)
    counts = torch.zeros(len(olds), dtype=torch.int64, device=DEV)
    ctx2.sync_extract_batched(old_ptrs, new_ptrs, gI.t, gV.t, counts)
    need = sum(ref.sizes) + 256 * ref.n_buckets + 4096
    if fused:
        gB = Guarded(int(need), torch.uint8)
        bl = ctx2.sync_compress_pack(gI.t, gV.t, counts, gB.t)
        gE = None
    else:
        enc_need = int(ref.stats["payload_bytes"]) + 4096
        gE = Guarded(enc_need, torch.uint8)
        ctx2.sync_compress(gI.t, gV.t, counts, gE.t)
        gB = Guarded(int(need), torch.uint8)
        bl = ctx2.sync_bucket_pack(gE.t, gB.t)
    torch.cuda.synchronize()
    ctx2.check()
    got = [gB.t[o:o + z].cpu().numpy().tobytes() for o, z in bl]
    assert got == [ref.bucket(b) for b in range(ref.n_buckets)]
    # Rollout: weights laid out with canary gaps between the tensors
    gaps = [Guarded(max(o.size, 1), torch.int16) for o in olds]
    rol = [g.t[:o.size] for g, o in zip(gaps, olds)]
    for r, o in zip(rol, olds):
        r.copy_(to_dev(o))
    rcv = ss.SyncContext(m.numel, bucket_limit=L, codec=codec, crc=crc, device=DEV, max_changed=nnz)
    rptrs = ss.ptr_table(rol, DEV)
    for o, z in bl:
        rcv.sync_decompress_apply(gB.t[o:o + z], z, rptrs)
    ctx2.sync_commit_snapshot_batched(old_ptrs, gI.t, gV.t, counts)
    torch.cuda.synchronize()
    rcv.check()
    ctx2.check()
    for r, o, n in zip(rol, old_d, news):
        assert (host16(r) == n).all() and (host16(o) == n).all()
    for g in [ws, gI, gV, gB] + ([gE] if gE is not None else []) + gaps:
        assert g.intact(), "a write landed outside its buffer"
    ctx2.close()


def test_extract_single_over_capacity_stays_in_bounds():
    n = 300_001
    rng = np.random.default_rng(4)
    old = rng.integers(0, 65536, n, dtype=np.uint16)
    new = old.copy()
    new[::2] ^= np.uint16(7)
    cap = 5000
    gI, gV = Guarded(cap, torch.int32), Guarded(cap, torch.int16)
    I, V, cnt, ws = ss.sync_extract(to_dev(old), to_dev(new), I=gI.t, V=gV.t)
    torch.cuda.synchronize()
    assert ss.sync_extract_status(ws) == ss.SYNC_ERR_CAPACITY
    assert int(cnt.item()) == (n + 1) // 2
    assert (gI.t.cpu().numpy() == np.arange(0, 2 * cap, 2)).all()
    assert gI.intact() and gV.intact()
