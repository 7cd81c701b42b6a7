"""GPU <-> oracle parity (run on a B200 with -m gpu). All calls go through the C ABI.

Bar: bit-exact (integer / byte / index work; DESIGN C17 — exactly one correct byte
string exists per input). Inputs: the shared seeded generator (synth), both its
numpy twin (oracle side) and its CUDA twin (GPU side) — the two must agree too.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

ss = pytest.importorskip("paper_2605_07330_b200")


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_07330_b200 import build
    build.build()
    torch.cuda.set_device(0)


DEV = "cuda:0"


def to_dev(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(a.view(np.int16).copy()).to(DEV)


def host16(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint16)


# ----------------------------------------------------------------------------- a1 single tensor
@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 255, 8191, 8192, 8193, 65536 + 3, 1 << 20, 1_000_003])
@pytest.mark.parametrize("rho", [0.0, 0.01, 0.3, 1.0])
def test_extract_single_vs_oracle(n, rho):
    rng = np.random.default_rng(n + int(rho * 1000))
    old = rng.integers(0, 65536, n, dtype=np.uint16)
    new = old.copy()
    m = rng.random(n) < rho
    new[m] ^= rng.integers(1, 65536, int(m.sum()), dtype=np.uint16)
    I, V, cnt, ws = ss.sync_extract(to_dev(old), to_dev(new))
    torch.cuda.synchronize()
    assert ss.sync_extract_status(ws) == ss.SYNC_OK
    Io, Vo = oracle.extract(old, new)
    c = int(cnt.item())
    assert c == Io.size
    assert (I[:c].cpu().numpy().view(np.uint32) == Io).all()
    assert (host16(V[:c]) == Vo).all()


def test_extract_bf16_edge_cases():
    old = np.array([0x0000, 0x7FC0, 0x7FC0, 0xFF80, 0x3F80] * 3000, np.uint16)
    new = np.array([0x8000, 0x7FC0, 0x7FC1, 0xFF80, 0x3F81] * 3000, np.uint16)
    I, V, cnt, ws = ss.sync_extract(to_dev(old), to_dev(new))
    Io, Vo = oracle.extract(old, new)
    c = int(cnt.item())
    assert c == Io.size == 9000
    assert (I[:c].cpu().numpy().view(np.uint32) == Io).all() and (host16(V[:c]) == Vo).all()


def test_extract_capacity_reports_true_count():
    n = 100_000
    old = np.zeros(n, np.uint16)
    new = old.copy()
    new[::3] = 1
    cap = 1000
    I = torch.empty(cap, dtype=torch.int32, device=DEV)
    V = torch.empty(cap, dtype=torch.int16, device=DEV)
    I2, V2, cnt, ws = ss.sync_extract(to_dev(old), to_dev(new), I=I, V=V)
    torch.cuda.synchronize()
    assert int(cnt.item()) == len(range(0, n, 3))
    assert ss.sync_extract_status(ws) == ss.SYNC_ERR_CAPACITY
    assert (I.cpu().numpy() == np.arange(0, 3 * cap, 3)).all()   # first cap entries are exact


def test_generator_twins_agree():
    m = synth.Manifest("g", [synth.Tensor("a", (300, 1000)), synth.Tensor("n", (64,), synth.KIND_NORM),
                             synth.Tensor("e", (96, 40), layer=3, expert=5)])
    import synth.gpu as sg
    for mask in [synth.MASK_U, synth.MASK_R, synth.MASK_E]:
        _, old = sg.arena(m, DEV)
        _, new = sg.arena(m, DEV)
        sg.fill_old(old, m, seed=7, tid0=11)
        sg.fill_new(old, new, m, seed=7, rho=0.05, mask=mask, tid0=11)
        olds, news = synth.generate(m, seed=7, rho=0.05, mask=mask, tid0=11)
        for a, b in zip(old, olds):
            assert (host16(a) == b).all()
        for a, b in zip(new, news):
            assert (host16(a) == b).all()
        # the batched generator of the bench's streaming mode writes the same new weights (tensors larger
        # than its 1 Mi-element tile included)
        _, new2 = sg.arena(m, DEV)
        sg.FillNewPlan(old, new2, m, seed=7, rho=0.05, mask=mask, tid0=11).run()
        for a, b in zip(new2, news):
            assert (host16(a) == b).all()
    big = synth.Manifest("b", [synth.Tensor("w", (1100, 1000)), synth.Tensor("t", (8,))])
    _, old = sg.arena(big, DEV)
    _, new = sg.arena(big, DEV)
    sg.fill_old(old, big, seed=3)
    sg.FillNewPlan(old, new, big, seed=3, rho=0.01).run()
    _, news = synth.generate(big, seed=3, rho=0.01)
    for a, b in zip(new, news):
        assert (host16(a) == b).all()


# ----------------------------------------------------------------------------- whole path
def mixed_manifest():
    T = [synth.Tensor("embed", (3000, 64)), synth.Tensor("norm", (64,), synth.KIND_NORM),
         synth.Tensor("empty", (0,)), synth.Tensor("tiny", (8,)), synth.Tensor("odd", (1,)),
         synth.Tensor("big", (70_000,)), synth.Tensor("q", (256, 512))]
    T += [synth.Tensor(f"e{k}", (48, 64), layer=0, expert=k) for k in range(40)]
    T += [synth.Tensor("tail", (8192 * 3 + 8,))]
    return synth.Manifest("mixed", T)


def run_path(olds, news, codec, limit, crc, max_changed=None, fused=True):
    """GPU sender on device copies; returns (sender, receiver weights after apply, bucket bytes list).
    fused: sync_compress_pack (records encoded in place) vs sync_compress + sync_bucket_pack."""
    old_d = [to_dev(o) for o in olds]
    new_d = [to_dev(n) for n in news]
    rol_d = [to_dev(o) for o in olds]
    snd = ss.SparseSyncSender(old_d, new_d, bucket_limit=limit, codec=codec, crc=crc, max_changed=max_changed)
    rcv = ss.SparseSyncReceiver(rol_d, bucket_limit=limit, codec=codec, crc=crc)
    bl = snd.sync(fused=fused)
    got = [snd.bucket(b).cpu().numpy().tobytes() for b in range(len(bl))]
    for b in range(len(bl)):
        rcv.apply(snd.bucket(b))
    snd.commit()
    torch.cuda.synchronize()
    snd.check()
    rcv.check()
    return snd, old_d, rol_d, got


@pytest.mark.parametrize("codec", [ss.SYNC_CODEC_COMPRESSED, ss.SYNC_CODEC_RAW])
@pytest.mark.parametrize("limit", [1024, 64 << 10, 1 << 30])
@pytest.mark.parametrize("crc", [False, True])
@pytest.mark.parametrize("rho,mask", [(0.01, synth.MASK_U), (0.2, synth.MASK_U), (0.02, synth.MASK_R)])
@pytest.mark.parametrize("fused", [True, False])
def test_bucket_bytes_and_apply_bit_exact(codec, limit, crc, rho, mask, fused):
    m = mixed_manifest()
    olds, news = synth.generate(m, seed=1, rho=rho, mask=mask)
    ref = oracle.sync_pack(olds, news, codec=codec, limit=limit, crc=crc)
    snd, old_d, rol_d, got = run_path(olds, news, codec, limit, crc, fused=fused)
    assert len(got) == ref.n_buckets
    for b in range(ref.n_buckets):
        assert got[b] == ref.bucket(b), f"bucket {b} bytes differ"
    for r, o, n in zip(rol_d, old_d, news):
        assert (host16(r) == n).all()        # receiver bit-identical (G1)
        assert (host16(o) == n).all()        # snapshot committed
    st = snd.stats()
    assert st["nnz"] == ref.stats["nnz"] and st["n_records"] == ref.stats["n_records"]


@pytest.mark.parametrize("codec", [ss.SYNC_CODEC_COMPRESSED, ss.SYNC_CODEC_RAW])
@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("crc", [False, True])
def test_routing_full_records_bit_exact(codec, fused, crc):
    """f3: tensors updated on (nearly) every element go FULL — GPU bucket bytes == oracle's, the
    replica applies them, and the sender's snapshot commit is unaffected."""
    m = mixed_manifest()
    olds, news = synth.generate(m, seed=21, rho=0.02)
    rng = np.random.default_rng(21)
    for k in (0, 5, 6, len(news) - 1):            # dense updates: LoRA-like / fully retrained tensors
        if news[k].size:
            news[k] = olds[k] ^ np.uint16(1)
    k = 9                                          # a 50%-dense expert: FULL for raw, sparse or FULL otherwise
    idx = rng.choice(news[k].size, news[k].size // 2, replace=False)
    news[k] = olds[k].copy()
    news[k][idx] ^= np.uint16(2)
    ref = oracle.sync_pack(olds, news, codec=codec, limit=64 << 10, crc=crc, route=True)
    assert ref.stats["full"] >= 3
    old_d = [to_dev(o) for o in olds]
    new_d = [to_dev(n) for n in news]
    rol_d = [to_dev(o) for o in olds]
    snd = ss.SparseSyncSender(old_d, new_d, bucket_limit=64 << 10, codec=codec, crc=crc, route=True,
                              max_changed=sum(o.size for o in olds))
    rcv = ss.SparseSyncReceiver(rol_d, bucket_limit=64 << 10, codec=codec, crc=crc)
    bl = snd.sync(fused=fused)
    got = [snd.bucket(b).cpu().numpy().tobytes() for b in range(len(bl))]
    assert got == [ref.bucket(b) for b in range(ref.n_buckets)]
    assert snd.stats()["n_full"] == ref.stats["full"]
    rcv.apply_many([snd.bucket(b) for b in range(len(bl))])
    snd.commit()
    torch.cuda.synchronize()
    snd.check()
    rcv.check()
    for r, o, n in zip(rol_d, old_d, news):
        assert (host16(r) == n).all() and (host16(o) == n).all()
    # the EMIT debug path returns every element of a FULL record, like the oracle's decoder
    b0 = torch.from_numpy(np.frombuffer(ref.bucket(0), np.uint8).copy()).to(DEV)
    st, recs = oracle.bucket_decode(ref.bucket(0), cap=sum(o.size for o in olds))
    n_out = sum(r[1].size for r in recs)
    I = torch.empty(max(n_out, 1), dtype=torch.int32, device=DEV)
    V = torch.empty(max(n_out, 1), dtype=torch.int16, device=DEV)
    rcv.ctx.sync_decompress(b0, b0.numel(), I, V)
    torch.cuda.synchronize()
    rcv.check()
    assert (I[:n_out].cpu().numpy().view(np.uint32) == np.concatenate([r[1] for r in recs])).all()
    assert (V[:n_out].cpu().numpy().view(np.uint16) == np.concatenate([r[2] for r in recs])).all()


def test_routing_needs_current_weights():
    m = mixed_manifest()
    ctx = ss.SyncContext(m.numel, route=True, device=DEV, max_changed=1000)
    I = torch.zeros(1000, dtype=torch.int32, device=DEV)
    V = torch.zeros(1000, dtype=torch.int16, device=DEV)
    counts = torch.zeros(len(m.numel), dtype=torch.int64, device=DEV)
    buf = torch.zeros(1 << 16, dtype=torch.uint8, device=DEV)
    with pytest.raises(ss.SyncError) as e:
        ctx.sync_compress_pack(I, V, counts, buf)
    assert e.value.code == ss.SYNC_ERR_ARG


@pytest.mark.parametrize("codec", [ss.SYNC_CODEC_COMPRESSED, ss.SYNC_CODEC_RAW])
def test_fp16_bit_exact_and_tag_checked(codec):
    """f2 FP16: synthetic FP16 weights (GPU generator == CPU twin), GPU buckets == the oracle's FP16
    buckets, an FP16 replica reconstructs them; a BF16 receiver rejects them (SYNC_ERR_DTYPE, no write)."""
    import synth.gpu as sg
    m = mixed_manifest()
    olds, news = synth.generate(m, seed=31, rho=0.03, dtype=synth.DTYPE_FP16)
    _, views = sg.arena(m, DEV)
    _, nviews = sg.arena(m, DEV)
    sg.fill_old(views, m, 31, dtype=synth.DTYPE_FP16)
    sg.fill_new(views, nviews, m, 31, 0.03)
    assert all((host16(v) == o).all() for v, o in zip(views, olds))
    assert all((host16(v) == n).all() for v, n in zip(nviews, news))
    ref = oracle.sync_pack(olds, news, codec=codec, limit=32 << 10, dtype=oracle.DTYPE_FP16)
    snd = ss.SparseSyncSender(views, nviews, bucket_limit=32 << 10, codec=codec, dtype=ss.SYNC_DTYPE_FP16,
                              max_changed=sum(o.size for o in olds))
    bl = snd.sync()
    got = [snd.bucket(b).cpu().numpy().tobytes() for b in range(len(bl))]
    assert got == [ref.bucket(b) for b in range(ref.n_buckets)]
    R = [to_dev(o) for o in olds]
    rcv = ss.SparseSyncReceiver(R, bucket_limit=32 << 10, codec=codec, dtype=ss.SYNC_DTYPE_FP16)
    rcv.apply_many([snd.bucket(b) for b in range(len(bl))])
    torch.cuda.synchronize()
    rcv.check()
    assert all((host16(r) == n).all() for r, n in zip(R, news))
    B = [to_dev(o) for o in olds]
    wrong = ss.SparseSyncReceiver(B, bucket_limit=32 << 10, codec=codec)     # a BF16 context
    wrong.apply_many([snd.bucket(b) for b in range(len(bl))])
    torch.cuda.synchronize()
    assert wrong.ctx.sync_status() == ss.SYNC_ERR_DTYPE
    assert all((host16(b) == o).all() for b, o in zip(B, olds))


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("crc", [False, True])
def test_escape_delta16_bit_exact(fused, crc):
    """f4: on the clustered-row mask, records with gaps > 32767 are coded DELTA16E — GPU buckets
    == the oracle's, the replica applies them, the EMIT path returns the oracle's (I, V), and a damaged
    word-offset table is detected."""
    m = synth.Manifest("r", [synth.Tensor(f"w{k}", (300, 2048)) for k in range(3)] +
                       [synth.Tensor("n", (2048,), synth.KIND_NORM), synth.Tensor("big", (64, 40000))])
    olds, news = synth.generate(m, seed=41, rho=0.02, mask=synth.MASK_R)
    ref = oracle.sync_pack(olds, news, limit=96 << 10, crc=crc, escape=True)
    assert ref.stats["delta16e"] >= 3
    old_d = [to_dev(o) for o in olds]
    new_d = [to_dev(n) for n in news]
    rol_d = [to_dev(o) for o in olds]
    snd = ss.SparseSyncSender(old_d, new_d, bucket_limit=96 << 10, crc=crc, escape=True,
                              max_changed=sum(o.size for o in olds))
    rcv = ss.SparseSyncReceiver(rol_d, bucket_limit=96 << 10, crc=crc)
    bl = snd.sync(fused=fused)
    got = [snd.bucket(b).cpu().numpy().tobytes() for b in range(len(bl))]
    assert got == [ref.bucket(b) for b in range(ref.n_buckets)]
    assert snd.stats()["n_delta16e"] == ref.stats["delta16e"]
    rcv.apply_many([snd.bucket(b) for b in range(len(bl))])
    snd.commit()
    torch.cuda.synchronize()
    snd.check()
    rcv.check()
    for r, o, n in zip(rol_d, old_d, news):
        assert (host16(r) == n).all() and (host16(o) == n).all()
    for b in range(ref.n_buckets):
        st, recs = oracle.bucket_decode(ref.bucket(b), cap=sum(o.size for o in olds))
        n_out = sum(r[1].size for r in recs)
        I = torch.empty(max(n_out, 1), dtype=torch.int32, device=DEV)
        V = torch.empty(max(n_out, 1), dtype=torch.int16, device=DEV)
        bk = torch.from_numpy(np.frombuffer(ref.bucket(b), np.uint8).copy()).to(DEV)
        rcv.ctx.sync_decompress(bk, bk.numel(), I, V)
        torch.cuda.synchronize()
        rcv.check()
        assert (I[:n_out].cpu().numpy().view(np.uint32) == np.concatenate([r[1] for r in recs])).all()
        assert (V[:n_out].cpu().numpy().view(np.uint16) == np.concatenate([r[2] for r in recs])).all()
    if not crc:   # damage the first DELTA16E record's chunk-1 word offset
        for b in range(ref.n_buckets):
            a = np.frombuffer(ref.bucket(b), np.uint8).copy()
            nrec = int(a[12:16].view(np.uint32)[0])
            ros = [int(x) for x in a[32:32 + 8 * nrec].view(np.uint32)[0::2]]
            hit = [ro for ro in ros if a[ro + 12] == 3 and int(a[ro + 4:ro + 8].view(np.uint32)[0]) > 16384]
            if hit:
                ro = hit[0]
                a[ro + 20] ^= 1
                W = [to_dev(o) for o in olds]
                bad = ss.SparseSyncReceiver(W, bucket_limit=96 << 10)
                bad.apply(torch.from_numpy(a).to(DEV))
                torch.cuda.synchronize()
                assert bad.ctx.sync_status() == ss.SYNC_ERR_CORRUPT
                break
        else:
            pytest.fail("no multi-chunk DELTA16E record to damage")


@pytest.mark.parametrize("codec,escape,route,crc", [(ss.SYNC_CODEC_COMPRESSED, False, False, False),
                                                     (ss.SYNC_CODEC_COMPRESSED, True, True, True),
                                                     (ss.SYNC_CODEC_RAW, False, True, False)])
@pytest.mark.parametrize("fused", [True, False])
def test_fp8_bit_exact(codec, escape, route, crc, fused):
    """f2 FP8 E4M3 (8-bit elements): GPU generator == CPU twin; extraction, one-plane records,
    FULL / escape records, CRC: GPU buckets == the oracle's; replica and snapshot commit bit-exact."""
    import synth.gpu as sg
    m = synth.Manifest("f8", [synth.Tensor("a", (300, 512)), synth.Tensor("n", (64,), synth.KIND_NORM),
                              synth.Tensor("b", (70_000,)), synth.Tensor("c", (64, 40000)), synth.Tensor("z", (0,)),
                              synth.Tensor("t", (33,))])
    mask = synth.MASK_R if escape else synth.MASK_U
    olds, news = synth.generate(m, seed=51, rho=0.03, mask=mask, dtype=synth.DTYPE_FP8)
    _, ov = sg.arena(m, DEV, dtype=torch.uint8)
    _, nv = sg.arena(m, DEV, dtype=torch.uint8)
    sg.fill_old(ov, m, 51, dtype=synth.DTYPE_FP8)
    sg.fill_new(ov, nv, m, 51, 0.03, mask)
    h8 = lambda x: x.cpu().numpy().reshape(-1)  # noqa: E731
    assert all((h8(v) == o).all() for v, o in zip(ov, olds))
    assert all((h8(v) == n).all() for v, n in zip(nv, news))
    if route:
        news[0] = olds[0] ^ np.uint8(1)
        nv[0].copy_(torch.from_numpy(news[0]))
    ref = oracle.sync_pack(olds, news, codec=codec, limit=32 << 10, crc=crc, route=route, escape=escape,
                           dtype=oracle.DTYPE_FP8)
    snd = ss.SparseSyncSender(ov, nv, bucket_limit=32 << 10, codec=codec, crc=crc, route=route, escape=escape,
                              dtype=ss.SYNC_DTYPE_FP8, max_changed=sum(o.size for o in olds))
    bl = snd.sync(fused=fused)
    got = [snd.bucket(b).cpu().numpy().tobytes() for b in range(len(bl))]
    assert got == [ref.bucket(b) for b in range(ref.n_buckets)]
    R = [torch.from_numpy(o.copy()).to(DEV) for o in olds]
    rcv = ss.SparseSyncReceiver(R, bucket_limit=32 << 10, codec=codec, crc=crc, dtype=ss.SYNC_DTYPE_FP8)
    rcv.apply_many([snd.bucket(b) for b in range(len(bl))])
    snd.commit()
    torch.cuda.synchronize()
    snd.check()
    rcv.check()
    assert all((h8(r) == n).all() for r, n in zip(R, news))
    assert all((h8(o) == n).all() for o, n in zip(ov, news))


def test_delta16_abs32_boundary():
    # gap of exactly 32767 stays DELTA16, 32768 forces ABS32 (DESIGN C4)
    n = 70_000
    olds = [np.zeros(n, np.uint16), np.zeros(n, np.uint16), np.zeros(n, np.uint16)]
    news = [o.copy() for o in olds]
    news[0][[32767, 65534]] = 5
    news[1][[32768]] = 5
    news[2][[0, 32767 + 0, 32767 + 32768]] = 5
    ref = oracle.sync_pack(olds, news, limit=1 << 20)
    _, _, rol, got = run_path(olds, news, ss.SYNC_CODEC_COMPRESSED, 1 << 20, False)
    assert got == [ref.bucket(b) for b in range(ref.n_buckets)]
    assert ref.stats["delta16"] == 1 and ref.stats["abs32"] == 2


def test_gpu_decoder_applies_oracle_buckets():
    """Decoder checked independently of the GPU encoder: apply the oracle's bytes."""
    m = mixed_manifest()
    olds, news = synth.generate(m, seed=2, rho=0.05)
    for codec in [ss.SYNC_CODEC_COMPRESSED, ss.SYNC_CODEC_RAW]:
        ref = oracle.sync_pack(olds, news, codec=codec, limit=32 << 10, crc=True)
        W = [to_dev(o) for o in olds]
        rcv = ss.SparseSyncReceiver(W, crc=True, codec=codec)
        for b in range(ref.n_buckets):
            bk = torch.from_numpy(np.frombuffer(ref.bucket(b), np.uint8).copy()).to(DEV)
            rcv.apply(bk)
        torch.cuda.synchronize()
        rcv.check()
        for w, n in zip(W, news):
            assert (host16(w) == n).all()


@pytest.mark.parametrize("crc", [False, True])
def test_batched_decoder_applies_oracle_buckets(crc):
    """sync_decompress_apply_batched over > 32 oracle buckets (two launches), given in shuffled order:
    the buckets of one sync touch disjoint records, so any order yields the new weights bit-exactly."""
    m = mixed_manifest()
    olds, news = synth.generate(m, seed=12, rho=0.05)
    ref = oracle.sync_pack(olds, news, limit=1024, crc=crc)
    assert ref.n_buckets > 32
    W = [to_dev(o) for o in olds]
    rcv = ss.SparseSyncReceiver(W, crc=crc, bucket_limit=1024)
    dev = [torch.from_numpy(np.frombuffer(ref.bucket(b), np.uint8).copy()).to(DEV) for b in range(ref.n_buckets)]
    order = np.random.default_rng(0).permutation(len(dev))
    rcv.apply_many([dev[k] for k in order])
    torch.cuda.synchronize()
    rcv.check()
    for w, n in zip(W, news):
        assert (host16(w) == n).all()


@pytest.mark.parametrize("rho", [0.004, 0.3])
def test_decoder_variants_apply_oracle_buckets(rho):
    """Both decode launch variants (chosen per call from payload bytes per model element, so one
    call over all buckets of a dense sync takes the high-occupancy one and a call per small bucket the other)
    apply the oracle's buckets bit-exactly."""
    m = mixed_manifest()
    olds, news = synth.generate(m, seed=21, rho=rho)
    ref = oracle.sync_pack(olds, news, limit=16 << 10)
    dev = [torch.from_numpy(np.frombuffer(ref.bucket(b), np.uint8).copy()).to(DEV) for b in range(ref.n_buckets)]
    for batched in (True, False):
        W = [to_dev(o) for o in olds]
        rcv = ss.SparseSyncReceiver(W, bucket_limit=16 << 10)
        if batched:
            rcv.apply_many(dev)
        else:
            for bk in dev:
                rcv.apply(bk)
        torch.cuda.synchronize()
        rcv.check()
        for w, n in zip(W, news):
            assert (host16(w) == n).all()


def test_batched_decoder_isolates_a_bad_bucket():
    """With CRC on, a corrupted bucket inside a batch is rejected (SYNC_ERR_CRC, none of its records applied)
    while the other buckets of the same launch are applied."""
    m = mixed_manifest()
    olds, news = synth.generate(m, seed=13, rho=0.05)
    ref = oracle.sync_pack(olds, news, limit=4096, crc=True)
    bks = [np.frombuffer(ref.bucket(b), np.uint8).copy() for b in range(ref.n_buckets)]
    bad = len(bks) // 2
    bks[bad][len(bks[bad]) // 2] ^= 1
    W = [to_dev(o) for o in olds]
    rcv = ss.SparseSyncReceiver(W, crc=True, bucket_limit=4096)
    rcv.apply_many([torch.from_numpy(b).to(DEV) for b in bks])
    torch.cuda.synchronize()
    assert rcv.ctx.sync_status() == ss.SYNC_ERR_CRC
    # expected: the oracle applies every bucket except the bad one
    exp = [o.copy() for o in olds]
    for b in range(ref.n_buckets):
        if b != bad:
            assert oracle.bucket_apply(ref.bucket(b), exp) == oracle.OK
    for w, e in zip(W, exp):
        assert (host16(w) == e).all()


def test_decompress_emits_extract():
    m = mixed_manifest()
    olds, news = synth.generate(m, seed=3, rho=0.1)
    ref = oracle.sync_pack(olds, news, limit=1 << 30)
    ctx = ss.SyncContext([t.numel for t in m.tensors], bucket_limit=1 << 30)
    bk = torch.from_numpy(np.frombuffer(ref.bucket(0), np.uint8).copy()).to(DEV)
    cap = sum(t.numel for t in m.tensors)
    I = torch.empty(cap, dtype=torch.int32, device=DEV)
    V = torch.empty(cap, dtype=torch.int16, device=DEV)
    ctx.sync_decompress(bk, bk.numel(), I, V)
    views = torch.zeros(32 * len(m.tensors), dtype=torch.uint8, device=DEV)
    nrec = torch.zeros(1, dtype=torch.int32, device=DEV)
    ctx.sync_bucket_unpack(bk, bk.numel(), views, nrec)
    torch.cuda.synchronize()
    ctx.check()
    st, recs = oracle.bucket_decode(ref.bucket(0), cap=cap)
    assert st == oracle.OK and int(nrec.item()) == len(recs)
    vv = views.cpu().numpy().view(np.uint32).reshape(-1, 8)
    off = 0
    Ih, Vh = I.cpu().numpy().view(np.uint32), host16(V)
    for q, (tid, Io, Vo) in enumerate(recs):
        assert vv[q, 0] == tid and vv[q, 1] == Io.size
        assert (Ih[off:off + Io.size] == Io).all() and (Vh[off:off + Io.size] == Vo).all()
        off += Io.size


def test_apply_and_commit_vs_oracle():
    rng = np.random.default_rng(5)
    n = 200_000
    W0 = rng.integers(0, 65536, n, dtype=np.uint16)
    I = np.unique(rng.integers(0, n, 20_000)).astype(np.uint32)
    V = rng.integers(0, 65536, I.size, dtype=np.uint16)
    Wo = W0.copy()
    assert oracle.apply(Wo, I, V) == oracle.OK
    for fn in (ss.sync_apply, ss.sync_commit_snapshot):
        Wd = to_dev(W0)
        st = torch.zeros(1, dtype=torch.int32, device=DEV)
        fn(Wd, torch.from_numpy(I.view(np.int32)).to(DEV), to_dev(V), status=st)
        torch.cuda.synchronize()
        assert int(st.item()) == 0 and (host16(Wd) == Wo).all()
    # out of range: skipped and latched
    Wd = to_dev(W0)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    bad = np.array([1, n + 5, 3], np.uint32)
    ss.sync_apply(Wd, torch.from_numpy(bad.view(np.int32)).to(DEV), to_dev(np.array([7, 8, 9], np.uint16)), status=st)
    torch.cuda.synchronize()
    assert -int(st.item()) == ss.SYNC_ERR_INDEX_RANGE
    h = host16(Wd)
    assert h[1] == 7 and h[3] == 9


def rans_word_offset(bk: np.ndarray) -> int:
    """Byte offset (in the bucket) of a middle rANS word of the first RANS chunk with >= 16 words."""
    u32 = lambda o: int(bk[o:o + 4].view(np.uint32)[0])
    nrec = u32(12)
    for q in range(nrec):
        ro = u32(32 + 8 * q)
        nnz, mode = u32(ro + 4), int(bk[ro + 12])
        ib = (4 if mode else 2) * nnz
        dir_off = ro + 16 + (ib + 3) // 4 * 4 + (nnz + 3) // 4 * 4
        for k in range((nnz + 16383) // 16384):
            hi_off, hb, cm = u32(dir_off + 16 * k), u32(dir_off + 16 * k + 4), u32(dir_off + 16 * k + 8)
            if cm == 1:
                blk = ro + hi_off
                nwords, nsym = u32(blk + 128), u32(blk + 132) & 0xFFFF
                if nwords >= 16:
                    return blk + 136 + 4 * nsym + 2 * (nwords // 2)
    raise AssertionError("no rANS chunk with words")


def test_corruption_is_detected():
    m = mixed_manifest()
    olds, news = synth.generate(m, seed=4, rho=0.05)
    ref = oracle.sync_pack(olds, news, limit=1 << 30, crc=True)
    good = np.frombuffer(ref.bucket(0), np.uint8).copy()
    cases = []
    b = good.copy(); b[len(b) // 2] ^= 1; cases.append((b, True, ss.SYNC_ERR_CRC))
    b = good.copy(); b[0] ^= 1; cases.append((b, True, ss.SYNC_ERR_BAD_MAGIC))
    b = good.copy(); b[4] = 2; cases.append((b, True, ss.SYNC_ERR_VERSION))
    # without CRC: damage a rANS word deep inside the big record -> end-state check
    ref2 = oracle.sync_pack(olds, news, limit=1 << 30, crc=False)
    g2 = np.frombuffer(ref2.bucket(0), np.uint8).copy()
    b = g2.copy(); b[rans_word_offset(g2) + 1] ^= 0x55; cases.append((b, False, ss.SYNC_ERR_CORRUPT))
    for data, crc, want in cases:
        W = [to_dev(o) for o in olds]
        rcv = ss.SparseSyncReceiver(W, crc=crc)
        rcv.apply(torch.from_numpy(data).to(DEV))
        torch.cuda.synchronize()
        assert rcv.ctx.sync_status() == want


def test_config1_one_million_end_to_end():
    """BASELINE config 1: one 2^20-element bf16 tensor, 99% sparsity, uniform mask."""
    m = synth.single_manifest(1 << 20)
    olds, news = synth.generate(m, seed=0, rho=0.01)
    ref = oracle.sync_pack(olds, news, limit=256 << 20)
    snd, old_d, rol_d, got = run_path(olds, news, ss.SYNC_CODEC_COMPRESSED, 256 << 20, False)
    assert got == [ref.bucket(b) for b in range(ref.n_buckets)]
    assert (host16(rol_d[0]) == news[0]).all()
    x_comp = 2 * (1 << 20) / sum(len(g) for g in got)
    assert 55 < x_comp < 65                      # ≈ 60x at ρ = 1% (Eq. 4, α ≈ 0.67)


# ----------------------------------------------------------------------------- maximum tensor size
NMAX = (1 << 31) - 1   # largest numel the format allows (DESIGN C2: tensor-local u32 index < 2^31)


@pytest.mark.parametrize("mode", ["abs32", "delta16e", "delta16"])
def test_max_numel_tensor_bit_exact(mode):
    """One tensor of 2^31 - 1 elements with changes at both ends and between: extract is the definition (the
    changed positions are the input), the buckets equal the oracle's byte for byte and the replica is
    bit-identical. abs32 / delta16e: 3000 scattered changes (gaps ~ 2^31 / 3000 > 32767: ABS32, or DELTA16E
    with an escape pair per gap); delta16: every 30000th element (71.6K changes, 5 chunks whose base
    indices run up to 2^31 - 1)."""
    rng = np.random.default_rng(31)
    escape = mode == "delta16e"
    if mode == "delta16":
        pos = np.concatenate([np.arange(0, NMAX, 30000), [NMAX - 1]]).astype(np.int64)
    else:
        pos = np.unique(np.concatenate([rng.integers(0, NMAX, 3000), [0, 1, NMAX - 2, NMAX - 1]])).astype(np.int64)
    val = rng.integers(1, 65536, pos.size, dtype=np.uint16)
    old_h = np.zeros(NMAX, np.uint16)
    new_h = old_h.copy()
    new_h[pos] = val                      # old is all zero and val != 0: every listed position changes
    old = torch.zeros(NMAX, dtype=torch.int16, device=DEV)
    new = torch.from_numpy(new_h.view(np.int16)).to(DEV)
    cap = 1 << 17
    I, V, cnt, ws = ss.sync_extract(old, new, I=torch.empty(cap, dtype=torch.int32, device=DEV),
                                    V=torch.empty(cap, dtype=torch.int16, device=DEV))
    torch.cuda.synchronize()
    assert ss.sync_extract_status(ws) == ss.SYNC_OK
    c = int(cnt.item())
    assert c == pos.size
    assert (I[:c].cpu().numpy().view(np.uint32) == pos.astype(np.uint32)).all()
    assert (host16(V[:c]) == val).all()
    ref = oracle.sync_pack([old_h], [new_h], limit=64 << 20, crc=True, escape=escape)
    assert ref.stats[mode] == 1
    rol = old.clone()
    snd = ss.SparseSyncSender([old], [new], bucket_limit=64 << 20, crc=True, escape=escape, max_changed=cap)
    rcv = ss.SparseSyncReceiver([rol], bucket_limit=64 << 20, crc=True)
    bl = snd.sync()
    assert [snd.bucket(b).cpu().numpy().tobytes() for b in range(len(bl))] == \
        [ref.bucket(b) for b in range(ref.n_buckets)]
    for b in range(len(bl)):
        rcv.apply(snd.bucket(b))
    torch.cuda.synchronize()
    snd.check()
    rcv.check()
    assert torch.equal(rol, new)


def test_numel_2_31_is_rejected():
    big = torch.zeros(1 << 31, dtype=torch.int16, device=DEV)
    small = torch.empty(16, dtype=torch.int32, device=DEV)
    with pytest.raises(ss.SyncError):
        ss.sync_extract(big, big, I=small, V=small.view(torch.int16)[:16])
    with pytest.raises(ss.SyncError):
        ss.SparseSyncSender([big], [big], max_changed=16)


@pytest.mark.parametrize("off", [0, 8, 1, 3])
@pytest.mark.parametrize("rho,mask", [(0.01, synth.MASK_U), (0.3, synth.MASK_U), (0.02, synth.MASK_R)])
def test_iv_views_alignment_contract(off, rho, mask):
    """I / V must be 16-byte aligned (include/sparsesync.h; k_chunk_stats and k_encode use 16- / 8-byte vector
    loads of them): views at a 16-byte multiple give the oracle's bytes (ABS32 records under the R mask, dense
    chunks at 30%); any other offset is refused with SYNC_ERR_ALIGNMENT before a kernel runs."""
    m = mixed_manifest()
    olds, news = synth.generate(m, seed=5, rho=rho, mask=mask)
    old_d = [to_dev(o) for o in olds]
    new_d = [to_dev(n) for n in news]
    snd = ss.SparseSyncSender(old_d, new_d, bucket_limit=64 << 10)
    cap = snd.cap
    bi = torch.empty(cap + 8, dtype=torch.int32, device=DEV)
    bv = torch.empty(cap + 8, dtype=torch.int16, device=DEV)
    snd.I, snd.V = bi[off:off + cap], bv[off:off + cap]
    if off % 8:
        with pytest.raises(ss.SyncError) as e:
            snd.sync(fused=True)
        assert e.value.code == ss.SYNC_ERR_ALIGNMENT
        return
    ref = oracle.sync_pack(olds, news, codec=ss.SYNC_CODEC_COMPRESSED, limit=64 << 10, crc=False)
    bl = snd.sync(fused=True)
    torch.cuda.synchronize()
    snd.check()
    assert len(bl) == ref.n_buckets
    for b in range(ref.n_buckets):
        assert snd.bucket(b).cpu().numpy().tobytes() == ref.bucket(b), f"off={off}: bucket {b} bytes differ"
