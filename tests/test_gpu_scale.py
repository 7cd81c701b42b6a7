"""GPU <-> oracle parity at the control-path sizes of the full manifests, and K1 forward progress.

VERDICT r1 W1/W2: the single-CTA plan kernels (k_plan_scan, k_plan_sizes) work in rounds of 8192 tensors or
chunks and k_unpack in rounds of 1024 records; the 30B manifest has 18,867 records (3 rounds) and the 235B one
36,945. These tests drive every one of those loops past round 1 and compare the bucket bytes with the oracle
(bit-exact: DESIGN C17 — one correct byte string per input). K1 is run with many tiles per CTA (the dense
overflow path and the FP8 instantiation included) via sync_set_max_ctas, and under a kernel that holds half
of the SMs for the whole launch (it must finish without every CTA co-resident).
"""
import time

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

ss = pytest.importorskip("paper_2605_07330_b200")
DEV = "cuda:0"


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_07330_b200 import build
    build.build()
    torch.cuda.set_device(0)
    yield
    ss.set_max_ctas(0)


def to_dev(a: np.ndarray) -> torch.Tensor:
    if a.dtype == np.uint8:
        return torch.from_numpy(a.copy()).to(DEV)
    return torch.from_numpy(a.view(np.int16).copy()).to(DEV)


def host(t: torch.Tensor) -> np.ndarray:
    a = t.cpu().numpy()
    return a if a.dtype == np.uint8 else a.view(np.uint16)


# ----------------------------------------------------------------------------- many records / chunks
T_SMALL = 20_480


def many_manifest():
    """20,480 small tensors (every one changes: 20.5K records and chunks -> 3 rounds of k_plan_scan and of both
    k_plan_sizes loops), 3 large tensors with escapes (gaps > 32767), dense tensors (FULL under routing)."""
    rng = np.random.default_rng(7)
    T = [synth.Tensor(f"s{k}", (int(rng.integers(1, 65)) * 8,)) for k in range(T_SMALL)]
    T[5] = synth.Tensor("empty", (0,))
    T += [synth.Tensor("wide0", (300_000,)), synth.Tensor("wide1", (1_000_008,)), synth.Tensor("dense", (70_000,))]
    return synth.Manifest("many", T)


_MANY = {}


def many_inputs():
    if "x" not in _MANY:
        m = many_manifest()
        olds, news = synth.generate(m, seed=11, rho=0.2)
        for k in range(0, T_SMALL, 97):                     # dense small tensors (FULL under routing)
            news[k] = olds[k] ^ np.uint16(1)
        for name, step in (("wide0", 40_000), ("wide1", 33_000)):   # gaps > 32767: ABS32 / DELTA16E
            k = [t.name for t in m.tensors].index(name)
            news[k] = olds[k].copy()
            news[k][7::step] ^= np.uint16(3)
            news[k][100:20_000:5] ^= np.uint16(1)          # plus a dense run (several chunks)
        k = [t.name for t in m.tensors].index("dense")
        news[k] = olds[k] ^ np.uint16(2)
        _MANY["x"] = (m, olds, news)
    return _MANY["x"]


@pytest.mark.parametrize("codec,crc,escape,route,limit,fused", [
    (ss.SYNC_CODEC_COMPRESSED, False, False, False, 1 << 30, True),
    (ss.SYNC_CODEC_COMPRESSED, True, True, False, 1 << 30, False),
    (ss.SYNC_CODEC_COMPRESSED, True, True, True, 64 << 10, True),
    (ss.SYNC_CODEC_COMPRESSED, False, False, True, 1 << 30, False),
    (ss.SYNC_CODEC_RAW, True, False, False, 1 << 30, True),
    (ss.SYNC_CODEC_RAW, False, False, True, 256 << 10, False),
])
def test_many_records_bucket_bytes_bit_exact(codec, crc, escape, route, limit, fused):
    m, olds, news = many_inputs()
    ref = oracle.sync_pack(olds, news, codec=codec, limit=limit, crc=crc, route=route, escape=escape)
    assert ref.stats["n_records"] > 2 * 8192                 # rounds >= 3 of the record loops
    old_d = [to_dev(o) for o in olds]
    new_d = [to_dev(n) for n in news]
    rol_d = [to_dev(o) for o in olds]
    snd = ss.SparseSyncSender(old_d, new_d, bucket_limit=limit, codec=codec, crc=crc, route=route, escape=escape,
                              max_changed=sum(o.size for o in olds))
    rcv = ss.SparseSyncReceiver(rol_d, bucket_limit=limit, codec=codec, crc=crc)
    bl = snd.sync(fused=fused)
    st = snd.stats()
    assert st["n_chunks"] > 9000 or codec == ss.SYNC_CODEC_RAW
    assert st["nnz"] == ref.stats["nnz"] and st["n_records"] == ref.stats["n_records"]
    assert len(bl) == ref.n_buckets
    for b in range(ref.n_buckets):
        assert snd.bucket(b).cpu().numpy().tobytes() == ref.bucket(b), f"bucket {b} differs from the oracle"
    if limit == 1 << 30:
        assert ref.n_buckets == 1                            # > 20K records in one bucket: k_unpack rounds
    if escape:
        assert st["n_delta16e"] >= 2
    if route:
        assert st["n_full"] == ref.stats["full"] >= T_SMALL // 97
    rcv.apply_many([snd.bucket(b) for b in range(len(bl))])
    snd.commit()
    torch.cuda.synchronize()
    snd.check()
    rcv.check()
    for r, o, n in zip(rol_d, old_d, news):
        assert (host(r) == n).all() and (host(o) == n).all()


def test_many_records_unpack_and_decompress_vs_oracle():
    """sync_bucket_unpack + sync_decompress on one bucket of > 20K records (k_unpack rounds >= 20, the decoder's
    record table past 1024 entries): every view (tensor id, nnz, offset, bytes, out_offset) and every emitted
    (I, V) equals the oracle's decode of the same bucket."""
    m, olds, news = many_inputs()
    ref = oracle.sync_pack(olds, news, limit=1 << 30, escape=True)
    buf = ref.bucket(0)
    cap = sum(o.size for o in olds)
    st, recs = oracle.bucket_decode(buf, cap=cap)
    assert st == oracle.OK and len(recs) > 20_000
    ctx = ss.SyncContext(m.numel, bucket_limit=1 << 30, device=DEV, max_changed=cap, escape=True)
    bk = torch.from_numpy(np.frombuffer(buf, np.uint8).copy()).to(DEV)
    views = torch.zeros(32 * len(recs), dtype=torch.uint8, device=DEV)
    nrec = torch.zeros(1, dtype=torch.int32, device=DEV)
    ctx.sync_bucket_unpack(bk, bk.numel(), views, nrec)
    I = torch.empty(cap, dtype=torch.int32, device=DEV)
    V = torch.empty(cap, dtype=torch.int16, device=DEV)
    ctx.sync_decompress(bk, bk.numel(), I, V)
    torch.cuda.synchronize()
    ctx.check()
    assert int(nrec.item()) == len(recs)
    vv = views.cpu().numpy().view(np.uint32).reshape(-1, 8)
    tids = np.array([r[0] for r in recs], np.uint32)
    sizes = np.array([r[1].size for r in recs], np.uint64)
    assert (vv[:, 0] == tids).all() and (vv[:, 1] == sizes).all()
    out_off = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.uint64)
    assert (vv[:, 6].astype(np.uint64) | (vv[:, 7].astype(np.uint64) << np.uint64(32)) == out_off).all()
    rec_off = vv[:, 2].astype(np.int64)
    rec_len = vv[:, 3].astype(np.int64)
    hdr = np.frombuffer(buf, np.uint32)
    for q in (0, 1, len(recs) // 2, len(recs) - 1):          # each view points at that record's header
        o = int(rec_off[q])
        assert hdr[o // 4] == tids[q] and hdr[o // 4 + 2] == rec_len[q]
    assert (rec_off[1:] == rec_off[:-1] + rec_len[:-1]).all()
    Ih, Vh = I.cpu().numpy().view(np.uint32), host(V)
    Io = np.concatenate([r[1] for r in recs])
    Vo = np.concatenate([r[2] for r in recs])
    assert (Ih[:Io.size] == Io).all() and (Vh[:Vo.size] == Vo).all()


# ----------------------------------------------------------------------------- K1: many tiles per CTA
@pytest.mark.parametrize("ctas", [1, 3, 37])
@pytest.mark.parametrize("rho", [0.01, 0.3, 1.0])
@pytest.mark.parametrize("dtype", ["bf16", "fp8"])
def test_extract_many_tiles_per_cta(ctas, rho, dtype):
    """n_tiles >> grid (a CTA walks tens of tiles, its writer window spans other CTAs' tiles): the sparse
    staging path (rho = 1%), the dense overflow path (> 12.5% of a tile) and the FP8 instantiation; GPU bucket
    bytes and replica == the oracle's."""
    fp8 = dtype == "fp8"
    m = synth.Manifest("tiles", [synth.Tensor("a", (1000, 1024)), synth.Tensor("n", (64,), synth.KIND_NORM),
                                 synth.Tensor("b", (3_000_001 // 8 * 8,)), synth.Tensor("c", (24,)),
                                 synth.Tensor("d", (65_536 + 40,))])
    dt = synth.DTYPE_FP8 if fp8 else synth.DTYPE_BF16
    olds, news = synth.generate(m, seed=int(rho * 100) + ctas, rho=rho, dtype=dt)
    kw = dict(dtype=oracle.DTYPE_FP8) if fp8 else {}
    ref = oracle.sync_pack(olds, news, limit=4 << 20, **kw)
    old_d = [to_dev(o) for o in olds]
    new_d = [to_dev(n) for n in news]
    rol_d = [to_dev(o) for o in olds]
    skw = dict(dtype=ss.SYNC_DTYPE_FP8) if fp8 else {}
    ss.set_max_ctas(ctas)
    try:
        snd = ss.SparseSyncSender(old_d, new_d, bucket_limit=4 << 20, max_changed=sum(o.size for o in olds), **skw)
        rcv = ss.SparseSyncReceiver(rol_d, bucket_limit=4 << 20, **skw)
        bl = snd.sync()
        got = [snd.bucket(b).cpu().numpy().tobytes() for b in range(len(bl))]
        rcv.apply_many([snd.bucket(b) for b in range(len(bl))])
        snd.commit()
        torch.cuda.synchronize()
        snd.check()
        rcv.check()
    finally:
        ss.set_max_ctas(0)
    assert sum((o.size + 32767) // 32768 for o in olds) >= 3 * ctas   # 129 tiles: >= 3 per CTA
    assert got == [ref.bucket(b) for b in range(ref.n_buckets)]
    for r, o, n in zip(rol_d, old_d, news):
        assert (host(r) == n).all() and (host(o) == n).all()


@pytest.mark.parametrize("ctas", [1, 5])
def test_extract_single_many_tiles_per_cta(ctas):
    n = 2_500_003
    rng = np.random.default_rng(ctas)
    old = rng.integers(0, 65536, n, dtype=np.uint16)
    new = old.copy()
    msk = rng.random(n) < 0.2
    new[msk] ^= np.uint16(5)
    ss.set_max_ctas(ctas)
    try:
        I, V, cnt, ws = ss.sync_extract(to_dev(old), to_dev(new))
        torch.cuda.synchronize()
        assert ss.sync_extract_status(ws) == ss.SYNC_OK
    finally:
        ss.set_max_ctas(0)
    Io, Vo = oracle.extract(old, new)
    c = int(cnt.item())
    assert c == Io.size
    assert (I[:c].cpu().numpy().view(np.uint32) == Io).all() and (host(V[:c]) == Vo).all()


# ----------------------------------------------------------------------------- K1 forward progress
def test_extract_finishes_while_half_the_sms_are_held():
    """A kernel on another stream holds half of the SMs (one 200 KB-shared-memory CTA per SM) until K1 has
    finished. K1's default grid (SMs x 2) can then never be co-resident; with ticketed tiles it must still
    finish. The holder is released after K1 completes — or after 60 s, so a regression fails
    the test instead of hanging the GPU."""
    from gpuhelpers import spin_lib
    L = spin_lib()
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    hold = n_sm // 2
    m = synth.Manifest("fp", [synth.Tensor("a", (4096, 4096)), synth.Tensor("b", (16_000_000,)),
                              synth.Tensor("c", (2048, 2048))])
    olds, news = synth.generate(m, seed=3, rho=0.01)
    old_d = [to_dev(o) for o in olds]
    new_d = [to_dev(n) for n in news]
    snd = ss.SparseSyncSender(old_d, new_d, bucket_limit=64 << 20, max_changed=sum(o.size for o in olds))
    torch.cuda.synchronize()
    s_hold = torch.cuda.Stream()
    s_work = torch.cuda.Stream()
    assert L.spin_start(hold, 200 * 1024, ctypes_stream(s_hold)) == 0
    t0 = time.time()
    while L.spin_started() < hold and time.time() - t0 < 30:
        time.sleep(0.01)
    started = L.spin_started()
    ev = torch.cuda.Event()
    finished = False
    try:
        assert started == hold, f"only {started}/{hold} holder CTAs started"
        with torch.cuda.stream(s_work):
            snd.extract_compress(stream=s_work)
            ev.record(s_work)
        t1 = time.time()
        while time.time() - t1 < 60:
            if ev.query():
                finished = True
                break
            time.sleep(0.01)
        still_held = L.spin_started() == hold
    finally:
        L.spin_release()
        torch.cuda.synchronize()
    assert finished, "K1 did not finish while half of the SMs were held (needs co-residency)"
    assert still_held
    bl = snd.pack()
    ref = oracle.sync_pack(olds, news, limit=64 << 20)
    assert [snd.bucket(b).cpu().numpy().tobytes() for b in range(len(bl))] == \
        [ref.bucket(b) for b in range(ref.n_buckets)]


def ctypes_stream(s):
    import ctypes
    return ctypes.c_void_p(s.cuda_stream)


# ----------------------------------------------------------------------------- enqueue-only sender
def test_sender_captured_in_a_cuda_graph_matches_oracle():
    """sync_extract_batched + sync_compress_pack_async are enqueue-only (the bucket plan runs on the device and
    lands in mapped host memory): the whole sender is captured once in a CUDA graph and replayed; after each
    replay sync_pack_result returns the plan and the buckets equal the oracle's bytes."""
    m = synth.Manifest("cg", [synth.Tensor("a", (700, 512)), synth.Tensor("n", (64,), synth.KIND_NORM),
                              synth.Tensor("b", (300_001 // 8 * 8,)), synth.Tensor("c", (24,))])
    olds, news = synth.generate(m, seed=17, rho=0.02)
    L = 64 << 10
    ref = oracle.sync_pack(olds, news, limit=L, crc=True)
    old_d = [to_dev(o) for o in olds]
    new_d = [to_dev(n) for n in news]
    cap = sum(o.size for o in olds)
    ctx = ss.SyncContext(m.numel, bucket_limit=L, max_changed=cap, crc=True, device=DEV)
    op, np_ = ss.ptr_table(old_d, DEV), ss.ptr_table(new_d, DEV)
    I = torch.empty(cap, dtype=torch.int32, device=DEV)
    V = torch.empty(cap, dtype=torch.int16, device=DEV)
    counts = torch.zeros(len(olds), dtype=torch.int64, device=DEV)
    buckets = torch.zeros(4 * cap + (1 << 20), dtype=torch.uint8, device=DEV)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):        # warm-up outside the capture (first-use attributes, constant uploads)
        ctx.sync_extract_batched(op, np_, I, V, counts, stream=s)
        ctx.sync_compress_pack_async(I, V, counts, buckets, stream=s)
    s.synchronize()
    first = ctx.sync_pack_result()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ctx.sync_extract_batched(op, np_, I, V, counts, stream=s)
        ctx.sync_compress_pack_async(I, V, counts, buckets, stream=s)
    for _ in range(3):
        buckets.zero_()
        g.replay()
        torch.cuda.synchronize()
        bl = ctx.sync_pack_result()
        assert bl == first
        got = [buckets[o:o + z].cpu().numpy().tobytes() for o, z in bl]
        assert got == [ref.bucket(b) for b in range(ref.n_buckets)]
    ctx.check()


def test_bucket_plan_long_chain_and_global_walk():
    """The device bucket plan with more records than its shared-memory staging holds (> 51,200: the chain of
    bucket starts is walked from global memory) and tiny buckets (~3,900 buckets of ~14 records: the
    per-bucket scans past their first rounds of 1024): bucket bytes == the oracle's; too small a bucket table
    returns SYNC_ERR_CAPACITY and writes nothing."""
    T = 53_000
    m = synth.Manifest("chain", [synth.Tensor(f"t{k}", (16,)) for k in range(T)])
    olds, news = synth.generate(m, seed=29, rho=0.3)
    for k in range(0, T, 7):
        news[k] = olds[k] ^ np.uint16(1)          # every tensor has a change (few enough for 16 elements)
    for k in range(T):
        if (olds[k] == news[k]).all():
            news[k] = olds[k].copy()
            news[k][3] ^= np.uint16(2)
    L = 1024
    ref = oracle.sync_pack(olds, news, limit=L)
    assert ref.stats["n_records"] == T and ref.n_buckets > 2048   # > 51,200 records; several bucket-scan rounds
    old_d = [to_dev(o) for o in olds]
    new_d = [to_dev(n) for n in news]
    snd = ss.SparseSyncSender(old_d, new_d, bucket_limit=L, max_changed=16 * T)
    bl = snd.sync()
    assert len(bl) == ref.n_buckets
    for b in (0, 1, len(bl) // 2, len(bl) - 1):
        assert snd.bucket(b).cpu().numpy().tobytes() == ref.bucket(b)
    got = b"".join(snd.bucket(b).cpu().numpy().tobytes() for b in range(len(bl)))
    assert got == b"".join(ref.bucket(b) for b in range(ref.n_buckets))
    # a bucket table smaller than the plan: SYNC_ERR_CAPACITY, nothing encoded
    import ctypes
    ctx = snd.ctx
    n = ctypes.c_uint32()
    need = ctypes.c_uint64()
    code = ss.lib().sync_compress_pack(ctx._h, ss._ptr(snd.I), ss._ptr(snd.V), ss._dev_ptr(snd.counts),
                                       ss._dev_ptr(snd.buckets), snd.buckets.numel(), ctypes.byref(n), ctx._h_off,
                                       ctx._h_size, 100, ctypes.byref(need), ss._stream(None))
    assert code == ss.SYNC_ERR_CAPACITY and n.value == 0
    assert ss.lib().sync_status(ctx._h, ss._stream(None)) == ss.SYNC_ERR_CAPACITY


def test_whole_loopback_sync_in_cuda_graphs():
    """Sender and receiver with no host in the loop: extract + sync_compress_pack_async + the decode over the
    sender's device bucket table (sync_decompress_apply_table), captured as two CUDA graphs (v0 -> v1 and
    v1 -> v0, the double-buffered commit) and replayed alternately: after every replay the replica equals the
    version just synced, and the v0 -> v1 buckets equal the oracle's."""
    m = synth.Manifest("g2", [synth.Tensor("a", (700, 512)), synth.Tensor("n", (64,), synth.KIND_NORM),
                              synth.Tensor("b", (300_000,)), synth.Tensor("c", (24,))])
    olds, news = synth.generate(m, seed=41, rho=0.02)
    L = 64 << 10
    ref = oracle.sync_pack(olds, news, limit=L)
    X = [to_dev(o) for o in olds]
    Y = [to_dev(n) for n in news]
    R = [to_dev(o) for o in olds]
    cap = sum(o.size for o in olds)
    tx = ss.SyncContext(m.numel, bucket_limit=L, max_changed=cap, device=DEV)
    rx = ss.SyncContext(m.numel, bucket_limit=L, max_changed=cap, device=DEV)
    A, B = ss.ptr_table(X, DEV), ss.ptr_table(Y, DEV)
    Rp = ss.ptr_table(R, DEV)
    I = torch.empty(cap, dtype=torch.int32, device=DEV)
    V = torch.empty(cap, dtype=torch.int16, device=DEV)
    counts = torch.zeros(len(olds), dtype=torch.int64, device=DEV)
    buckets = torch.zeros(4 * cap + (1 << 20), dtype=torch.uint8, device=DEV)
    table = tx.sync_pack_table()
    s = torch.cuda.Stream()

    def sync(old, new):
        tx.sync_extract_batched(old, new, I, V, counts, stream=s)
        tx.sync_compress_pack_async(I, V, counts, buckets, stream=s)
        rx.sync_decompress_apply_table(buckets, table, 64, Rp, stream=s)

    with torch.cuda.stream(s):    # warm-up (first-use attributes) with the identity update
        sync(A, A)
    s.synchronize()
    graphs = []
    for old, new in ((A, B), (B, A)):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            sync(old, new)
        graphs.append(g)
    for k in range(4):
        graphs[k % 2].replay()
        torch.cuda.synchronize()
        want = news if k % 2 == 0 else olds
        assert all((host(r) == w).all() for r, w in zip(R, want)), f"replica after replay {k}"
        if k == 0:
            bl = tx.sync_pack_result()
            assert [buckets[o:o + z].cpu().numpy().tobytes() for o, z in bl] == \
                [ref.bucket(b) for b in range(ref.n_buckets)]
    tx.check()
    rx.check()
