"""Pins of the oracle's f2 FP16 synchronisation precision (the paper measures FP16 and FP8 update
densities next to BF16).

FP16 elements are 16-bit patterns like BF16, so every step of the path is the same integer work; only the
record's dtype tag differs (C20). Pins: FP16 records / buckets equal the (already pinned) BF16
encodings of the same bit patterns except the dtype byte; the round trip on FP16-shaped data; the value
coder's size against the empirical entropy of the FP16 hi byte (sign, 5 exponent bits, 2 mantissa bits);
the decoder accepts dtype 1 and 2 and rejects anything else.
"""
import numpy as np

import oracle
import synth


def _records(pack):
    out = []
    for b in range(pack.n_buckets):
        a = np.frombuffer(pack.bucket(b), np.uint8)
        nrec = int(a[12:16].view(np.uint32)[0])
        dirv = a[32:32 + 8 * nrec].view(np.uint32).reshape(-1, 2)
        for q in range(nrec):
            ro = int(dirv[q, 0])
            rb = int(a[ro + 8:ro + 12].view(np.uint32)[0])
            out.append(a[ro:ro + rb].copy())
    return out


def test_fp16_records_equal_bf16_encoding_but_the_tag():
    m = synth.Manifest("m", [synth.Tensor("a", (300, 200)), synth.Tensor("n", (64,), synth.KIND_NORM),
                             synth.Tensor("b", (70_000,))])
    olds, news = synth.generate(m, seed=5, rho=0.03, dtype=synth.DTYPE_FP16)
    for codec in (oracle.CODEC_RAW, oracle.CODEC_COMPRESSED):
        a = oracle.sync_pack(olds, news, codec=codec, limit=1 << 16, dtype=oracle.DTYPE_FP16)
        b = oracle.sync_pack(olds, news, codec=codec, limit=1 << 16, dtype=oracle.DTYPE_BF16)
        ra, rb = _records(a), _records(b)
        assert len(ra) == len(rb) > 0
        for x, y in zip(ra, rb):
            assert x[13] == 2 and y[13] == 1
            y = y.copy()
            y[13] = 2
            assert (x == y).all()
        W = [o.copy() for o in olds]
        for k in range(a.n_buckets):
            assert oracle.bucket_apply(a.bucket(k), W) == oracle.OK
        assert all((w == n).all() for w, n in zip(W, news))


def test_fp16_value_coder_vs_entropy():
    rng = np.random.default_rng(0)
    v = (rng.standard_normal(200_000) * 0.02).astype(np.float16).view(np.uint16)
    I = np.arange(0, 2 * v.size, 2, dtype=np.uint32)   # gap 2: DELTA16
    rec = np.frombuffer(oracle.encode_record(0, I, v, dtype=oracle.DTYPE_FP16), np.uint8)
    hi = (v >> 8).astype(np.int64)
    p = np.bincount(hi, minlength=256) / hi.size
    H = -(p[p > 0] * np.log2(p[p > 0])).sum()
    value_bytes = rec.size - 16 - 2 * v.size
    lower = v.size * (1 + H / 8)               # lo plane raw + entropy of the hi plane
    chunks = v.size // 16384 + 1                # + per chunk: directory 16, states/header 136, model <= 4*256
    assert lower <= value_bytes <= lower + 0.01 * v.size * H / 8 + (16 + 136 + 1024) * chunks


def test_decoder_dtype_tags():
    I = np.array([3, 9], np.uint32)
    V = np.array([0x3C00, 0x4000], np.uint16)
    for dt, ok in ((1, True), (2, True), (3, False), (0, False)):
        rec = bytearray(oracle.encode_record(0, I, V, dtype=1))
        rec[13] = dt
        W = [np.zeros(16, np.uint16)]
        bk = bytearray(32 + 16) + rec
        bk[0:4] = (0x424C5253).to_bytes(4, "little")
        bk[4:6] = (1).to_bytes(2, "little")
        bk[12:16] = (1).to_bytes(4, "little")
        bk[16:20] = (1).to_bytes(4, "little")
        bk[24:32] = len(bk).to_bytes(8, "little")
        bk[32:36] = (48).to_bytes(4, "little")
        st = oracle.bucket_apply(bytes(bk), W)
        assert (st == oracle.OK) == ok
        if ok:
            assert W[0][3] == 0x3C00 and W[0][9] == 0x4000
