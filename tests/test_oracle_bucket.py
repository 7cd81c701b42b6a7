"""Pins for oracle bucketing / whole sender->receiver path (rows a5, a7, a8) and the cost model.

Bucketing: DESIGN C11 with SPEC's examples. Integrity: CRC-32/IEEE
check value and zlib. Whole path: the paper's bit-exact
methodology. Payload size: Eq. (1)-(4), the worked
example and the 671B anchors.
"""
import zlib

import numpy as np
import pytest

import oracle
import synth


def test_crc32_check_value_and_zlib():
    assert oracle.crc32(b"123456789") == 0xCBF43926
    assert oracle.crc32(b"") == 0
    rng = np.random.default_rng(0)
    for n in [1, 7, 1000, 65537]:
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert oracle.crc32(b) == zlib.crc32(b)


def test_bucketize_spec_examples():
    # 10 x 1 KB records with a 4 KB limit -> at most 4 per bucket.
    # Here a bucket also holds its 32 B header and 8 B/record directory, so 3 fit (3136 B), 4 do not (4160 B).
    nb, of = oracle.bucketize([1024] * 10, 4096)
    assert nb == 4 and of.tolist() == [0, 0, 0, 1, 1, 1, 2, 2, 2, 3]
    # an oversized record sits alone; records are never split
    nb, of = oracle.bucketize([512, 10_000, 512, 512], 4096)
    assert nb == 3 and of.tolist() == [0, 1, 2, 2]
    assert oracle.bucketize([], 4096)[0] == 0


def _manifest():
    T = [synth.Tensor("a", (64, 64)), synth.Tensor("norm", (64,), synth.KIND_NORM),
         synth.Tensor("b", (3, 1000)), synth.Tensor("empty", (0,)), synth.Tensor("c", (40_000,)),
         synth.Tensor("d", (7,))]
    return synth.Manifest("mix", T)


@pytest.mark.parametrize("codec", [oracle.CODEC_RAW, oracle.CODEC_COMPRESSED])
@pytest.mark.parametrize("limit", [256, 4096, 1 << 30])
@pytest.mark.parametrize("crc", [False, True])
def test_pack_apply_bit_exact(codec, limit, crc):
    m = _manifest()
    olds, news = synth.generate(m, seed=3, rho=0.05)
    news[1][:] = olds[1]            # one tensor unchanged -> no record
    pk = oracle.sync_pack(olds, news, codec=codec, limit=limit, crc=crc)
    W = [o.copy() for o in olds]
    for b in range(pk.n_buckets):
        bk = pk.bucket(b)
        hdr = np.frombuffer(bk[:24], np.uint32)
        assert hdr[0] == 0x424C5253 and (hdr[1] & 0xFFFF) == 1 and hdr[2] == b
        assert int(np.frombuffer(bk[24:32], np.uint64)[0]) == len(bk)
        assert len(bk) <= limit or hdr[3] == 1          # oversized record sits alone
        assert pk.offsets[b] % 256 == 0
        assert oracle.bucket_apply(bk, W) == oracle.OK
    for w, n in zip(W, news):
        assert (w == n).all()                         # bit-exact reconstruction
    assert pk.stats["n_records"] == sum(int((o != n).any()) for o, n in zip(olds, news))


def test_bucket_errors():
    m = _manifest()
    olds, news = synth.generate(m, seed=4, rho=0.05)
    pk = oracle.sync_pack(olds, news, crc=True)
    bk = pk.bucket(0)
    W = [o.copy() for o in olds]
    flip = bytearray(bk)
    flip[len(bk) // 2] ^= 1
    assert oracle.bucket_apply(bytes(flip), W) == oracle.ERR_CRC
    bad = bytearray(bk)
    bad[0] ^= 1
    assert oracle.bucket_apply(bytes(bad), W) == oracle.ERR_BAD_MAGIC
    ver = bytearray(bk)
    ver[4] = 2
    assert oracle.bucket_apply(bytes(ver), W) == oracle.ERR_VERSION
    assert oracle.bucket_apply(bk[:len(bk) - 16], W) == oracle.ERR_TRUNCATED


def test_bucket_decode_matches_extract():
    m = _manifest()
    olds, news = synth.generate(m, seed=5, rho=0.2)
    pk = oracle.sync_pack(olds, news, limit=1 << 30)
    st, recs = oracle.bucket_decode(pk.bucket(0), cap=100_000)
    assert st == oracle.OK
    for tid, I, V in recs:
        I0, V0 = oracle.extract(olds[tid], news[tid])
        assert (I == I0).all() and (V == V0).all()


def test_raw_payload_is_exact_eq1_identity():
    """RAW codec: payload = Σ pad16(16 + 6 nnz_t) + Σ_b (32 + pad16(8 n_b)) — Eq. (1) with b_i=4, b_v=2."""
    m = synth.Manifest("x", [synth.Tensor(f"t{k}", (1000 + 8 * k,)) for k in range(20)])
    olds, news = synth.generate(m, seed=1, rho=0.03)
    pk = oracle.sync_pack(olds, news, codec=oracle.CODEC_RAW, limit=2048)
    nnz = [int(np.count_nonzero(o != n)) for o, n in zip(olds, news)]
    rec = [((16 + 6 * k + 15) // 16) * 16 for k in nnz if k]
    nb, of = oracle.bucketize(rec, 2048)
    per_b = [int((of == b).sum()) for b in range(nb)]
    expect = sum(rec) + sum(32 + ((8 * k + 15) // 16) * 16 for k in per_b)
    assert pk.stats["payload_bytes"] == expect and pk.n_buckets == nb
    assert pk.stats["nnz"] == sum(nnz)


def test_payload_model_eq2_eq4():
    """At sparsity 1-1/X the payload is ≈ S/X (north_star); Eq. (2) X_raw = 1/(3 rho); Eq. (4) with measured alpha."""
    t = synth.Tensor("w", (1 << 20,))
    m = synth.Manifest("one", [t])
    olds, news = synth.generate(m, seed=0, rho=0.01)
    S = 2 * t.numel
    raw = oracle.sync_pack(olds, news, codec=oracle.CODEC_RAW, limit=1 << 30)
    cmp = oracle.sync_pack(olds, news, codec=oracle.CODEC_COMPRESSED, limit=1 << 30)
    rho = raw.stats["nnz"] / t.numel
    assert abs(S / raw.stats["payload_bytes"] - oracle.eq2_ratio(rho)) / oracle.eq2_ratio(rho) < 0.01
    alpha = cmp.stats["value_bytes"] / (2 * cmp.stats["nnz"])
    x4 = oracle.eq4_ratio(rho, 2, 2, alpha)
    assert abs(S / cmp.stats["payload_bytes"] - x4) / x4 < 0.01
    assert 0.60 <= alpha <= 0.70


def test_paper_anchors():
    # worked example: X_c(0.0062) = 2 / (0.0062 (2 + 0.6*2)) ≈ 100.8
    assert oracle.eq4_ratio(0.0062, 2, 2, 0.60) == pytest.approx(100.806, abs=1e-3)
    # 3.2 B per changed element
    assert oracle.eq3_compressed_bytes(1.0, 1.0, 2, 2, 0.60) == pytest.approx(3.2)
    # Eq. (2): X = 1/(3 rho) with b_i=4, b_v=2
    assert oracle.eq2_ratio(0.01) == pytest.approx(100 / 3)
    # 671B full = 1342 GB; sparse at rho≈0.77% ≈ 31.0 GB (raw int32 path)
    N = 671e9
    assert 2 * N / 1e9 == pytest.approx(1342)
    assert oracle.eq1_sparse_bytes(0.0077, N) / 1e9 == pytest.approx(31.0, abs=0.05)
