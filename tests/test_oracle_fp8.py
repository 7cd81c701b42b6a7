"""Pins of the oracle's FP8 (E4M3) synchronisation precision (f2 second half; P:190 measures FP8 update
density next to BF16 / FP16, C21).

8-bit elements: extraction compares bytes; a record has one value plane (the byte itself, rANS-coded per
chunk, never-expand), no lo plane; RAW records carry u8 values; FULL records one byte per element. Pins:
the definition on hand bytes (±0, NaN bit patterns), the record layout against the (already pinned) 16-bit
layout of the same indices, the value coder against the byte plane's empirical entropy, RAW / FULL sizes,
and the round trip on FP8-shaped synthetic data (U and R masks, routing, escapes, CRC).
"""
import numpy as np
import pytest

import oracle
import synth

FP8 = oracle.DTYPE_FP8


def test_extract8_definition():
    old = np.array([0x00, 0x80, 0x7F, 0x7F, 0x38, 0x12], np.uint8)
    new = np.array([0x80, 0x80, 0x7F, 0x7E, 0x38, 0x13], np.uint8)
    I, V = oracle.extract8(old, new)
    assert list(I) == [0, 3, 5] and list(V) == [0x80, 0x7E, 0x13]   # +0 -> -0 is a change; same NaN bits not


def _rec(I, V, dtype, codec=oracle.CODEC_COMPRESSED):
    return np.frombuffer(oracle.encode_record(5, np.array(I, np.uint32), np.array(V, np.uint16), codec=codec,
                                              dtype=dtype), np.uint8)


def test_record_layout_shares_the_index_coding():
    rng = np.random.default_rng(0)
    n = 20000
    I = np.sort(rng.choice(1 << 20, n, replace=False)).astype(np.uint32)
    V8 = rng.integers(0, 256, n).astype(np.uint16)
    r8 = _rec(I, V8, FP8)
    r16 = _rec(I, V8 << 8, oracle.DTYPE_BF16)       # same hi plane, zero lo plane
    ib = 2 * n if r8[12] == oracle.DELTA16 else 4 * n
    ib_p = ib + (-ib) % 4
    assert r8[12] == r16[12] and r8[13] == FP8 and (r8[16:16 + ib] == r16[16:16 + ib]).all()
    # FP8: no lo plane, so the directory follows the index stream; the value chunks are those of the 16-bit
    # record's hi plane (identical symbols) shifted by the missing lo plane
    lo = n + (-n) % 4
    nch = (n + 16383) // 16384
    d8 = r8[16 + ib_p:16 + ib_p + 16 * nch].view(np.uint32).reshape(nch, 4)
    d16 = r16[16 + ib_p + lo:16 + ib_p + lo + 16 * nch].view(np.uint32).reshape(nch, 4)
    assert (d8[:, 1:] == d16[:, 1:]).all() and (d16[:, 0] - d8[:, 0] == lo).all()
    for k in range(nch):
        o8, o16, hb = int(d8[k, 0]), int(d16[k, 0]), int(d8[k, 1])
        assert (r8[o8:o8 + hb] == r16[o16:o16 + hb]).all()


def test_raw_and_full_sizes():
    r = _rec([1, 9, 100], [3, 4, 5], FP8, codec=oracle.CODEC_RAW)
    assert r.size == 32 and list(r[16:28].view(np.uint32)) == [1, 9, 100] and list(r[28:31]) == [3, 4, 5]
    f = np.frombuffer(oracle.encode_full_record(2, np.arange(20, dtype=np.uint8), dtype=FP8), np.uint8)
    assert f.size == 48 and f[12] == 2 and f[13] == FP8 and (f[16:36] == np.arange(20)).all() and not f[36:].any()


def test_value_coder_vs_entropy():
    rng = np.random.default_rng(1)
    v = synth.fp8_table()[rng.integers(0, 65536, 200_000)].astype(np.uint16)
    I = np.arange(0, 2 * v.size, 2, dtype=np.uint32)
    rec = _rec(I, v, FP8)
    p = np.bincount(v, minlength=256) / v.size
    H = -(p[p > 0] * np.log2(p[p > 0])).sum()
    chunks = v.size // 16384 + 1
    value_bytes = rec.size - 16 - 2 * v.size
    lower = v.size * H / 8
    assert lower <= value_bytes <= lower * 1.01 + (16 + 136 + 1024) * chunks


@pytest.mark.parametrize("mask,route,escape,crc", [(synth.MASK_U, False, False, False),
                                                    (synth.MASK_R, False, True, True),
                                                    (synth.MASK_U, True, False, False)])
def test_round_trip(mask, route, escape, crc):
    m = synth.Manifest("m", [synth.Tensor("a", (300, 512)), synth.Tensor("n", (64,), synth.KIND_NORM),
                             synth.Tensor("b", (70_000,)), synth.Tensor("c", (64, 40000))])
    olds, news = synth.generate(m, seed=9, rho=0.03, mask=mask, dtype=synth.DTYPE_FP8)
    if route:
        news[0] = olds[0] ^ np.uint8(1)
    assert all(o.dtype == np.uint8 for o in olds)
    for codec in (oracle.CODEC_COMPRESSED, oracle.CODEC_RAW):
        pk = oracle.sync_pack(olds, news, codec=codec, limit=64 << 10, crc=crc, route=route, escape=escape,
                              dtype=FP8)
        W = [o.copy() for o in olds]
        for b in range(pk.n_buckets):
            assert oracle.bucket_apply(pk.bucket(b), W) == oracle.OK
        assert all((w == n).all() for w, n in zip(W, news))
        if route:
            assert pk.stats["full"] >= 1
