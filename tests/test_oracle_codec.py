"""Pins for the oracle codec (rows a2, a3, a4; inverse a7).

Index coding: PAPER §3.3 "Index delta encoding" — SPEC examples
 and the exact 32767/32768 threshold.
Value coding: PAPER §3.3 "Value entropy coding" fixes no coder; the
reading is DESIGN C6. Pins: hand-derived golden vectors (tests/golden/),
hand-worked normalisation cases, lossless round trip, entropy bounds, the
paper's α range on N(0, 0.02) bf16 values, never-expand.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "rans_golden.json")


# ----------------------------------------------------------------------------- indices
def test_spec_index_examples():
    assert oracle.index_mode([2, 5, 9]) == oracle.DELTA16
    assert np.frombuffer(oracle.encode_indices([2, 5, 9], oracle.DELTA16), np.uint16).tolist() == [2, 3, 4]
    assert oracle.index_mode([3, 7, 40010]) == oracle.ABS32                     # S:208 gap 40003
    assert oracle.index_mode([]) == oracle.DELTA16
    assert oracle.encode_indices([], oracle.DELTA16) == b""
    assert oracle.decode_indices(np.array([2, 3, 4], np.uint16).tobytes(), 3, oracle.DELTA16).tolist() == [2, 5, 9]
    assert oracle.decode_indices(np.array([0], np.uint32).tobytes(), 1, oracle.ABS32).tolist() == [0]


@pytest.mark.parametrize("I,mode", [
    ([32767], oracle.DELTA16), ([32768], oracle.ABS32),                 # first delta from the prepended 0
    ([5, 5 + 32767], oracle.DELTA16), ([5, 5 + 32768], oracle.ABS32),
    ([0, 1, 2, 32769], oracle.DELTA16), ([0, 1, 2, 32771], oracle.ABS32),
])
def test_delta16_threshold(I, mode):
    assert oracle.index_mode(I) == mode


def test_index_round_trip_random():
    rng = np.random.default_rng(0)
    for trial in range(50):
        n = int(rng.integers(1, 3000))
        I = np.unique(rng.integers(0, 1 << 31, n)).astype(np.uint32)
        if trial % 2:
            I = np.cumsum(rng.integers(1, 32768, n)).astype(np.uint32)
        mode = oracle.index_mode(I)
        b = oracle.encode_indices(I, mode)
        assert len(b) == (2 if mode == oracle.DELTA16 else 4) * I.size
        assert (oracle.decode_indices(b, I.size, mode) == I).all()


# ----------------------------------------------------------------------------- frequencies
def test_normalize_hand_cases():
    c = np.zeros(256, np.uint32)
    c[[0x3C, 0xBC, 0xBB, 0x3B]] = [4, 2, 1, 1]
    f = oracle.normalize_freqs(c)
    assert {s: int(f[s]) for s in np.flatnonzero(f)} == {0x3B: 512, 0x3C: 2048, 0xBB: 512, 0xBC: 1024}
    # remainder goes to the largest count; ties -> lowest symbol
    c = np.zeros(256, np.uint32)
    c[[0x10, 0x20, 0x30]] = 1
    f = oracle.normalize_freqs(c)
    assert (f[0x10], f[0x20], f[0x30]) == (1366, 1365, 1365)
    # excess removed from the largest frequency: 255 singletons at f=1, the big one gets 4096-255
    c = np.ones(256, np.uint32)
    c[7] = 16384 - 255
    f = oracle.normalize_freqs(c)
    assert f[7] == 3841 and (np.delete(f, 7) == 1).all()


def test_normalize_properties():
    rng = np.random.default_rng(1)
    for _ in range(200):
        k = int(rng.integers(1, 257))
        c = np.zeros(256, np.uint32)
        syms = rng.choice(256, k, replace=False)
        c[syms] = rng.integers(1, 2000, k)
        f = oracle.normalize_freqs(c)
        assert f.sum() == 4096
        assert ((f > 0) == (c > 0)).all()


# ----------------------------------------------------------------------------- rANS goldens
def _hi_of(v):
    if "hi" in v:
        return np.array(v["hi"], np.uint8)
    if "hi_fill" in v:
        return np.full(v["n"], v["hi_fill"], np.uint8)
    n = v["n"]
    if v["name"].startswith("G3"):
        return np.array([60 if (p // 32) % 2 == 0 else 61 for p in range(n)], np.uint8)
    hi = np.full(n, 60, np.uint8)
    hi[[0, 32, 64]] = 61
    return hi


@pytest.mark.parametrize("v", json.load(open(GOLDEN))["vectors"], ids=lambda v: v["name"])
def test_rans_golden(v):
    hi = _hi_of(v)
    blk = oracle.rans_encode(hi)
    assert len(blk) == v["hi_bytes"]
    states = np.frombuffer(blk[:128], np.uint32)
    if "states_lane0_7" in v:
        assert states[:8].tolist() == v["states_lane0_7"]
        assert (states[8:] == v["states_rest"]).all()
    if "states_all" in v:
        assert (states == v["states_all"]).all()
    if "state_lane0" in v:
        assert states[0] == v["state_lane0"] and (states[1:] == v["states_lanes1_31"]).all()
    nwords = int(np.frombuffer(blk[128:132], np.uint32)[0])
    nsym = int(np.frombuffer(blk[132:134], np.uint16)[0])
    assert nwords == v["nwords"]
    ent = np.frombuffer(blk[136:136 + 4 * nsym], np.uint32)
    assert {str(int(e & 0xFFFF)): int(e >> 16) for e in ent} == v["freq"]
    if "words" in v:
        assert np.frombuffer(blk[136 + 4 * nsym:], np.uint16).tolist() == v["words"]
    st, dec = oracle.rans_decode(blk, hi.size)
    assert st == oracle.OK and (dec == hi).all()
    # in a record, the never-expand rule decides the stored chunk mode
    V = (hi.astype(np.uint16) << 8) | 0x11
    rec = oracle.encode_record(0, np.arange(hi.size, dtype=np.uint32), V)
    nnz = hi.size
    dir_off = 16 + ((2 * nnz + 3) // 4) * 4 + ((nnz + 3) // 4) * 4
    mode = int(np.frombuffer(rec[dir_off + 8:dir_off + 12], np.uint32)[0])
    assert mode == v["chunk_mode_in_record"]


# ----------------------------------------------------------------------------- rANS properties
def _entropy_bits(hi):
    p = np.bincount(hi, minlength=256) / hi.size
    p = p[p > 0]
    return float(-(p * np.log2(p)).sum())


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 100, 1000, 16383, 16384])
def test_rans_round_trip_sizes(n):
    rng = np.random.default_rng(n)
    for dist in range(3):
        if dist == 0:
            hi = rng.integers(0, 256, n).astype(np.uint8)
        elif dist == 1:
            hi = (synth.bf16_table()[rng.integers(0, 65536, n)] >> 8).astype(np.uint8)
        else:
            hi = np.full(n, 0x3F, np.uint8)
        blk = oracle.rans_encode(hi)
        st, dec = oracle.rans_decode(blk, n)
        assert st == oracle.OK and (dec == hi).all()


def test_rans_entropy_bound():
    """Size of a static order-0 rANS stream is within a hair of n*H (ANS theory; 12-bit model)."""
    rng = np.random.default_rng(7)
    hi = (synth.bf16_table()[rng.integers(0, 65536, 16384)] >> 8).astype(np.uint8)
    blk = oracle.rans_encode(hi)
    nsym = int(np.frombuffer(blk[132:134], np.uint16)[0])
    payload = len(blk) - 136 - 4 * nsym + 128           # words + lane states
    ideal = hi.size * _entropy_bits(hi) / 8
    assert ideal - 8 <= payload <= 1.01 * ideal + 136


def test_rans_detects_corruption():
    rng = np.random.default_rng(3)
    hi = (synth.bf16_table()[rng.integers(0, 65536, 4000)] >> 8).astype(np.uint8)
    blk = bytearray(oracle.rans_encode(hi))
    nsym = int(np.frombuffer(bytes(blk[132:134]), np.uint16)[0])
    bad = 0
    for k in range(20):
        b2 = bytearray(blk)
        b2[136 + 4 * nsym + 2 * (k * 37 % 200)] ^= 0x5A
        st, dec = oracle.rans_decode(bytes(b2), hi.size)
        bad += st == oracle.ERR_CORRUPT
    assert bad >= 18                                     # end-state check catches word damage
    b2 = bytearray(blk)
    b2[0] ^= 0xFF                                        # lane-state damage
    assert oracle.rans_decode(bytes(b2), hi.size)[0] == oracle.ERR_CORRUPT


# ----------------------------------------------------------------------------- records / alpha
def test_alpha_in_paper_range():
    """entropy coding reduces the value stream to alpha in [0.60, 0.70] on weight-like values."""
    t = synth.Tensor("w", (4096, 2048))
    old = synth.gen_old(t, 1, 0)
    new = synth.gen_new(old, t, 1, 0, 0.01)
    I, V = oracle.extract(old, new)
    rec = oracle.encode_record(1, I, V)
    nnz = I.size
    assert oracle.index_mode(I) == oracle.DELTA16
    value_bytes = len(rec) - 16 - ((2 * nnz + 3) // 4) * 4
    alpha = value_bytes / (2 * nnz)
    assert 0.60 <= alpha <= 0.70


def test_record_never_expand_uniform_values():
    rng = np.random.default_rng(4)
    nnz = 20000
    I = np.sort(rng.choice(1 << 20, nnz, replace=False)).astype(np.uint32)
    V = rng.integers(0, 65536, nnz).astype(np.uint16)
    rec = oracle.encode_record(0, I, V)
    st, tid, I2, V2 = oracle.decode_record(rec)
    assert st == oracle.OK and (I2 == I).all() and (V2 == V).all()
    dir_off = 16 + ((4 * nnz + 3) // 4) * 4 + ((nnz + 3) // 4) * 4 if oracle.index_mode(I) else \
        16 + ((2 * nnz + 3) // 4) * 4 + ((nnz + 3) // 4) * 4
    d = np.frombuffer(rec[dir_off:dir_off + 32], np.uint32).reshape(2, 4)
    assert (d[:, 2] == 0).all()                            # both chunks RAW: uniform bytes don't compress
    assert d[0, 1] == 16384 and d[1, 1] == nnz - 16384
    assert len(rec) <= 16 + 4 * nnz + nnz + 32 + nnz + 16  # never larger than raw hi + overhead


@pytest.mark.parametrize("nnz", [1, 7, 16383, 16384, 16385, 40000])
def test_record_round_trip_and_chunk_bases(nnz):
    rng = np.random.default_rng(nnz)
    gaps = rng.integers(1, 200, nnz)
    I = np.cumsum(gaps).astype(np.uint32)
    V = synth.bf16_table()[rng.integers(0, 65536, nnz)]
    rec = oracle.encode_record(11, I, V)
    assert len(rec) % 16 == 0
    hdr = np.frombuffer(rec[:12], np.uint32)
    assert hdr.tolist() == [11, nnz, len(rec)] and rec[12] == oracle.DELTA16 and rec[13] == 1 and rec[14] == 1
    st, tid, I2, V2 = oracle.decode_record(rec)
    assert st == oracle.OK and tid == 11 and (I2 == I).all() and (V2 == V).all()
    nch = (nnz + 16383) // 16384
    dir_off = 16 + ((2 * nnz + 3) // 4) * 4 + ((nnz + 3) // 4) * 4
    d = np.frombuffer(rec[dir_off:dir_off + 16 * nch], np.uint32).reshape(nch, 4)
    expect_base = [0] + [int(I[16384 * k - 1]) for k in range(1, nch)]
    assert d[:, 3].tolist() == expect_base                 # chunk k decodes alone from base_idx


def test_raw_record_is_eq1():
    """Codec RAW reproduces the paper's raw (I,V) path: 4 B index + 2 B value per change (Eq. 1)."""
    for nnz in [1, 2, 3, 8, 1000]:
        I = np.arange(nnz, dtype=np.uint32) * 3
        V = np.arange(nnz, dtype=np.uint16)
        rec = oracle.encode_record(0, I, V, oracle.CODEC_RAW)
        assert len(rec) == ((16 + 6 * nnz + 15) // 16) * 16
        st, tid, I2, V2 = oracle.decode_record(rec)
        assert st == oracle.OK and (I2 == I).all() and (V2 == V).all()
