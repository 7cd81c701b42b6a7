"""Pins of the oracle's f4 escape-coded DELTA16 (P:360 keeps int32 whenever a
gap does not fit in int16, which for row-clustered masks is every record).

* hand-worked streams at the 32767 / 32768 threshold and at the largest gap 2^31 - 1;
* round trip on random gap mixtures; stream length = 2 (nnz + escapes);
* the mode rule: no escape -> DELTA16, escapes < nnz -> DELTA16E, else ABS32;
* each chunk decodes on its own from the word-offset table (after the header, with the total word count
  last) + its directory base (what a chunk-parallel decoder relies on);
* on the R (clustered-row) mask every ABS32 record becomes DELTA16E, the payload shrinks, the replica is
  bit-exact; without the flag the bytes are the v1 format unchanged.
"""
import numpy as np

import oracle
import synth


def words(b: bytes):
    return list(np.frombuffer(b, np.uint16))


def test_hand_streams():
    assert words(oracle.encode_indices_escape([5, 5 + 32767])) == [5, 32767]
    assert words(oracle.encode_indices_escape([0, 32768])) == [0, 0x8000, 0x8000]
    big = (1 << 31) - 1
    assert words(oracle.encode_indices_escape([big])) == [0xFFFF, 0xFFFF]
    assert words(oracle.encode_indices_escape([70000, 70001])) == [0x8001, 70000 - 65536, 1]
    I, w = oracle.decode_indices_escape(bytes(np.array([0x8001, 4464, 1], np.uint16)), 2)
    assert list(I) == [70000, 70001] and w == 3
    assert oracle.decode_indices_escape(bytes(np.array([0x8001], np.uint16)), 1) == (None, None)


def test_round_trip_and_length():
    rng = np.random.default_rng(0)
    for _ in range(50):
        n = int(rng.integers(1, 3000))
        gaps = np.where(rng.random(n) < 0.05, rng.integers(32768, 1 << 24, n), rng.integers(1, 32768, n))
        I = np.cumsum(gaps).astype(np.uint32)
        s = oracle.encode_indices_escape(I)
        esc = int(lib_count(I))
        assert len(s) == 2 * (n + esc)
        J, w = oracle.decode_indices_escape(s, n)
        assert (J == I).all() and w == n + esc


def lib_count(I):
    I = np.ascontiguousarray(I, np.uint32)
    return oracle.lib().or_count_escapes(I.ctypes.data, I.size)


def test_mode_rule():
    def mode(I):
        rec = oracle.encode_record(0, np.array(I, np.uint32), np.ones(len(I), np.uint16), escape=True)
        return rec[12]
    assert mode([1, 2, 32769]) == oracle.DELTA16               # gaps 1, 1, 32767
    assert mode([1, 2, 40000, 40001]) == oracle.DELTA16E       # one escape of 4
    assert mode([40000, 80000]) == oracle.ABS32                # every gap escapes
    assert oracle.encode_record(0, np.array([1, 40000], np.uint32), np.ones(2, np.uint16))[12] == oracle.ABS32


def test_chunks_decode_independently():
    rng = np.random.default_rng(1)
    n = 3 * oracle.CHUNK + 77
    gaps = np.where(rng.random(n) < 0.02, rng.integers(40000, 90000, n), rng.integers(1, 50, n))
    I = np.cumsum(gaps).astype(np.uint32)
    V = rng.integers(0, 1 << 16, n, dtype=np.uint64).astype(np.uint16)
    rec = np.frombuffer(oracle.encode_record(7, I, V, escape=True), np.uint8)
    assert rec[12] == oracle.DELTA16E
    nch = (n + oracle.CHUNK - 1) // oracle.CHUNK
    esc = int(lib_count(I))
    ib = 2 * (n + esc)
    table = rec[16:16 + 4 * (nch + 1)].view(np.uint32)
    assert table[nch] == n + esc
    s0 = 16 + 4 * (nch + 1)
    lo_off = s0 + ib + (-ib) % 4
    dir_off = lo_off + n + (-n) % 4
    stream = rec[s0:s0 + ib].tobytes()
    for k in range(nch):
        p0 = k * oracle.CHUNK
        nk = min(oracle.CHUNK, n - p0)
        base = int(rec[dir_off + 16 * k + 12:dir_off + 16 * k + 16].view(np.uint32)[0])
        J, _ = oracle.decode_indices_escape(stream[2 * int(table[k]):], nk)
        assert (J + np.uint32(base) == I[p0:p0 + nk]).all()
    st, recs = oracle.bucket_decode(_bucket_of(rec), cap=n)
    assert st == oracle.OK and (recs[0][1] == I).all() and (recs[0][2] == V).all()


def _bucket_of(rec: np.ndarray) -> bytes:
    bk = bytearray(32 + 16) + rec.tobytes()
    bk[0:4] = (0x424C5253).to_bytes(4, "little")
    bk[4:6] = (1).to_bytes(2, "little")
    bk[12:16] = (1).to_bytes(4, "little")
    n = int(rec[4:8].view(np.uint32)[0])
    bk[16:20] = ((n + oracle.CHUNK - 1) // oracle.CHUNK).to_bytes(4, "little")
    bk[24:32] = len(bk).to_bytes(8, "little")
    bk[32:36] = (48).to_bytes(4, "little")
    return bytes(bk)


def test_row_clustered_mask():
    m = synth.Manifest("m", [synth.Tensor(f"w{k}", (512, 2048)) for k in range(4)] +
                       [synth.Tensor("n", (2048,), synth.KIND_NORM)])
    olds, news = synth.generate(m, seed=2, rho=0.01, mask=synth.MASK_R)
    plain = oracle.sync_pack(olds, news)
    esc = oracle.sync_pack(olds, news, escape=True)
    assert plain.stats["abs32"] >= 3 and esc.stats["delta16e"] == plain.stats["abs32"]
    assert esc.stats["payload_bytes"] < 0.8 * plain.stats["payload_bytes"]
    W = [o.copy() for o in olds]
    for b in range(esc.n_buckets):
        assert oracle.bucket_apply(esc.bucket(b), W) == oracle.OK
    assert all((w == n).all() for w, n in zip(W, news))
    off = oracle.sync_pack(olds, news, escape=False)
    assert [off.bucket(b) for b in range(off.n_buckets)] == [plain.bucket(b) for b in range(plain.n_buckets)]
