"""Pins of the oracle's f3 per-parameter routing (DESIGN §3.5 / C19).

* the rule: a record goes FULL exactly when the FULL record (16 B + 2 B per element) is smaller than the
  sparse record the same changes would produce — checked against the sizes of independently encoded
  records, at densities around the break-even point (raw codec: 3 nnz ~ numel, SPEC's 1/3);
* FULL records carry every element in order (nnz field = numel), so the decoder's (I, V) is (0..n-1, W_new);
* round trip: applying the routed buckets to the old weights reproduces the new weights bit-exactly;
* the LoRA example of P:389 (a small adapter updated on every element) goes FULL while a >= 99%-sparse
  base-model tensor stays sparse;
* routing off reproduces the unrouted format byte for byte.
"""
import numpy as np
import pytest

import oracle
import synth


def _tensors(n, rho, seed):
    rng = np.random.default_rng(seed)
    old = rng.integers(0, 1 << 16, n, dtype=np.uint64).astype(np.uint16)
    new = old.copy()
    idx = rng.choice(n, int(rho * n), replace=False)
    new[idx] ^= 1 + (rng.integers(0, 3, idx.size)).astype(np.uint16)
    return old, new


def _records(pack):
    out = {}
    for b in range(pack.n_buckets):
        a = np.frombuffer(pack.bucket(b), np.uint8)
        nrec = int(a[12:16].view(np.uint32)[0])
        dirv = a[32:32 + 8 * nrec].view(np.uint32).reshape(-1, 2)
        for q in range(nrec):
            ro = int(dirv[q, 0])
            tid, nnz, rb = (int(v) for v in a[ro:ro + 12].view(np.uint32))
            out[tid] = (a[ro:ro + rb].tobytes(), int(a[ro + 12]), nnz)
    return out


@pytest.mark.parametrize("codec", [oracle.CODEC_RAW, oracle.CODEC_COMPRESSED])
@pytest.mark.parametrize("rho", [0.01, 0.2, 0.3, 0.34, 0.5, 0.9, 1.0])
def test_rule_is_smaller_record(codec, rho):
    n = 3000
    old, new = _tensors(n, rho, seed=int(rho * 100))
    I, V = oracle.extract(old, new)
    if I.size == 0:
        return
    sparse = oracle.encode_record(0, I, V, codec)
    full = oracle.encode_full_record(0, new, codec)
    assert len(full) == 16 + 2 * n + (-(16 + 2 * n)) % 16
    pk = oracle.sync_pack([old], [new], codec=codec, route=True)
    rec, mode, nnz = _records(pk)[0]
    if len(full) < len(sparse):
        assert mode == 2 and rec == full and nnz == n and pk.stats["full"] == 1
    else:
        assert rec == sparse and mode in (0, 1) and pk.stats["full"] == 0


def test_full_record_layout_and_decode():
    new = np.array([7, 0x8000, 0xFFFF, 1, 2], np.uint16)
    rec = oracle.encode_full_record(3, new)
    a = np.frombuffer(rec, np.uint8)
    assert list(a[:16].view(np.uint32)[:3]) == [3, 5, 32] and a[12] == 2 and a[13] == 1
    assert (a[16:26].view(np.uint16) == new).all() and not a[26:].any()
    old = np.zeros(5, np.uint16)
    pk = oracle.sync_pack([old], [new], route=True)
    W = [old.copy()]
    assert oracle.bucket_apply(pk.bucket(0), W) == oracle.OK
    assert (W[0] == new).all()
    st, recs = oracle.bucket_decode(pk.bucket(0), cap=16)
    assert st == oracle.OK and recs[0][0] == 0
    assert list(recs[0][1]) == [0, 1, 2, 3, 4] and (recs[0][2] == new).all()


def test_lora_goes_full_base_stays_sparse():
    m = synth.Manifest("m", [synth.Tensor("base", (256, 512)), synth.Tensor("lora_A", (8, 512)),
                             synth.Tensor("lora_B", (512, 8))])
    olds, news = synth.generate(m, seed=3, rho=0.01)
    for k in (1, 2):    # adapters: every element changes
        news[k] = olds[k] ^ np.uint16(1)
    pk = oracle.sync_pack(olds, news, route=True)
    recs = _records(pk)
    assert recs[0][1] in (0, 1) and recs[1][1] == 2 and recs[2][1] == 2
    W = [o.copy() for o in olds]
    for b in range(pk.n_buckets):
        assert oracle.bucket_apply(pk.bucket(b), W) == oracle.OK
    assert all((w == n).all() for w, n in zip(W, news))


def test_routing_off_is_the_plain_format():
    m = synth.Manifest("m", [synth.Tensor("a", (64, 64)), synth.Tensor("b", (1000,))])
    olds, news = synth.generate(m, seed=4, rho=0.6)
    a = oracle.sync_pack(olds, news, route=False)
    b = oracle.sync_pack(olds, news)
    assert a.n_buckets == b.n_buckets and all(a.bucket(i) == b.bucket(i) for i in range(a.n_buckets))
    c = oracle.sync_pack(olds, news, route=True)
    assert c.stats["full"] == 2 and c.stats["payload_bytes"] < a.stats["payload_bytes"]
