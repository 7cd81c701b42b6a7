"""Pins for oracle extract/apply (rows a1, a8, a9).

extract follows Alg. 1 l.6 / Alg. 2 l.5 with bitwise '≠'
(DESIGN C1); apply follows Alg. 3 l.6. Pins: SPEC examples, hand bf16
edge cases, invariants (count == popcount of changed patterns; count == mask
popcount for generator inputs), round trip, idempotence,
superset harmlessness.
"""
import numpy as np
import pytest

import oracle
import synth


def bf(*vals):
    """float -> bf16 bit patterns (exact for the small values used here)."""
    f = np.array(vals, np.float32).view(np.uint32)
    assert ((f & 0xFFFF) == 0).all()
    return (f >> 16).astype(np.uint16)


def test_spec_example_one_change():
    # S:131 prev=[1.0,2.0,3.0], curr=[1.0,2.5,3.0] -> [1]
    I, V = oracle.extract(bf(1.0, 2.0, 3.0), bf(1.0, 2.5, 3.0))
    assert I.tolist() == [1]
    assert V.tolist() == [0x4020]          # bf16(2.5)


def test_identical_and_empty():
    x = bf(1.0, -2.0, 0.5)
    I, V = oracle.extract(x, x.copy())
    assert I.size == 0 and V.size == 0
    I, V = oracle.extract(np.zeros(0, np.uint16), np.zeros(0, np.uint16))
    assert I.size == 0


def test_signed_zero_and_nan_bits():
    old = np.array([0x0000, 0x7FC0, 0x7FC0, 0xFF80, 0x3F80], np.uint16)
    new = np.array([0x8000, 0x7FC0, 0x7FC1, 0xFF80, 0x3F81], np.uint16)
    I, V = oracle.extract(old, new)
    # +0 -> -0 changed; same NaN bits unchanged; NaN payload change changed; -inf same; ulp change
    assert I.tolist() == [0, 2, 4]
    assert V.tolist() == [0x8000, 0x7FC1, 0x3F81]


def test_first_and_last_changed():
    old = np.arange(1000, dtype=np.uint16)
    new = old.copy()
    new[0] ^= 1
    new[-1] ^= 0x8000
    I, V = oracle.extract(old, new)
    assert I.tolist() == [0, 999]
    assert V.tolist() == [new[0], new[-1]]


@pytest.mark.parametrize("n,seed", [(1, 0), (37, 1), (4096, 2), (100_003, 3)])
def test_count_invariant_random_bits(n, seed):
    rng = np.random.default_rng(seed)
    old = rng.integers(0, 65536, n, dtype=np.uint16)
    new = old.copy()
    flip = rng.random(n) < 0.3
    new[flip] ^= rng.integers(1, 65536, flip.sum(), dtype=np.uint16)
    I, V = oracle.extract(old, new)
    # invariant (north_star): count == number of elements whose xor is non-zero
    assert I.size == int(np.count_nonzero(old ^ new))
    assert (np.diff(I.astype(np.int64)) > 0).all()
    assert (V == new[I]).all() and (old[I] != new[I]).all()


@pytest.mark.parametrize("rho", [0.1, 0.01, 0.001])
def test_generator_mask_popcount(rho):
    t = synth.Tensor("w", (512, 256))
    old = synth.gen_old(t, 3, 0)
    new = synth.gen_new(old, t, 3, 0, rho)
    mask = synth.gen_mask(t, 3, 0, rho)
    I, _ = oracle.extract(old, new)
    # the perturbation always flips >= 1 bit, so count == mask popcount exactly
    assert I.size == int(mask.sum())
    assert (np.flatnonzero(mask) == I).all()


def test_spec_apply_example_and_round_trip():
    W = bf(1.0, 2.0, 3.0)
    assert oracle.apply(W, [1], bf(7.0)) == oracle.OK        # S:330 [a,b,c]+{1:v} -> [a,v,c]
    assert W.tolist() == bf(1.0, 7.0, 3.0).tolist()

    t = synth.Tensor("w", (300, 333))
    old = synth.gen_old(t, 0, 5)
    new = synth.gen_new(old, t, 0, 5, 0.02)
    I, V = oracle.extract(old, new)
    W = old.copy()
    assert oracle.apply(W, I, V) == oracle.OK
    assert (W == new).all()                 # G1 bit-exact
    assert oracle.apply(W, I, V) == oracle.OK
    assert (W == new).all()                 # idempotent


def test_superset_is_harmless():
    # redundant indices are harmless because absolute values are sent
    rng = np.random.default_rng(9)
    old = rng.integers(0, 65536, 5000, dtype=np.uint16)
    new = old.copy()
    ch = rng.choice(5000, 50, replace=False)
    new[ch] ^= 3
    I, _ = oracle.extract(old, new)
    extra = np.setdiff1d(rng.choice(5000, 500, replace=False), I)
    Isup = np.union1d(I, extra).astype(np.uint32)
    W = old.copy()
    assert oracle.apply(W, Isup, new[Isup]) == oracle.OK
    assert (W == new).all()


def test_apply_index_out_of_range():
    W = np.zeros(4, np.uint16)
    st = oracle.apply(W, [1, 9, 3], [5, 6, 7])
    assert st == oracle.ERR_INDEX_RANGE
    assert W.tolist() == [0, 5, 0, 7]       # valid indices written, no OOB write
