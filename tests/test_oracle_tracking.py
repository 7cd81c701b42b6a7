"""Pins of the oracle's f1 cast-fused tracking (Alg. 1) against things other than itself.

* round_BF16 (Alg. 1 l.5): PyTorch's own fp32 -> bf16 conversion (an independent implementation)
  on random and special bit patterns, plus hand-worked ties-to-even cases;
* the cumulative set (Alg. 1 l.6-7): brute force over several steps from the definition of a set
  union, the superset property the paper states (an element changed and changed back stays in the
  set), precision awareness (a master update that does not move the bf16 value never enters), and
  the round trip: applying (I, V = W[I]) to the last-synced copy reproduces W bit-exactly.
"""
import numpy as np
import pytest
import torch

import oracle


def torch_bf16_bits(f32: np.ndarray) -> np.ndarray:
    return torch.from_numpy(f32.astype(np.float32)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def test_bf16_rne_hand_cases():
    cases = [
        (1.0, 0x3F80),
        (-2.0, 0xC000),
        (1.0 + 2.0 ** -8, 0x3F80),          # exact tie between 0x3F80 and 0x3F81 -> even (0x3F80)
        (1.0 + 3 * 2.0 ** -8, 0x3F82),      # tie between 0x3F81 and 0x3F82 -> even (0x3F82)
        (1.0 + 2.0 ** -8 + 2.0 ** -20, 0x3F81),   # just above the tie -> up
        (float(np.finfo(np.float32).max), 0x7F80),  # overflow -> +Inf
        (float("inf"), 0x7F80),
        (float("-inf"), 0xFF80),
        (0.0, 0x0000),
        (-0.0, 0x8000),
    ]
    for v, want in cases:
        got = oracle.bf16_rne(np.array([v], np.float32))[0]
        assert got == want, (v, hex(got), hex(want))
    nan = np.array([0x7FC00000, 0x7F800001, 0xFFFFFFFF], np.uint32).view(np.float32)
    assert (oracle.bf16_rne(nan) == 0x7FC0).all()   # DESIGN C18


def test_bf16_rne_matches_torch():
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2 ** 32, 400_000, dtype=np.uint64).astype(np.uint32)
    f = bits.view(np.float32)
    ok = ~np.isnan(f)   # torch canonicalises NaN too; compared separately above
    assert (oracle.bf16_rne(f[ok]) == torch_bf16_bits(f[ok])).all()
    w = (rng.standard_normal(200_000) * 0.02).astype(np.float32)
    assert (oracle.bf16_rne(w) == torch_bf16_bits(w)).all()
    # every bf16 value itself (exact, no rounding) and the ties around each of them
    b = np.arange(0, 1 << 16, dtype=np.uint32)
    exact = (b << 16).view(np.float32)
    keep = ~np.isnan(exact)
    assert (oracle.bf16_rne(exact[keep]) == b[keep]).all()
    tie = ((b << 16) | 0x8000).view(np.float32)
    keep = ~np.isnan(tie)
    assert (oracle.bf16_rne(tie[keep]) == torch_bf16_bits(tie[keep])).all()


def _steps(n=5000, T=6, seed=1, frac=0.02):
    """A master trajectory: T optimizer steps touching a random frac of the elements each."""
    rng = np.random.default_rng(seed)
    m0 = (rng.standard_normal(n) * 0.02).astype(np.float32)
    ms = [m0]
    for _ in range(T):
        m = ms[-1].copy()
        idx = rng.choice(n, int(frac * n), replace=False)
        m[idx] += (rng.standard_normal(idx.size) * 1e-3).astype(np.float32)
        ms.append(m)
    return ms


def test_cumulative_set_is_the_union_and_round_trips():
    ms = _steps()
    n = ms[0].size
    W = oracle.bf16_rne(ms[0])
    synced = W.copy()            # what the Rollout holds
    tracked = np.zeros(n, np.uint8)
    union = set()
    for m in ms[1:]:
        prev = W.copy()
        c = oracle.cast_track(m, W, tracked)
        step = {i for i in range(n) if W[i] != prev[i]}   # Alg. 1 l.6 by brute force
        assert c == len(step)
        union |= step                                     # Alg. 1 l.7
    I, V = oracle.extract_tracked(W, tracked)
    assert list(I) == sorted(union)
    assert (V == W[I]).all()
    assert not tracked.any()                              # cleared: I_0 = {} for the next interval
    exact = set(oracle.extract(synced, W)[0].tolist())
    assert exact <= union                                 # superset of the true delta
    assert oracle.apply(synced, I, V) == oracle.OK
    assert (synced == W).all()                            # bit-exact replica


def test_changed_then_reverted_stays_in_the_set():
    m0 = np.array([1.0, 2.0, 3.0], np.float32)
    W = oracle.bf16_rne(m0)
    tracked = np.zeros(3, np.uint8)
    m1 = m0.copy(); m1[1] = 2.5
    oracle.cast_track(m1, W, tracked)
    oracle.cast_track(m0, W, tracked)      # back to the synced value
    I, V = oracle.extract_tracked(W, tracked)
    assert list(I) == [1] and V[0] == 0x4000   # redundant but harmless: V is the current value (2.0)


def test_sub_threshold_updates_never_enter():
    # a master change below half a bf16 ULP is absorbed by the cast (precision filter)
    m0 = np.array([1.0, 0.5, -3.0, 2.0 ** -10], np.float32)   # exact bf16 values
    W = oracle.bf16_rne(m0)
    tracked = np.zeros(4, np.uint8)
    ulp = np.array([2.0 ** -7, 2.0 ** -8, 2.0 ** -6, 2.0 ** -17], np.float32)
    m1 = (m0 + 0.49 * ulp * np.sign(m0)).astype(np.float32)
    assert oracle.cast_track(m1, W, tracked) == 0
    m2 = (m0 + 0.51 * ulp * np.sign(m0)).astype(np.float32)
    assert oracle.cast_track(m2, W, tracked) == 4
    assert tracked.all()


@pytest.mark.parametrize("n", [0, 1, 31, 32, 33, 1000])
def test_tracking_sizes(n):
    ms = _steps(n=max(n, 1), T=2, seed=n)
    m0 = ms[0][:n]
    W = oracle.bf16_rne(m0)
    tracked = np.zeros(n, np.uint8)
    oracle.cast_track(ms[1][:n], W, tracked)
    I, V = oracle.extract_tracked(W, tracked)
    assert I.size == int((oracle.bf16_rne(ms[1][:n]) != oracle.bf16_rne(m0)).sum())
