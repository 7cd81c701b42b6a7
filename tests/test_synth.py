"""The shared synthetic generator (no method arithmetic): pinned to SplitMix64 and to its recipe."""
import numpy as np

import synth


def test_splitmix64_reference_value():
    # SplitMix64 (Steele et al.) first output from state 0 is 0xE220A8397B1DCDAF
    assert synth.mix_int(0) == 0xE220A8397B1DCDAF
    z = np.array([0, 1, 2, 12345], np.uint64)
    assert [int(v) for v in synth.mix_np(z)] == [synth.mix_int(int(x)) for x in z]


def test_table_is_gaussian_bf16():
    t = synth.bf16_table()
    f = (t.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    assert np.all(np.diff(f) >= 0)                  # quantiles ascending
    assert abs(f.mean()) < 1e-4 and abs(f.std() - 0.02) < 5e-4


def test_manifest_totals_match_public_configs():
    # tensor counts and parameter totals
    assert (len(synth.qwen3_manifest("qwen3-4b").tensors), synth.qwen3_manifest("qwen3-4b").total) == (398, 4022468096)
    m = synth.qwen3_manifest("qwen3-30b-a3b")
    assert (len(m.tensors), m.total) == (18867, 30532122624)
    m = synth.qwen3_manifest("qwen3-235b-a22b")
    assert (len(m.tensors), m.total) == (36945, 235093634560)


def test_mask_density_and_perturbation():
    t = synth.Tensor("w", (1000, 1000))
    old = synth.gen_old(t, 0, 0)
    for rho in [0.1, 0.01, 0.001]:
        m = synth.gen_mask(t, 0, 1, rho)
        assert abs(m.mean() - rho) < 5 * np.sqrt(rho / t.numel) + 1e-6
        new = synth.gen_new(old, t, 0, 1, rho)
        d = old ^ new
        assert ((d != 0) == m).all() and d.max() <= 3      # low mantissa bits only, always >= 1 bit
    r = synth.gen_mask(t, 0, 1, 0.01, synth.MASK_R).reshape(1000, 1000)
    assert 0.05 < r.any(axis=1).mean() < 0.15               # ~10% rows active


def test_cpu_twin_matches_numpy_recipe():
    import synth.cpu
    m = synth.Manifest("g", [synth.Tensor("a", (300, 1000)), synth.Tensor("n", (64,), synth.KIND_NORM),
                             synth.Tensor("e", (96, 40), layer=3, expert=5), synth.Tensor("z", (0,))])
    for mask in [synth.MASK_U, synth.MASK_R, synth.MASK_E]:
        a = synth.generate(m, seed=7, rho=0.05, mask=mask, tid0=11)
        b = synth.cpu.generate(m, seed=7, rho=0.05, mask=mask, tid0=11)
        assert all((x == y).all() for x, y in zip(a[0] + a[1], b[0] + b[1]))


def test_shard_covers_manifest():
    m = synth.qwen3_manifest("qwen3-4b")
    parts = [synth.shard(m, r, 4) for r in range(4)]
    assert sum(len(p.tensors) for p in parts) == len(m.tensors)
    assert [t.name for p in parts for t in p.tensors] == [t.name for t in m.tensors]
