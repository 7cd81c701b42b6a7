"""CPU checks of bench.py's contract pieces that need no GPU: the reference arm (the oracle on a bounded
sample) prints one JSON line with the contract keys, and the product path refuses CPU tensors (no CPU
fallback exists)."""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "1m", "--steps", "2",
                          "--warmup", "1", "--ref-sample-elems", "2e6"], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_product_path_has_no_cpu_fallback():
    import paper_2605_07330_b200 as ss
    old = torch.zeros(64, dtype=torch.bfloat16)
    new = old.clone()
    with pytest.raises(Exception):
        ss.sync_extract(old, new)            # CPU tensors: the binding refuses, nothing runs on the host


def test_stream_groups_fit_the_scratch():
    """Config 5's streaming split: the fewest contiguous groups whose largest fits the scratch; a tensor larger
    than the scratch ends up alone (the scratch is then sized to it)."""
    sys.path.insert(0, ROOT)
    import synth
    from bench import stream_groups
    from paper_2605_07330_b200.transport import shard_ranges
    m = synth.qwen3_manifest("qwen3-235b-a22b")
    lo, hi = shard_ranges(m.numel, 4)[0]
    numel = m.numel[lo:hi]
    G = stream_groups(numel, 5)
    assert max(sum(numel[a:b]) for a, b in shard_ranges(numel, G)) * 2 <= 5e9
    assert G == 1 or max(sum(numel[a:b]) for a, b in shard_ranges(numel, G - 1)) * 2 > 5e9
    assert stream_groups([10, 10, 10], 1e-7) == 1          # 60 bytes fit a 100-byte scratch
    assert stream_groups([10, 10, 10], 4e-8) == 2          # 40-byte scratch: 20 + 10 elements
    assert stream_groups([100, 1, 1], 1e-7) == 3           # a 200-byte tensor can only go alone
