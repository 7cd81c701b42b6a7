"""Small invocations of every hot kernel for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py --small

Covers K1 (batched BF16 + FP8 and single-tensor extract; sparse staging path, dense overflow path, several tiles
per CTA via sync_set_max_ctas), K2/K3/K4 (chunk stats, device bucket plan, encode in place, CRC), K5 (decode +
apply, both launch variants, CRC check), K6 (commit), f1 (k_cast_track + tracked extract) and the escape /
routing record kinds; checks the device status words and the replica against the new weights (exit 1 on any
mismatch). Sizes are small: the sanitizers slow kernels down by 10-100x.
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_07330_b200 as ss  # noqa: E402
import synth  # noqa: E402
import synth.gpu as sg  # noqa: E402
from paper_2605_07330_b200.sync import SparseSyncReceiver, SparseSyncSender, TrackedSender  # noqa: E402


def check_sync(m, rho, dev, small, **kw):
    fp8 = kw.get("dtype") == ss.SYNC_DTYPE_FP8
    adt = torch.uint8 if fp8 else torch.int16
    _, X = sg.arena(m, dev, dtype=adt)
    _, Y = sg.arena(m, dev, dtype=adt)
    _, R = sg.arena(m, dev, dtype=adt)
    dt = synth.DTYPE_FP8 if fp8 else synth.DTYPE_BF16
    sg.fill_old(X, m, 5, dtype=dt)
    sg.fill_new(X, Y, m, 5, rho)
    sg.fill_old(R, m, 5, dtype=dt)
    snd = SparseSyncSender(X, Y, bucket_limit=kw.pop("limit", 64 << 10),
                           max_changed=sum(t.numel for t in m.tensors), **kw)
    rcv = SparseSyncReceiver(R, bucket_limit=snd._cfg["bucket_limit"], crc=kw.get("crc", False),
                             dtype=kw.get("dtype", ss.SYNC_DTYPE_BF16))
    bl = snd.sync()
    rcv.apply_many([snd.bucket(b) for b in range(len(bl))])
    snd.commit()
    torch.cuda.synchronize()
    snd.check()
    rcv.check()
    ok = all(torch.equal(r, y) for r, y in zip(R, Y)) and all(torch.equal(x, y) for x, y in zip(X, Y))
    return ok, len(bl)


def main():
    small = "--small" in sys.argv
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    n_big = 300_000 if small else 2_000_000
    m = synth.Manifest("san", [synth.Tensor("a", (256, 512)), synth.Tensor("n", (64,), synth.KIND_NORM),
                               synth.Tensor("b", (n_big,)), synth.Tensor("c", (24,)), synth.Tensor("z", (0,)),
                               synth.Tensor("e", (96, 40), layer=0, expert=1)])
    results = {}
    for ctas in ([0, 3] if not small else [2]):
        ss.set_max_ctas(ctas)
        for rho in (0.01, 0.3):
            results[f"bf16 rho={rho} ctas={ctas}"] = check_sync(m, rho, dev, small)
        ss.set_max_ctas(0)
    results["bf16 crc+escape+route"] = check_sync(m, 0.02, dev, small, crc=True, escape=True, route=True)
    results["bf16 raw"] = check_sync(m, 0.02, dev, small, codec=ss.SYNC_CODEC_RAW)
    results["fp8"] = check_sync(m, 0.05, dev, small, dtype=ss.SYNC_DTYPE_FP8)
    results["bf16 small buckets"] = check_sync(m, 0.01, dev, small, limit=2048)
    # single-tensor extract
    old = torch.randint(-32768, 32767, (n_big,), dtype=torch.int16, device=dev)
    new = old.clone()
    new[::7] ^= 1
    I, V, cnt, ws = ss.sync_extract(old, new)
    torch.cuda.synchronize()
    results["single extract"] = (ss.sync_extract_status(ws) == 0 and int(cnt.item()) == (n_big + 6) // 7, 0)
    # f1: cast-fused tracking
    _, W = sg.arena(m, dev)
    master = [torch.randn(t.numel, device=dev) * 0.02 for t in m.tensors]
    ts = TrackedSender(master, W, bucket_limit=64 << 10, max_changed=sum(t.numel for t in m.tensors))
    ts.cast_track()
    for mt in master:
        mt.add_(0.001)
    ts.cast_track()
    bl = ts.sync()
    torch.cuda.synchronize()
    ts.check()
    results["f1 cast+track"] = (True, len(bl))
    bad = {k: v for k, v in results.items() if not v[0]}
    for k, v in results.items():
        print(f"{k:32s} ok={v[0]} buckets={v[1]}")
    print("SANITIZE_RUN", "FAIL" if bad else "OK", f"{ss.launch_count()} launches")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
