"""Kernel-level timing of individual path stages (dev tool; bench.py is the contract).

usage: python tools/xbench.py [workload] [rho] [reps]
Prints one JSON line per stage with CUDA-event times and algorithmic GB/s.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import synth.gpu as sg  # noqa: E402
import paper_2605_07330_b200 as ss  # noqa: E402
from bench import manifest_for  # noqa: E402


def timeit(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "qwen3-4b"
    rho = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    m = manifest_for(wl)
    dev = torch.device("cuda:0")
    _, X = sg.arena(m, dev)
    _, Y = sg.arena(m, dev)
    sg.fill_old(X, m, 0)
    sg.fill_new(X, Y, m, 0, rho)
    snd = ss.SparseSyncSender(X, Y, max_changed=int(m.total * rho * 1.1) + (1 << 20))
    S = 2 * m.total
    tag = {"workload": wl, "rho": rho, "stages": os.environ.get("SS_XSTAGES", "3")}
    # read-only and copy references over the same bytes (torch kernels)
    xa = X[0].new_empty(0).set_(X[0].untyped_storage())  # whole arena
    t_rd = timeit(lambda: xa.view(torch.int64).sum(), reps)
    print(json.dumps({**tag, "stage": "ref_torch_sum_read", "ms": round(t_rd, 4),
                      "GBps": round(2 * m.total / t_rd / 1e6, 1)}))
    for trial in range(int(os.environ.get("XB_TRIALS", "3"))):
        t_ext = timeit(lambda: snd.ctx.sync_extract_batched(snd.old_ptrs, snd.new_ptrs, snd.I, snd.V, snd.counts),
                       reps)
        nnz = int(snd.counts.sum().item())
        snd.check()
        b = 2 * S + 6 * nnz
        print(json.dumps({**tag, "stage": "extract", "trial": trial, "ms": round(t_ext, 4),
                          "GBps": round(b / t_ext / 1e6, 1)}))
    if os.environ.get("XB_ONLY_EXTRACT"):
        return
    t_cmp = timeit(lambda: snd.compress_pack(), reps)   # fused K2-K4, the production path
    st = snd.stats()
    blist = snd.bucket_list
    print(json.dumps({**tag, "stage": "compress_pack", "ms": round(t_cmp, 4), "nnz": nnz, "chunks": st["n_chunks"],
                      "payload": sum(z for _, z in blist)}))
    _, R = sg.arena(m, dev)
    for r, x in zip(R, X):
        r.copy_(x)
    rcv = ss.SparseSyncReceiver(R)

    def apply_all():
        for k in range(len(blist)):
            rcv.apply(snd.bucket(k))
    t_app = timeit(apply_all, reps)
    print(json.dumps({**tag, "stage": "decode_apply", "ms": round(t_app, 4), "buckets": len(blist)}))
    t_com = timeit(lambda: snd.ctx.sync_commit_snapshot_batched(snd.old_ptrs, snd.I, snd.V, snd.counts), reps)
    print(json.dumps({**tag, "stage": "commit", "ms": round(t_com, 4)}))
    rcv.check()
    snd.check()


if __name__ == "__main__":
    main()
