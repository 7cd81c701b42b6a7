"""Regenerate BASELINE.md §4's table from the committed sweep JSONs (dev tool).
usage: python tools/baseline_table.py [sweep dir under profiles/, default r2_sweep]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SWEEP = sys.argv[1] if len(sys.argv) > 1 else "r2_sweep"
try:
    P = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    P = 6537.6
ROWS = [
    ("1M bf16, 99% U (config 1)", "one_1m_r01", "tiny"),
    ("Qwen3-4B 99% U, 1 GPU loopback", "one_4b_r01", ""),
    ("Qwen3-4B 99% U, 1T→1R (config 2)", "pair2_4b_r01", ""),
    ("30B 99% U, 1 GPU (headline)", "one_r01", ""),
    ("30B 99.9% U, 1 GPU", "one_r001", ""),
    ("30B 90% U, 1 GPU (snapshot loopback; the toggle between syncs untimed)", "one_r10_snap", ""),
    ("30B 99% U, ring 2 GPUs", "ring2_r01", ""),
    ("30B 99.9% U, ring 2 GPUs", "ring2_r001", ""),
    ("30B 99% U, 1T→1R", "pair2_r01", ""),
    ("30B 90% U, 1T→1R", "pair2_r10", ""),
    ("30B 99.9% U, 1T→1R", "pair2_r001", ""),
    ("30B 99% U, ring 4 GPUs", "ring4_r01", ""),
    ("30B 99.9% U, ring 4 GPUs", "ring4_r001", ""),
    ("30B 99% U, 2T→2R fanout", "fanout4_r01_U_b256", ""),
    ("30B 90% U, 2T→2R fanout", "fanout4_r10_U_b256", ""),
    ("30B 99.9% U, 2T→2R fanout", "fanout4_r001_U_b256", ""),
    ("30B 99% U, 2T→2R sharded", "sharded4_r01", ""),
    ("235B 99% U, 2 of the 4 shard pairs of 4T→4R, Trainer streaming (config 5)", "sharded4_235b_stream", "stream"),
    ("235B 99% U, 2 of the 4 shard pairs of 4T→4R, f1 tracking, optimizer outside the sync (config 5)",
     "sharded4_235b_f1", "f1"),
    ("235B 99% U, 1 of the 4 shard pairs, f1 tracking (config 5)", "sharded2_235b_f1", "f1"),
    ("30B 99% U, 2T→2R fanout, NCCL sends", "fanout4_r01_U_b256_nccl", ""),
    ("30B 99% U, 2T→2R fanout, NCCL broadcast", "fanout4_r01_U_b256_bcast", ""),
    ("30B 99% R, 2T→2R, 16 MB buckets (config 4)", "fanout4_r01_R_b16", "clustered"),
    ("30B 99% R, 2T→2R, 1 GB buckets (config 4)", "fanout4_r01_R_b1024", "clustered"),
    ("30B 99% E, 2T→2R, 256 MB (config 4)", "fanout4_r01_E_b256", "clustered"),
    ("30B 99% R, 1 GPU, escape-coded (f4)", "one_r01_R_escape", "clustered"),
    ("30B 99% U, 1 GPU, FP16 (f2)", "one_r01_fp16", ""),
    ("30B 99% U, 1 GPU, FP8 (f2)", "one_r01_fp8", "fp8"),
    ("30B 90% U, 1 GPU, FP8 (f2)", "one_r10_fp8", "fp8"),
    ("4B 99% U, f1 cast tracking, 1 GPU", "one_4b_cast", "f1"),
    ("30B 99% U, f1 cast tracking, 2T→2R", "fanout4_r01_cast", "f1"),
]


def main():
    out = ["| Config | GPUs | sync GB/s of weights | % HBM peak, extract+compress | % HBM peak, decompress+apply "
           "(sector model) | Per-update latency (ms) | X_raw / X_comp / α | Bit-exact | JSON |",
           "|---|---|---|---|---|---|---|---|---|"]
    for name, key, kind in ROWS:
        f = os.path.join(ROOT, "profiles", SWEEP, key + ".json")
        if not os.path.exists(f):
            continue
        txt = open(f).read()
        d = json.loads(txt[txt.index("{"):])
        ph, p, c = d["ms_per_phase"], d["payload"], d["config"]
        topo = c["topology_mode"]
        ntr = d["n_gpus"] if topo == "ring" else max(1, d["n_gpus"] // 2)
        eb = 1 if kind == "fp8" else 2
        n_el = c["elements_per_trainer_rank"]
        s_tr = eb * n_el
        pc = p["bytes"] / ntr
        t_xc = (ph["extract"] + ph["compress_pack"]) / 1e3
        if kind == "tiny":
            xc = "launch-bound"
        elif kind == "f1":
            xc = "n/a (f1 reads no 2S)"
        else:
            xc = "%.0f%%" % ((2 * s_tr + pc) / t_xc / 1e9 / P * 100)
        ta = ph["transfer_apply"] / 1e3
        if topo != "ring":
            da = "overlapped (2-GPU pipeline)"
        elif kind == "tiny":
            da = "launch-bound"
        elif kind == "clustered":
            da = "— (clustered sectors)"
        else:
            per = 32 // eb   # elements per 32-byte sector
            fsec = 1 - (1 - p["rho_measured"]) ** per
            da = "%.0f%%" % ((pc + 64 * fsec * n_el / per) / ta / 1e9 / P * 100)
        lat = (d.get("latency_per_update") or {}).get("median_ms")
        lat_s = f"{lat:.2f}"
        if kind == "stream" and "latency_excl_generation_ms" in d.get("stream", {}):   # sync alone
            s = d["stream"]
            lat_s = (f"{s['latency_excl_generation_ms']:.2f} (sync; + {s['generate_ms_per_step']:.0f} ms of input "
                     f"generation per step)")
            xc = "%.0f%%" % ((2 * s_tr + pc) / ((ph["extract"] + ph["compress_pack"]) / 1e3) / 1e9 / P * 100)
        out.append(f"| {name} | {d['n_gpus']} | {d['value']:.0f} | {xc} | {da} | {lat_s} | "
                   f"{p['x_raw_eq1']} / {p['x_comp']} / {p['alpha']} | {d['bit_exact_replica']} | "
                   f"`profiles/{SWEEP}/{key}.json` |")
    tab = "\n".join(out) + "\n"
    path = os.path.join(ROOT, "BASELINE.md")
    b = open(path).read()
    i = b.index("| Config | GPUs | sync GB/s of weights | % HBM peak, extract+compress")
    open(path, "w").write(b[:i] + tab)
    print(tab)


if __name__ == "__main__":
    main()
