"""Summarise ncu outputs from gpurun_out/ into tracked files under profiles/ (dev tool).

usage: python tools/summarize_profiles.py <tag> <launches.csv> <full.ncu-rep> [algorithmic_bytes_of_profiled_extract]
Writes profiles/<tag>_launches.md, profiles/<tag>_ncu_full.md and (if the
algorithmic byte count of the profiled extract launch is given)
profiles/extract_traffic_<workload>.json for bench.py's roofline.traffic.
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    agg = {}
    for r in rows[hdr + 1:]:
        if len(r) > iv:
            n = r[ik].split("(")[0].replace("void ", "")
            agg.setdefault(n, []).append(float(r[iv].replace(",", "")) / 1e6)
    return agg


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        res.append({"kernel": d["Kernel Name"].split("(")[0].replace("void ", ""),
                    **{k: (d.get(k, ""), units[h.index(k)] if k in h else "") for k in KEYS},
                    "stalls": sorted(((k.replace("smsp__average_warps_issue_stalled_", "")
                                       .replace("_per_issue_active.ratio", ""), float(v or 0))
                                      for k, v in d.items()
                                      if k.startswith("smsp__average_warps_issue_stalled_")
                                      and k.endswith("_per_issue_active.ratio")), key=lambda kv: -kv[1])[:4]})
    return res


def main():
    tag, lpath, fpath = sys.argv[1:4]
    alg = float(sys.argv[4]) if len(sys.argv) > 4 else None
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    agg = launches(lpath)
    synth_k = ("k_fill_old", "k_fill_new")
    timed = {n: v for n, v in agg.items() if n not in synth_k}
    tot = sum(sum(v) for v in timed.values())
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches.md"), "w") as f:
        f.write(f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n")
        f.write("Cold-cache, serialised per-launch times: compare SHARES, not absolutes. Input generation kernels "
                "(k_fill_*) excluded from the shares.\n\n| kernel | launches | total ms | ms/launch | share |\n|---|---|---|---|---|\n")
        for n, v in sorted(timed.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"| {n} | {len(v)} | {sum(v):.3f} | {sum(v) / len(v):.3f} | {100 * sum(v) / tot:.1f}% |\n")
    res = full(fpath)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full.md"), "w") as f:
        f.write(f"# {tag}: ncu --set full (one launch per kernel)\n\n")
        for r in res:
            f.write(f"## {r['kernel']}\n\n| metric | value | unit |\n|---|---|---|\n")
            for k in KEYS:
                v, u = r[k]
                f.write(f"| {k} | {v} | {u} |\n")
            f.write("| top stalls (cycles/issue) | " + ", ".join(f"{a} {b:.2f}" for a, b in r["stalls"]) + " | |\n\n")
    ext = [r for r in res if "k_extract" in r["kernel"]]
    if ext and alg:
        rd, wr = float(ext[0]["dram__bytes_read.sum"][0]), float(ext[0]["dram__bytes_write.sum"][0])
        unit = ext[0]["dram__bytes_read.sum"][1]
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}.get(unit, 1)
        measured = (rd + wr) * scale
        with open(os.path.join(ROOT, "profiles", f"{tag}_extract_traffic.json"), "w") as f:
            json.dump({"profiled_launch_dram_bytes": measured, "profiled_launch_algorithmic_bytes": alg,
                       "ratio": measured / alg}, f, indent=1)
    print("wrote profiles for", tag)


if __name__ == "__main__":
    main()
