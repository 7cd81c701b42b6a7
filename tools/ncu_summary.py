"""Summarise an ncu report: key metrics per kernel + top SASS stall sites (dev tool).
usage: python tools/ncu_summary.py <file.ncu-rep> [kernel-regex] [--sass N]"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        yield {h: (v, u) for h, v, u in zip(hdr, r, units)}


def main():
    rep = sys.argv[1]
    rx = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
    for d in raw(rep):
        name = d["Kernel Name"][0].split("(")[0]
        if rx and rx not in name:
            continue
        print(f"## {name}")
        for k in KEYS:
            if k in d:
                print(f"  {k:60s} {d[k][0]:>16s} {d[k][1]}")
        stalls = sorted(((float(v[0]), k) for k, v in d.items() if k.startswith("smsp__average_warp_latency_issue_stalled")
                         or k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                         and v[0] not in ("", "n/a")), reverse=True)[:6]
        for v, k in stalls:
            print(f"  stall {k[len('smsp__average_warps_issue_stalled_'):]:52s} {v:8.2f}")


if __name__ == "__main__":
    main()
