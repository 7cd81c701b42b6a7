"""Summarise sweep JSONs (tools/sweep.py) into a markdown table (dev tool).

usage: python tools/sweep_table.py <dir> [<dir> ...] > profiles/<tag>_sweep.md
"""
import glob
import json
import os
import sys


def main():
    rows = []
    for d in sys.argv[1:]:
        for f in sorted(glob.glob(os.path.join(d, "*.json"))):
            try:
                j = json.load(open(f))
            except Exception:
                continue
            c, p, ph = j["config"], j["payload"], j["ms_per_phase"]
            lat = (j.get("latency_per_update") or {}).get("median_ms")
            rows.append([os.path.basename(f)[:-5], j["n_gpus"], c.get("topology_mode"), c.get("workload"),
                         c.get("bucket_mb"), j["value"], j["scaling"], j["ms_per_step"], lat,
                         ph.get("extract"), ph.get("compress_pack"), ph.get("transfer_apply"),
                         j["roofline"]["frac"], p["x_comp"], p["x_raw_eq1"], p["alpha"], p["abs32_records"],
                         j["bit_exact_replica"]])
    hdr = ["run", "N", "topology", "workload", "bucket MB", "GB/s", "scaling", "ms/step", "latency ms",
           "extract ms", "compress+pack ms", "transfer+apply ms", "K1 frac", "X_comp", "X_raw", "alpha",
           "ABS32 records", "bit-exact"]
    print("| " + " | ".join(hdr) + " |")
    print("|" + "---|" * len(hdr))
    for r in rows:
        print("| " + " | ".join("" if v is None else (f"{v:.4g}" if isinstance(v, float) else str(v)) for v in r)
              + " |")


if __name__ == "__main__":
    main()
