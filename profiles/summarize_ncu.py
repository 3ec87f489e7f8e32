"""Summarise ncu raw CSVs (profiles/ncu_capture.sh output): per launch duration,
DRAM traffic, achieved DRAM bandwidth, occupancy, registers."""
import csv
import glob
import json
import os
import sys

KEYS = {"dur_us": "gpu__time_duration.sum", "dram_rd": "dram__bytes_read.sum", "dram_wr": "dram__bytes_write.sum",
        "grid": "launch__grid_size", "regs": "launch__registers_per_thread",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1,
         "msecond": 1e3, "ms": 1e3}


def load(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:70]}
        for k, m in KEYS.items():
            if m in h:
                i = h.index(m)
                try:
                    d[k] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
                except ValueError:
                    d[k] = None
        if d.get("dur_us"):
            d["dram_gbs"] = (d.get("dram_rd", 0) + d.get("dram_wr", 0)) / (d["dur_us"] * 1e-6) / 1e9
        out.append(d)
    return out


if __name__ == "__main__":
    res = {}
    for p in sorted(glob.glob(os.path.join(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out", "ncu_raw_*.csv"))):
        tag = os.path.basename(p)[len("ncu_raw_"):-4]
        res[tag] = load(p)
    print(json.dumps(res, indent=1))
