"""Summarise an ncu launch list of profiles/conv_probe.py: per (shape, path, mode)
device time (GEMM + split reduction) and achieved TFLOP/s."""
import csv
import re
import sys


def main(csv_path, log_path):
    rows = list(csv.reader(open(csv_path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[data[0]["Metric Unit"]]
    i = 0
    for line in open(log_path):
        m = re.match(r"shape \((.*)\) tc (\d) mode (\d) gflop ([\d.]+)", line)
        if not m:
            continue
        # one probe call = [weight prep] + GEMM + [split reduction]
        t = 0.0
        if i < len(data) and "wprep" in data[i]["Kernel Name"]:
            t += float(data[i]["Metric Value"]) * scale
            i += 1
        t += float(data[i]["Metric Value"]) * scale
        i += 1
        if i < len(data) and "reduce" in data[i]["Kernel Name"]:
            t += float(data[i]["Metric Value"]) * scale
            i += 1
        gf = float(m.group(4))
        print(f"{m.group(1):26s} tc{m.group(2)} mode{m.group(3)} {t:8.1f} us {gf / (t * 1e-6) / 1e3:7.1f} TFLOP/s")


if __name__ == "__main__":
    main(*sys.argv[1:3])
