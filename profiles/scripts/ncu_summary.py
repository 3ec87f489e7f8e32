"""Summarise an ncu capture exported by profiles/scripts/ncu_group_src.sh: speed-of-light,
occupancy, stall reasons (pc sampling) and the hottest SASS lines with their neighbours.
    python profiles/scripts/ncu_summary.py <tag>   (reads gpurun_out/ncu_{details,raw,sass}_<tag>.csv)"""
import csv
import sys

tag = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/ncu_details_{tag}.csv")))
hdr = rows[0]
keep = ("Duration", "DRAM Throughput", "Memory Throughput", "Issue Slots Busy", "Achieved Active Warps Per SM",
        "Registers Per Thread", "Warp Cycles Per Issued Instruction", "L2 Hit Rate", "L1/TEX Hit Rate")
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in keep:
        print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
rows = list(csv.reader(open(f"gpurun_out/ncu_raw_{tag}.csv")))
for h, x in zip(rows[0], rows[2]):
    if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
        try:
            if float(x.replace(",", "")) > 200:
                print("  stall", h.replace("smsp__pcsamp_warps_issue_stalled_", ""), x)
        except ValueError:
            pass
rows = list(csv.reader(open(f"gpurun_out/ncu_sass_{tag}.csv")))
hdr, data = rows[1], rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
samp = [int(r[iS]) if r[iS].isdigit() else 0 for r in data]
print("samples", sum(samp))
for i in sorted(range(len(data)), key=lambda i: -samp[i])[:int(sys.argv[2]) if len(sys.argv) > 2 else 6]:
    print("----")
    for j in range(max(0, i - 6), min(len(data), i + 2)):
        print(f"{samp[j]:6d} {data[j][0][-5:]} {data[j][1].strip()[:100]}")
