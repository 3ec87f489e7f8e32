#!/bin/bash
# dram bytes per launch of a kernel over the SECOND chunk of profiles/c5_probe.py --chunks 2 (the
# bench headline's workload): every launch of both chunks is captured, the last <per_chunk> averaged.
#   profiles/scripts/ncu_chunk_traffic.sh <tag> <kernel-regex> <per_chunk>
tag=$1; k=$2; n=$3
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --kernel-name-base demangled -k "regex:$k" -c $((2 * n + 8)) --csv \
  python profiles/c5_probe.py --chunks 2 > gpurun_out/ncu_chunk_$tag.csv 2>gpurun_out/ncu_chunk_$tag.err
python - "$tag" "$n" <<'PY'
import csv, json, sys
tag, n = sys.argv[1], int(sys.argv[2])
rows = [r for r in csv.reader(open(f"gpurun_out/ncu_chunk_{tag}.csv")) if len(r) > 10]
h = rows[0]
ki, ni, mi, ui, vi = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}
per, name = {}, None
for r in rows[1:]:
    per.setdefault(int(r[ki]), {})[r[mi]] = float(r[vi].replace(",", "")) * sc.get(r[ui], 1)
    name = r[ni]
ids = sorted(per)[-n:]
dram = sum(per[i]["dram__bytes_read.sum"] + per[i]["dram__bytes_write.sum"] for i in ids) / len(ids)
dur = sum(per[i]["gpu__time_duration.sum"] for i in ids) / len(ids)
out = {"kernel": name, "launches_captured": len(per), "launches_averaged": len(ids), "dram_bytes_per_launch": dram,
       "dur_us": dur, "dram_gbs": dram / (dur * 1e-6) / 1e9}
json.dump(out, open(f"gpurun_out/ncu_chunk_{tag}.json", "w"), indent=1)
print(out)
PY
gzip -f gpurun_out/ncu_chunk_$tag.csv
