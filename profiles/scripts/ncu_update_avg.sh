#!/bin/bash
# dram bytes of EVERY update_stream_kernel launch of one C5 chunk (the second; the first builds the
# graph), to set beside bench.py's per-launch algorithmic bytes averaged over the same chunk
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --kernel-name-base demangled -k regex:update_stream_kernel -s 224 -c 224 --csv \
  python profiles/c5_probe.py --chunks 2 > gpurun_out/ncu_update_stream_chunk.csv 2>gpurun_out/ncu_update_stream_chunk.err
python - <<'PY'
import csv, json
rows = [r for r in csv.reader(open("gpurun_out/ncu_update_stream_chunk.csv")) if len(r) > 10]
h = rows[0]
ki, mi, ui, vi = h.index("ID"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
per = {}
for r in rows[1:]:
    per.setdefault(r[ki], {})[r[mi]] = float(r[vi].replace(",", "")) * sc.get(r[ui], 1)
n = len(per)
dram = sum(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in per.values()) / n
dur = sum(v["gpu__time_duration.sum"] for v in per.values()) / n
out = {"launches": n, "dram_bytes_per_launch": dram, "dur_us_per_launch": dur, "dram_gbs": dram / (dur * 1e-6) / 1e9}
json.dump(out, open("gpurun_out/ncu_update_stream_chunk.json", "w"), indent=1)
print(out)
PY
