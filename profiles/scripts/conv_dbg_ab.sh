#!/bin/bash
# conv_mma_kernel with its operand copies skipped (FERRET_CONV_DBG=3: A and B not loaded) vs
# normal, 3xTF32 (tc 3) and tf32 (tc 1), forward / input gradient: how much of the kernel time
# the cp.async gathers account for (the bound a TMA operand path could remove)
for dbg in 0 3; do
  FERRET_CONV_DBG=$dbg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python profiles/conv_probe.py --tc 1,3 --modes 0,1 > gpurun_out/conv_dbg_$dbg.csv 2>/dev/null
done
python - <<'PY'
import csv, collections
for dbg in (0, 3):
    rows = [r for r in csv.reader(open(f"gpurun_out/conv_dbg_{dbg}.csv")) if len(r) > 10]
    h = rows[0]
    ni, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot = collections.defaultdict(float)
    for r in rows[1:]:
        if "conv_mma_kernel" in r[ni]:
            key = r[ni].split("(")[0].split("conv_mma_kernel")[1]
            tot[key] += float(r[vi].replace(",", "")) / 1e3
    print("DBG", dbg, {k: round(v, 1) for k, v in sorted(tot.items())}, "us")
PY
