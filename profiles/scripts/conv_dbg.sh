# time split of the tensor-core conv kernel: all copies / no A copies / no B copies / neither (results invalid, timing only)
for d in 0 1 2 3; do
  FERRET_CONV_DBG=$d timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_mma --csv --log-file gpurun_out/dbg$d.csv python profiles/conv_probe.py --tc 1,3 --modes 0,2 > gpurun_out/dbg$d.log 2>&1
  echo "dbg $d"; python - <<PY
import csv
rows=list(csv.reader(open("gpurun_out/dbg$d.csv")))
h=None
for r in rows:
    if r and r[0]=="ID": h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); print(d["Kernel Name"][30:60], d["Grid Size"], d["Metric Value"])
PY
done
