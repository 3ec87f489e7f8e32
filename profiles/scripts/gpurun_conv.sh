timeout 600 python -m pytest tests/test_gpu_conv.py -x -q > gpurun_out/conv_tests.log 2>&1; echo exit=$? >> gpurun_out/conv_tests.log; tail -15 gpurun_out/conv_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv --csv --log-file gpurun_out/conv_probe_ncu.csv python profiles/conv_probe.py --tc 1,3 > gpurun_out/conv_probe.log 2>&1
python profiles/parse_conv_probe.py gpurun_out/conv_probe_ncu.csv gpurun_out/conv_probe.log > gpurun_out/conv_probe_summary.txt
for p in fp32 tf32; do timeout 300 python profiles/c3_resnet.py --prec $p --out gpurun_out/c3_$p.json > gpurun_out/c3_$p.log 2>&1; done
for f in fp32 tf32; do python -c "import json;r=json.load(open(\"gpurun_out/c3_$f.json\"));print(\"$f\", round(r[\"samples_per_s\"]), round(r[\"tflops\"],1), r[\"oacc_last_chunk\"], {k:round(v[\"ms\"],1) for k,v in r[\"classes\"].items()}, r[\"critical_ms\"])"; done
