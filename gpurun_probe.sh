timeout 300 python -m pytest tests/test_gpu_conv.py -x -q -k kernels > gpurun_out/conv_unit.log 2>&1; echo exit=$? >> gpurun_out/conv_unit.log; tail -2 gpurun_out/conv_unit.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv --csv --log-file gpurun_out/conv_probe_ncu.csv python profiles/conv_probe.py --tc 1,2,3 > gpurun_out/conv_probe.log 2>&1
