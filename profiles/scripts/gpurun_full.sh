python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log; tail -1 gpurun_out/bench.log | cut -c1-1500
