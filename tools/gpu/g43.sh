python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_cube.py tests/test_gpu_multirank.py tests/test_gpu_next2.py -x -q > gpurun_out/r2_t36.log 2>&1; echo rc=$? >> gpurun_out/r2_t36.log
timeout 600 python tools/time_next2.py > gpurun_out/r2_next2b.log 2>&1
timeout 600 python tools/time_configs.py C5 > gpurun_out/r2_c5i.log 2>&1
