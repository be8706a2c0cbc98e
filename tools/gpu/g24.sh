python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_counts.py tests/test_gpu_multirank.py -x -q > gpurun_out/r2_t15.log 2>&1; echo rc=$? >> gpurun_out/r2_t15.log
timeout 600 python tools/time_configs.py C4 > gpurun_out/r2_c4a.log 2>&1
LMFAO_CNT_ROWS_ONLY=1 timeout 600 python tools/time_configs.py C4 >> gpurun_out/r2_c4a.log 2>&1
timeout 600 python tools/time_configs.py C4 >> gpurun_out/r2_c4a.log 2>&1
