python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_keys.py tests/test_gpu_parity.py tests/test_gpu_snowflake.py tests/test_gpu_load.py -q -m gpu > gpurun_out/r2_t13.log 2>&1; echo rc=$? >> gpurun_out/r2_t13.log
