python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_cube.py tests/test_gpu_next2.py -q -x > gpurun_out/r2s3_t13.log 2>&1; echo rc=$? >> gpurun_out/r2s3_t13.log
timeout 600 python tools/time_configs.py C5 > gpurun_out/r2s3_c5b.log 2>&1
LMFAO_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launch_C5t.csv python tools/run_config.py C5 2 > /dev/null 2>&1
