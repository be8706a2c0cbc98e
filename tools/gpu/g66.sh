python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gram.py tests/test_gpu_rt.py tests/test_gpu_snowflake.py tests/test_gpu_next2.py -q -x > gpurun_out/r2s3_t9.log 2>&1; echo rc=$? >> gpurun_out/r2s3_t9.log
timeout 300 python bench.py --steps 2000 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2s3_bench2.log 2>&1
timeout 600 python tools/time_configs.py C1 C2 C3 C4 C5 > gpurun_out/r2s3_cfg.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launch_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
