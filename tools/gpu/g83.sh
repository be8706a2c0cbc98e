python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_cube.py tests/test_gpu_fullsize_c5.py tests/test_gpu_multirank.py tests/test_gpu_load.py -q -x > gpurun_out/r2s3_t15.log 2>&1; echo rc=$? >> gpurun_out/r2s3_t15.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/r2s3_smi2.log 2>&1
for r in 1 2; do timeout 600 python tools/time_configs.py C1 C2 C3 C4 C5 >> gpurun_out/r2s3_cfg4.log 2>&1; done
LMFAO_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launch_C5g.csv python tools/run_config.py C5 2 > /dev/null 2>&1
