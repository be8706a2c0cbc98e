python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_counts.py tests/test_gpu_multirank.py tests/test_gpu_fullsize.py::test_c4_full_sampled_queries -x -q > gpurun_out/r2_t49.log 2>&1; echo rc=$? >> gpurun_out/r2_t47.log
for i in 1 2; do timeout 600 python tools/time_configs.py C4 | cut -c1-100 >> gpurun_out/r2_c4j.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launch_C4d.csv python tools/run_config.py C4 2 > /dev/null 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $N -k "regex:k_cnt_rows" -c 1 -o gpurun_out/r2_cnt4 python tools/run_config.py C4 1 > gpurun_out/r2_ncu_cnt4.log 2>&1
