python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_cube.py tests/test_gpu_multirank.py tests/test_gpu_fullsize_c5.py -x -q > gpurun_out/r2_t22.log 2>&1; echo rc=$? >> gpurun_out/r2_t22.log
timeout 600 python tools/time_configs.py C5 > gpurun_out/r2_c5f.log 2>&1
LMFAO_CUBE_MERGE=0 timeout 600 python tools/time_configs.py C5 >> gpurun_out/r2_c5f.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launch_C5h.csv python tools/run_config.py C5 2 > /dev/null 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $N -k "regex:k_cube_rec" -c 1 -o gpurun_out/r2_cuberec2 python tools/run_config.py C5 1 > gpurun_out/r2_ncu_cuberec2.log 2>&1
