python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $N -k "regex:k_cube" -c 1 -o gpurun_out/r2_cube python tools/run_config.py C5 1 > gpurun_out/r2_ncu_cube.log 2>&1
timeout 900 $N -k "regex:k_rec_reduce" -c 1 -o gpurun_out/r2_recred python tools/run_config.py C5 1 > gpurun_out/r2_ncu_recred.log 2>&1
timeout 900 $N -k "regex:k_radix_scatter" -s 8 -c 1 -o gpurun_out/r2_radix python tools/run_config.py C5 1 > gpurun_out/r2_ncu_radix.log 2>&1
timeout 900 $N -k "regex:k_cnt_rows" -c 1 -o gpurun_out/r2_cnt python tools/run_config.py C4 1 > gpurun_out/r2_ncu_cnt.log 2>&1
