python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2_gpufull3.log 2>&1; echo rc=$? >> gpurun_out/r2_gpufull3.log
timeout 600 python tools/time_configs.py C5 C2 > gpurun_out/r2_c5b.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launch_C5d.csv python tools/run_config.py C5 2 > /dev/null 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $N -k "regex:k_cube" -s 1 -c 1 -o gpurun_out/r2_cube2 python tools/run_config.py C5 1 > gpurun_out/r2_ncu_cube2.log 2>&1
