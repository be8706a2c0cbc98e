python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $N -k "regex:k_rt_fact" -c 1 -o gpurun_out/r2s3_rtfact python tools/run_config.py C3 1 > gpurun_out/r2s3_ncu_rtfact.log 2>&1
timeout 900 $N -k "regex:k_rt_views" -c 1 -o gpurun_out/r2s3_rtviews python tools/run_config.py C3 1 > gpurun_out/r2s3_ncu_rtviews.log 2>&1
timeout 900 $N -k "regex:k_rt_big" -c 1 -o gpurun_out/r2s3_rtbig python tools/run_config.py C3 1 > gpurun_out/r2s3_ncu_rtbig.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launch_C3.csv python tools/run_config.py C3 2 > /dev/null 2>&1
