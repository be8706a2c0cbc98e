python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3_smoke2.log 2>&1; echo rc=$? >> gpurun_out/r2s3_smoke2.log
timeout 2700 python -m pytest tests -q -m gpu > gpurun_out/r2s3_gpufull3.log 2>&1; echo rc=$? >> gpurun_out/r2s3_gpufull3.log
timeout 600 python bench.py > gpurun_out/r2s3_bench_final2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launch_c2_final2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $N -k "regex:k_cov<" -s 3 -c 1 -o gpurun_out/r2s3_cov2 python tools/run_config.py C2 6 > gpurun_out/r2s3_ncu_cov2.log 2>&1
timeout 600 python tools/time_configs.py C1 C2 C3 C4 C5 > gpurun_out/r2s3_cfg2.log 2>&1
