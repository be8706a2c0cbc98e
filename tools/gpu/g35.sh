python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_smoke.log 2>&1
timeout 1800 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/r2_gpufull4.log 2>&1; echo rc=$? >> gpurun_out/r2_gpufull4.log
timeout 600 python bench.py > gpurun_out/r2_bench_default.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/r2_bench_ref.log 2>&1
timeout 600 python bench.py --config C5 --no-cpu-baseline > gpurun_out/r2_bench_c5.log 2>&1
timeout 900 python tools/time_configs.py C1 C2 C3 C4 C5 > gpurun_out/r2_cfg_final1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launch_bench.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $N -k "regex:k_cov<" -s 3 -c 1 -o gpurun_out/r2_cov_final python tools/run_config.py C2 6 > gpurun_out/r2_ncu_cov_final.log 2>&1
