python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s5_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2s5_smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2s5_gpufull.log 2>&1; echo rc=$? >> gpurun_out/r2s5_gpufull.log
timeout 600 python bench.py > gpurun_out/r2s5_bench_final.log 2>&1
timeout 600 python bench.py > gpurun_out/r2s5_bench_final2.log 2>&1
timeout 600 python tools/time_configs.py C1 C2 C3 C4 C5 > gpurun_out/r2s5_cfg.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2s5_launches_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
