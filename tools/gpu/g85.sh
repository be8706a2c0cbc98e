python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3_smoke3.log 2>&1; echo rc=$? >> gpurun_out/r2s3_smoke3.log
timeout 2700 python -m pytest tests -q -m gpu > gpurun_out/r2s3_gpufull5.log 2>&1; echo rc=$? >> gpurun_out/r2s3_gpufull5.log
timeout 600 python bench.py > gpurun_out/r2s3_bench_final4.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2s3_bench_ref2.log 2>&1
timeout 600 python tools/time_configs.py C1 C2 C3 C4 C5 > gpurun_out/r2s3_cfg5.log 2>&1
LMFAO_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launch_C5h.csv python tools/run_config.py C5 2 > /dev/null 2>&1
