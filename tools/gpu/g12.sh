python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/r2_gpufull.log 2>&1; echo rc=$? >> gpurun_out/r2_gpufull.log
timeout 300 python bench.py --steps 500 --warmup 5 > gpurun_out/r2_bench4.log 2>&1
timeout 600 python tools/time_configs.py C1 C3 C4 C5 > gpurun_out/r2_cfg4.log 2>&1
