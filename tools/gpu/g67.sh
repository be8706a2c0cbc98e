python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 2700 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/r2s3_gpufull.log 2>&1; echo rc=$? >> gpurun_out/r2s3_gpufull.log
timeout 600 python bench.py > gpurun_out/r2s3_bench_full.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2s3_bench_ref.log 2>&1
