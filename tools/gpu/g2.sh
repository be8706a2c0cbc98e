set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gram.py tests/test_gpu_parity.py -x -q > gpurun_out/r2_t1.log 2>&1; echo rc=$? >> gpurun_out/r2_t1.log
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench1.log 2>&1
