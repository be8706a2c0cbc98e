python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 600 python -m pytest tests/test_gpu_gram.py tests/test_gpu_parity.py -x -q > gpurun_out/r2_t3.log 2>&1; echo rc=$? >> gpurun_out/r2_t3.log
LMFAO_NO_GRAPH=1 timeout 600 python tools/cov_sweep.py "PLAN=LMFAO_COV_IB=24,LMFAO_COV_TB=6;LMFAO_COV_IB=16,LMFAO_COV_TB=4;LMFAO_COV_IB=32,LMFAO_COV_TB=8;LMFAO_COV_IB=24,LMFAO_COV_TB=2;LMFAO_COV_IB=48,LMFAO_COV_TB=6" ABLATE=0,32,16 > gpurun_out/r2_sweep3.log 2>&1
timeout 300 python bench.py --steps 500 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench3.log 2>&1
