python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_load.py tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_edge.py tests/test_gpu_keys.py -q -x > gpurun_out/r2s3_t10.log 2>&1; echo rc=$? >> gpurun_out/r2s3_t10.log
LMFAO_TRACE=1 timeout 600 python tools/e2e_phases.py --keep > gpurun_out/r2s3_e2e2.log 2>&1
timeout 600 python bench.py --steps 500 --e2e-steps 5 > gpurun_out/r2s3_bench3.log 2>&1
