python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_counts.py -x -q > gpurun_out/r2s3_t1.log 2>&1; echo rc=$? >> gpurun_out/r2s3_t1.log
for v in 1 0 1; do LMFAO_CNT_VIEWS=$v timeout 600 python tools/time_configs.py C4 >> gpurun_out/r2s3_c4.log 2>&1; done
