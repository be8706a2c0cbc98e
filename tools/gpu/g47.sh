python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_counts.py tests/test_gpu_multirank.py -x -q > gpurun_out/r2_t41.log 2>&1; echo rc=$? >> gpurun_out/r2_t41.log
for k in 8 0 4 16; do LMFAO_CNT_HOT=$k timeout 600 python tools/time_configs.py C4 | sed "s/^/hot=$k /" >> gpurun_out/r2_c4hot.log 2>&1; done
