python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_counts.py -x -q > gpurun_out/r2_t50.log 2>&1; echo rc=$? >> gpurun_out/r2_t50.log
for k in 4 0 2 8 16; do LMFAO_CNT_HOT=$k timeout 600 python tools/time_configs.py C4 | sed "s/^/hot=$k /" | cut -c1-100 >> gpurun_out/r2_c4hot2.log 2>&1; done
