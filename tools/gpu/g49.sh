python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
for v in "" "LMFAO_CNT_SMEM_CELLS=0" "LMFAO_CNT_SMEM_CELLS=8192" "LMFAO_CNT_SMEM_CELLS=50000" "LMFAO_CNT_THREADS=512"; do env $v timeout 600 python tools/time_configs.py C4 | sed "s/^/[$v] /" | cut -c1-120 >> gpurun_out/r2_c4ab.log 2>&1; done
