python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_counts.py -q -x > gpurun_out/r2s3_t7.log 2>&1; echo rc=$? >> gpurun_out/r2s3_t7.log
o=gpurun_out/r2s3_c4h.log
echo default > $o; timeout 600 python tools/time_configs.py C4 >> $o 2>&1
echo runpos0 >> $o; LMFAO_CNT_RUN_POS=0 timeout 600 python tools/time_configs.py C4 >> $o 2>&1
echo runs0 >> $o; LMFAO_CNT_RUNS=0 timeout 600 python tools/time_configs.py C4 >> $o 2>&1
echo viewpos1 >> $o; LMFAO_CNT_VIEW_POS=1 timeout 600 python tools/time_configs.py C4 >> $o 2>&1
echo default >> $o; timeout 600 python tools/time_configs.py C4 >> $o 2>&1
