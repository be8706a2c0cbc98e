python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_counts.py -q > gpurun_out/r2s3_t3.log 2>&1; echo rc=$? >> gpurun_out/r2s3_t3.log
o=gpurun_out/r2s3_c4c.log
echo default > $o; timeout 600 python tools/time_configs.py C4 >> $o 2>&1
echo off >> $o; LMFAO_CNT_VIEWS=0 timeout 600 python tools/time_configs.py C4 >> $o 2>&1
echo min0pos0 >> $o; LMFAO_CNT_VIEW_MIN=0 LMFAO_CNT_VIEW_POS=0 timeout 600 python tools/time_configs.py C4 >> $o 2>&1
echo min0pos1 >> $o; LMFAO_CNT_VIEW_MIN=0 timeout 600 python tools/time_configs.py C4 >> $o 2>&1
echo min500pos1 >> $o; LMFAO_CNT_VIEW_MIN=500 timeout 600 python tools/time_configs.py C4 >> $o 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launch_C4b.csv python tools/run_config.py C4 2 > /dev/null 2>&1
LMFAO_CNT_VIEW_MIN=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launch_C4c.csv python tools/run_config.py C4 2 > /dev/null 2>&1
