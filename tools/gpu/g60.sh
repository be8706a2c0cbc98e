python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_counts.py -q > gpurun_out/r2s3_t4.log 2>&1; echo rc=$? >> gpurun_out/r2s3_t4.log
o=gpurun_out/r2s3_c4d.log
echo default > $o; timeout 600 python tools/time_configs.py C4 >> $o 2>&1
echo off >> $o; LMFAO_CNT_VIEWS=0 timeout 600 python tools/time_configs.py C4 >> $o 2>&1
echo min0pos0 >> $o; LMFAO_CNT_VIEW_MIN=0 LMFAO_CNT_VIEW_POS=0 timeout 600 python tools/time_configs.py C4 >> $o 2>&1
echo min0pos1 >> $o; LMFAO_CNT_VIEW_MIN=0 timeout 600 python tools/time_configs.py C4 >> $o 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launch_C4d.csv python tools/run_config.py C4 2 > /dev/null 2>&1
LMFAO_CNT_VIEW_MIN=0 LMFAO_CNT_VIEW_POS=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launch_C4e.csv python tools/run_config.py C4 2 > /dev/null 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
LMFAO_CNT_VIEWS=0 timeout 900 $N -k "regex:k_cnt_rows" -c 1 -o gpurun_out/r2s3_cnt python tools/run_config.py C4 1 > gpurun_out/r2s3_ncu_cnt.log 2>&1
