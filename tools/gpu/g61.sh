python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_counts.py -q > gpurun_out/r2s3_t5.log 2>&1; echo rc=$? >> gpurun_out/r2s3_t5.log
o=gpurun_out/r2s3_c4f.log
echo default > $o; timeout 600 python tools/time_configs.py C4 >> $o 2>&1
echo nopack >> $o; LMFAO_CNT_PACK=0 timeout 600 python tools/time_configs.py C4 >> $o 2>&1
echo noviews >> $o; LMFAO_CNT_VIEWS=0 timeout 600 python tools/time_configs.py C4 >> $o 2>&1
echo default >> $o; timeout 600 python tools/time_configs.py C4 >> $o 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launch_C4f.csv python tools/run_config.py C4 2 > /dev/null 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $N -k "regex:k_cnt_rows" -c 1 -o gpurun_out/r2s3_cnt2 python tools/run_config.py C4 1 > gpurun_out/r2s3_ncu_cnt2.log 2>&1
