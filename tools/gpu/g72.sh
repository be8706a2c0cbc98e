python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_rt.py tests/test_gpu_rt_path.py tests/test_gpu_views.py -q -x > gpurun_out/r2s3_t11.log 2>&1; echo rc=$? >> gpurun_out/r2s3_t11.log
o=gpurun_out/r2s3_c3b.log
for r in 1 2; do
echo new >> $o; timeout 600 python tools/time_configs.py C3 >> $o 2>&1
echo old >> $o; LMFAO_LIB=paper_1906_08687_b200/build/var_rtold/lib.so timeout 600 python tools/time_configs.py C3 >> $o 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launch_C3c.csv python tools/run_config.py C3 2 > /dev/null 2>&1
