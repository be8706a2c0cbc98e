python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_counts.py -x -q > gpurun_out/r2s3_t2.log 2>&1; echo rc=$? >> gpurun_out/r2s3_t2.log
for v in 1 0 1; do LMFAO_CNT_VIEWS=$v timeout 600 python tools/time_configs.py C4 >> gpurun_out/r2s3_c4b.log 2>&1; done
LMFAO_CNT_VIEW_POS=0 timeout 600 python tools/time_configs.py C4 >> gpurun_out/r2s3_c4b.log 2>&1
LMFAO_CNT_VIEW_MIN=0 timeout 600 python tools/time_configs.py C4 >> gpurun_out/r2s3_c4b.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launch_C4.csv python tools/run_config.py C4 2 > /dev/null 2>&1
for r in 1 2; do for lib in paper_1906_08687_b200/liblmfao_gpu.so paper_1906_08687_b200/build/var_xtdfma/lib.so; do
  echo "== $lib"; LMFAO_LIB=$lib LMFAO_NO_GRAPH=1 timeout 300 python tools/cov_sweep.py ABLATE=0,32
done; done > gpurun_out/r2s3_xt.log 2>&1
