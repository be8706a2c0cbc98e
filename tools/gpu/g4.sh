L1=paper_1906_08687_b200/build/var_xxd/lib.so
for lib in paper_1906_08687_b200/liblmfao_gpu.so $L1; do
  echo "== $lib"
  LMFAO_LIB=$lib LMFAO_NO_GRAPH=1 timeout 600 python tools/cov_sweep.py COST=4,5,6 ABLATE=0,32
done > gpurun_out/r2_sweep2.log 2>&1
LMFAO_COV_COLD_ALL=0 timeout 300 python -m pytest tests/test_gpu_gram.py -x -q -k cov > gpurun_out/r2_t2.log 2>&1
LMFAO_LIB=$L1 timeout 300 python -m pytest tests/test_gpu_gram.py -x -q -k cov >> gpurun_out/r2_t2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_cov<" -s 3 -c 1 -o gpurun_out/r2_cov2 python tools/run_config.py C2 6 > gpurun_out/r2_ncu2.log 2>&1
