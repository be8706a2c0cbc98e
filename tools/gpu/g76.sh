python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
B=paper_1906_08687_b200/build
LMFAO_LIB=$B/var_xthyb/lib.so timeout 900 python -m pytest tests/test_gpu_gram.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "cov or parity or repeated or c2" -q -x > gpurun_out/r2s3_t14.log 2>&1; echo rc=$? >> gpurun_out/r2s3_t14.log
bash tools/ab_libs.sh paper_1906_08687_b200/liblmfao_gpu.so $B/var_xthyb/lib.so $B/var_xt0/lib.so > gpurun_out/r2s3_ab_xt.log 2>&1
for lib in $B/var_xthyb/lib.so paper_1906_08687_b200/liblmfao_gpu.so; do echo "== $lib"; LMFAO_LIB=$lib LMFAO_NO_GRAPH=1 timeout 300 python tools/cov_sweep.py ABLATE=0,32; done > gpurun_out/r2s3_xt2.log 2>&1
