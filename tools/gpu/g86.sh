python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
B=paper_1906_08687_b200/build
o=gpurun_out/r2s3_bigab.log
for r in 1 2; do for lib in paper_1906_08687_b200/liblmfao_gpu.so $B/var_u8/lib.so $B/var_t1k/lib.so $B/var_t1ku8/lib.so; do
echo "== $lib" >> $o; LMFAO_LIB=$lib timeout 600 python tools/time_configs.py C3 >> $o 2>&1
done; done
LMFAO_LIB=$B/var_t1ku8/lib.so timeout 600 python -m pytest tests/test_gpu_rt.py -q -x > gpurun_out/r2s3_t16.log 2>&1; echo rc=$? >> gpurun_out/r2s3_t16.log
