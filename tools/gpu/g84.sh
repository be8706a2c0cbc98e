python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
B=paper_1906_08687_b200/build
o=gpurun_out/r2s3_rrab2.log
for r in 1 2 3; do for lib in paper_1906_08687_b200/liblmfao_gpu.so $B/var_rr1/lib.so; do
echo "== $lib" >> $o; LMFAO_LIB=$lib timeout 600 python tools/time_configs.py C5 >> $o 2>&1
done; done
