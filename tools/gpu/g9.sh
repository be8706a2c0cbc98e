B=paper_1906_08687_b200/build
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
for lib in paper_1906_08687_b200/liblmfao_gpu.so $B/var_w14/lib.so $B/var_w16/lib.so $B/var_dfma/lib.so $B/var_w14dfma/lib.so; do
  echo "== $lib"; LMFAO_LIB=$lib LMFAO_NO_GRAPH=1 timeout 300 python tools/cov_sweep.py ABLATE=0,32,16
done > gpurun_out/r2_sweep7.log 2>&1
