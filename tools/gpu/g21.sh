python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
for r in 1 2; do for lib in paper_1906_08687_b200/liblmfao_gpu.so paper_1906_08687_b200/build/var_dual/lib.so; do
  echo "== $lib"; LMFAO_LIB=$lib LMFAO_NO_GRAPH=1 timeout 300 python tools/cov_sweep.py ABLATE=0,32
done; done > gpurun_out/r2_sweep8.log 2>&1
