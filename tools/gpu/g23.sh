B=paper_1906_08687_b200/build
for n in p4r4 p3r4 p2r5; do echo "== $n"; LMFAO_LIB=$B/var_$n/lib.so LMFAO_NO_GRAPH=1 timeout 300 python tools/cov_sweep.py ABLATE=0,16; done > gpurun_out/r2_sweep10.log 2>&1
