python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
B=paper_1906_08687_b200/build
bash tools/ab_libs.sh paper_1906_08687_b200/liblmfao_gpu.so $B/var_ss16/lib.so $B/var_ss4/lib.so $B/var_fb148/lib.so $B/var_ss16fb148/lib.so > gpurun_out/r2s3_ab_fin.log 2>&1
