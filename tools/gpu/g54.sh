python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
L2=$(bash tools/variant.sh cntnm paper_1906_08687_b200/csrc/counts.cu "-DCNT_NOMATCH=1" | tail -1)
for i in 1 2; do
timeout 600 python tools/time_configs.py C4 | cut -c1-100 >> gpurun_out/r2_c4nm.log 2>&1
LMFAO_LIB=$L2 timeout 600 python tools/time_configs.py C4 | sed 's/^/[NOMATCH] /' | cut -c1-100 >> gpurun_out/r2_c4nm.log 2>&1
done
