python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
LMFAO_NO_GRAPH=1 timeout 600 python tools/cov_sweep.py COST=3,5,7,10,14 ABLATE=0,1,8,32,16 > gpurun_out/r2_sweep1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cov -s 3 -c 1 -o gpurun_out/r2_cov1 python tools/run_config.py C2 6 > gpurun_out/r2_ncu1.log 2>&1
