python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 600 python -m pytest tests/test_gpu_gram.py tests/test_gpu_parity.py -x -q > gpurun_out/r2_t5.log 2>&1; echo rc=$? >> gpurun_out/r2_t5.log
LMFAO_NO_GRAPH=1 timeout 600 python tools/cov_sweep.py "PLAN=LMFAO_COV_TAIL=10;LMFAO_COV_TAIL=20;LMFAO_COV_TAIL=10,LMFAO_COV_COST_COLD=5;LMFAO_COV_TAIL=20,LMFAO_COV_COST_COLD=5" ABLATE=0,32,16,1 > gpurun_out/r2_sweep5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_cov<" -s 3 -c 1 -o gpurun_out/r2_cov5 python tools/run_config.py C2 6 > gpurun_out/r2_ncu5.log 2>&1
