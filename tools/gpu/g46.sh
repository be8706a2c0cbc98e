python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gram.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py::test_c2_full_all_780_outputs tests/test_gpu_multirank.py -x -q > gpurun_out/r2_t40.log 2>&1; echo rc=$? >> gpurun_out/r2_t40.log
LMFAO_TRACE=1 timeout 600 python tools/e2e_phases.py > gpurun_out/r2_e2e_trace2.log 2>&1
timeout 600 python bench.py --steps 500 > gpurun_out/r2_bench_e2e.log 2>&1
