python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 600 python -m pytest tests/test_gpu_gram.py tests/test_gpu_parity.py -x -q -k "cov or parity or repeated" > gpurun_out/r2_t14a.log 2>&1; echo rc=$? >> gpurun_out/r2_t14a.log
LMFAO_COV_WS=1 timeout 600 python -m pytest tests/test_gpu_gram.py tests/test_gpu_parity.py -x -q -k "cov or parity or repeated" > gpurun_out/r2_t14b.log 2>&1; echo rc=$? >> gpurun_out/r2_t14b.log
for r in 1 2; do
LMFAO_NO_GRAPH=1 timeout 300 python tools/cov_sweep.py ABLATE=0,32,16 > gpurun_out/r2_sweep9_$r.log 2>&1
LMFAO_COV_WS=1 LMFAO_NO_GRAPH=1 timeout 300 python tools/cov_sweep.py ABLATE=0,32,16 > gpurun_out/r2_sweep9ws_$r.log 2>&1
done
