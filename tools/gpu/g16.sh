python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_views.py tests/test_gpu_parity.py tests/test_gpu_snowflake.py tests/test_gpu_revgroups.py tests/test_gpu_edge.py tests/test_gpu_keys.py -x -q > gpurun_out/r2_t9.log 2>&1; echo rc=$? >> gpurun_out/r2_t9.log
timeout 300 python tools/view_bench.py > gpurun_out/r2_view1.log 2>&1
LMFAO_VIEW_SCAN=1 timeout 300 python tools/view_bench.py >> gpurun_out/r2_view1.log 2>&1
timeout 300 python tools/view_bench.py >> gpurun_out/r2_view1.log 2>&1
