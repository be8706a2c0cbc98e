python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_revgroups.py tests/test_apps.py -q -m gpu > gpurun_out/r2_t12.log 2>&1; echo rc=$? >> gpurun_out/r2_t12.log
