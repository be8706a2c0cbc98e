python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_rt_path.py tests/test_apps.py tests/test_gpu_rt.py -x -q -m gpu > gpurun_out/r2_t11.log 2>&1; echo rc=$? >> gpurun_out/r2_t11.log
timeout 900 python tools/cart_c3.py > gpurun_out/r2_cart.log 2>&1
