python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_rt.py tests/test_gpu_rt_path.py tests/test_apps.py tests/test_gpu_fullsize.py::test_c3_full_sampled_outputs -x -q -m gpu > gpurun_out/r2_t46.log 2>&1; echo rc=$? >> gpurun_out/r2_t42.log
timeout 600 python tools/time_configs.py C3 C3 > gpurun_out/r2_c3c.log 2>&1
timeout 600 python tools/time_rt_path.py > gpurun_out/r2_rtpath3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launch_C3d.csv python tools/run_config.py C3 2 > /dev/null 2>&1
