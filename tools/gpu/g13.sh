python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu --durations=10 --deselect tests/test_gpu_fullsize.py::test_c4_full_sampled_queries > gpurun_out/r2_gpufull2.log 2>&1; echo rc=$? >> gpurun_out/r2_gpufull2.log
