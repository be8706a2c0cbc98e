python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
for i in 1 2; do timeout 300 python tools/view_bench.py >> gpurun_out/r2_view12.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/r2_vb_launch12.csv python tools/view_bench.py > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_views.py tests/test_gpu_parity.py tests/test_gpu_load.py -x -q > gpurun_out/r2_t34.log 2>&1; echo rc=$? >> gpurun_out/r2_t34.log
