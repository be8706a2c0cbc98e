python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_views.py tests/test_gpu_parity.py tests/test_gpu_revgroups.py -x -q > gpurun_out/r2_t24.log 2>&1; echo rc=$? >> gpurun_out/r2_t24.log
for i in 1 2; do
timeout 300 python tools/view_bench.py >> gpurun_out/r2_view2.log 2>&1
LMFAO_VIEW_FAST=0 timeout 300 python tools/view_bench.py >> gpurun_out/r2_view2.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_vb_launch.csv python tools/view_bench.py > /dev/null 2>&1
