python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_views.py tests/test_gpu_parity.py -x -q > gpurun_out/r2_t30.log 2>&1; echo rc=$? >> gpurun_out/r2_t30.log
for i in 1 2; do timeout 300 python tools/view_bench.py >> gpurun_out/r2_view8.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_vb_launch8.csv python tools/view_bench.py > /dev/null 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $N -k "regex:k_view_lin_fast" -s 2 -c 2 -o gpurun_out/r2_vlf6 python tools/view_bench.py > gpurun_out/r2_ncu_vlf2.log 2>&1
