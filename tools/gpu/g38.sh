python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $N -k "regex:k_view_lin_fast" -s 1 -c 1 -o gpurun_out/r2_vlf python tools/view_bench.py > gpurun_out/r2_ncu_vlf.log 2>&1
