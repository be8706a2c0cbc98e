python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $N -k "regex:k_rec_reduce" -c 1 -o gpurun_out/r2_recred2 python tools/run_config.py C5 1 > gpurun_out/r2_ncu_recred2.log 2>&1
