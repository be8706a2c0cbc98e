python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
LMFAO_NO_GRAPH=1 timeout 900 $N -k "regex:k_radix_scatter" -s 49 -c 1 -o gpurun_out/r2s3_radix_scatter python tools/run_config.py C5 1 > gpurun_out/r2s3_ncu_radix.log 2>&1
LMFAO_NO_GRAPH=1 timeout 900 $N -k "regex:k_radix_hist" -s 49 -c 1 -o gpurun_out/r2s3_radix_hist python tools/run_config.py C5 1 >> gpurun_out/r2s3_ncu_radix.log 2>&1
