python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
for v in "" "LMFAO_RT_NOHASH_KEYS=50000" "LMFAO_RT_NOHASH_KEYS=5000" "LMFAO_RT_NOHASH_KEYS=500"; do env $v timeout 600 python tools/time_configs.py C3 | sed "s/^/[$v] /" | cut -c1-110 >> gpurun_out/r2_c3nh.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_rt.py -x -q > gpurun_out/r2_t44.log 2>&1; echo rc=$? >> gpurun_out/r2_t44.log
