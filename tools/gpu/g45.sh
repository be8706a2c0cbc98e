python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
timeout 900 python -m pytest tests/test_gpu_next2.py tests/test_gpu_gram.py tests/test_gpu_parity.py -x -q > gpurun_out/r2_t39.log 2>&1; echo rc=$? >> gpurun_out/r2_t37.log
timeout 600 python tools/gram_only.py > gpurun_out/r2_gram_only4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_gram_only_launch4.csv python tools/gram_only.py 100000000 > /dev/null 2>&1
timeout 600 python tools/time_next2.py > gpurun_out/r2_next2c.log 2>&1
