python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
LMFAO_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launch_C5.csv python tools/run_config.py C5 2 > /dev/null 2>&1
LMFAO_NO_GRAPH=1 LMFAO_CUBE_ABLATE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3_launch_C5abl.csv python tools/run_config.py C5 2 > /dev/null 2>&1
