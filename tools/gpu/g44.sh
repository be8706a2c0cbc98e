python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_smoke4.log 2>&1
timeout 1800 python -m pytest tests -x -q -m gpu --durations=10 > gpurun_out/r2_gpufull7.log 2>&1; echo rc=$? >> gpurun_out/r2_gpufull7.log
timeout 600 python bench.py > gpurun_out/r2_bench_default4.log 2>&1
timeout 600 python bench.py --config C5 --no-cpu-baseline > gpurun_out/r2_bench_c5d.log 2>&1
timeout 900 python tools/time_configs.py C1 C2 C3 C4 C5 > gpurun_out/r2_cfg_final4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launch_bench4.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launch_C5m.csv python tools/run_config.py C5 2 > /dev/null 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $N -k "regex:k_view_lin_fast" -s 1 -c 1 -o gpurun_out/r2_vlf_final3 python tools/view_bench.py > gpurun_out/r2_ncu_vlf_final2.log 2>&1
timeout 900 $N -k "regex:k_rec_reduce" -c 1 -o gpurun_out/r2_recred5 python tools/run_config.py C5 1 > gpurun_out/r2_ncu_recred3.log 2>&1
timeout 600 python tools/gram_only.py > gpurun_out/r2_gram_only6.log 2>&1
timeout 600 python tools/view_bench.py > gpurun_out/r2_view14.log 2>&1
timeout 600 python tools/time_next2.py > gpurun_out/r2_next2e.log 2>&1
