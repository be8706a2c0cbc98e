python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
L2=$(bash tools/variant.sh minb2 paper_1906_08687_b200/csrc/cube.cu "-DREC_MINB=2" | tail -1)
timeout 900 python -m pytest tests/test_gpu_cube.py tests/test_gpu_multirank.py -x -q > gpurun_out/r2_t20.log 2>&1; echo rc=$? >> gpurun_out/r2_t20.log
for i in 1 2; do
timeout 600 python tools/time_configs.py C5 C5:40000000 > gpurun_out/r2_c5d_$i.log 2>&1
LMFAO_LIB=$L2 timeout 600 python tools/time_configs.py C5 C5:40000000 > gpurun_out/r2_c5d2_$i.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launch_C5f.csv python tools/run_config.py C5 2 > /dev/null 2>&1
N="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $N -k "regex:k_cube_rec" -s 1 -c 1 -o gpurun_out/r2_cuberec python tools/run_config.py C5 1 > gpurun_out/r2_ncu_cuberec.log 2>&1
