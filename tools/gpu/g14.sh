python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
for c in C5 C4 C3; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launch_$c.csv python tools/run_config.py $c 2 > gpurun_out/r2_launch_$c.log 2>&1
done
