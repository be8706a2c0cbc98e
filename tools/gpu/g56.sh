python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2s3_smi.log 2>&1
for r in 1 2; do
LMFAO_NO_GRAPH=1 timeout 300 python tools/cov_sweep.py ABLATE=0,1,8,16,17,32,33 > gpurun_out/r2s3_sweep_$r.log 2>&1
done
timeout 300 python bench.py --steps 500 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2s3_bench.log 2>&1
