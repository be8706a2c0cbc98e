python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_b.log 2>&1
LMFAO_TRACE=1 timeout 600 python tools/e2e_phases.py --keep > gpurun_out/r2s3_e2e.log 2>&1
