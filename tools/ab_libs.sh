#!/bin/bash
# tools/ab_libs.sh LIB... — C2 scan time per build, two passes (bench.py, no cpu baseline / e2e; diagnostics)
for r in 1 2; do for lib in "$@"; do
  LMFAO_LIB=$lib python bench.py --no-cpu-baseline --no-e2e --steps 2000 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$lib', round(d['ms_per_step'],5), round(d['roofline']['kernel_ms_avg'],5), round(d['roofline']['frac'],4))"
done; done
