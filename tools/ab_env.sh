#!/bin/bash
# tools/ab_env.sh "VAR=a" "VAR=b" ... — C2 step and scan time per environment setting, alternated over
# three passes on one box (bench.py without cpu baseline / e2e; diagnostics)
for r in 1 2 3; do for kv in "$@"; do
  env $kv python bench.py --no-cpu-baseline --no-e2e --steps 2000 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$kv', round(d['ms_per_step'],5), round(d['roofline']['kernel_ms_avg'],5), round(d['roofline']['frac'],4))"
done; done
