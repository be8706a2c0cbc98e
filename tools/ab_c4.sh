#!/bin/bash
# tools/ab_c4.sh [LIB ...] — C4 lmfao_run ms per build (LMFAO_CNT_* knobs from the environment; diagnostics)
for r in 1 2; do
for lib in "$@"; do
  echo "$(LMFAO_LIB=$lib python tools/time_configs.py C4 2>&1 | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["run_ms"])') $lib"
done
done
