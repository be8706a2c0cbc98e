#!/bin/bash
# tools/ab_cfg.sh CONFIG LIB_A LIB_B — alternate two builds on tools/time_configs.py CONFIG (lmfao_run ms)
for lib in "$2" "$3" "$2" "$3" "$2" "$3"; do
  echo "$lib $(LMFAO_LIB=$lib python tools/time_configs.py $1 2>&1 | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["run_ms"])')"
done
