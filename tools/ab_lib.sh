#!/bin/bash
# tools/ab_lib.sh LIB_A LIB_B [ENV=..] — alternate two builds of liblmfao_gpu.so on bench.py (C2 scan time)
for lib in "$1" "$2" "$1" "$2"; do
  LMFAO_LIB=$lib python bench.py --no-cpu-baseline --no-e2e --steps 2000 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$lib', d['ms_per_step'], d['roofline']['kernel_ms_avg'], d['roofline']['frac'])"
done
