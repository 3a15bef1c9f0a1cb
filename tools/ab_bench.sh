#!/bin/bash
# A/B of two library builds on the bench's device step: bash tools/ab_bench.sh OLD.so workload...
old=$1; shift
for wl in "$@"; do
  for rep in 1 2; do
    for lib in "$old" ""; do
      MDSX_LIB=$lib python bench.py --workload $wl --steps 10 --warmup 3 --no-e2e --no-cpu --no-companions 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms_per_step_serialised']
print('$wl', '${lib:-new}'[-12:], round(d['ms_per_step'],4), {a:round(b,3) for a,b in k.items() if b>0.05})"
    done
  done
done
