#!/bin/bash
# GPU box: run the gpu test suite, then per-kernel breakdowns of the given workloads.
#   bash tools/gpu_check.sh [workload ...]   (default: dc2 fast3 interp4)
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for wl in ${@:-dc2 fast3 interp4}; do
  python bench.py --workload $wl --steps 10 --warmup 3 --no-e2e --no-cpu --no-companions > gpurun_out/w_$wl.json 2>gpurun_out/w_$wl.log || tail -3 gpurun_out/w_$wl.log
  python -c "
import json; d=json.loads(open('gpurun_out/w_$wl.json').read().strip().splitlines()[-1]); print('$wl', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['kernels_ms_per_step_serialised'].items() if v>0.04})"
done
