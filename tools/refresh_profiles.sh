#!/bin/bash
# GPU box: bench lines for every workload, the ncu launch lists of dc2 /
# interp4 / fast3, and --set full captures of their top kernels (exported to
# text on the box: tools/ncu_full.sh).
#   bash tools/refresh_profiles.sh <tag>      -> gpurun_out/<tag>_*
tag=${1:-r02}
o=gpurun_out
python bench.py --steps 10 --warmup 3 > $o/${tag}_bench_dc2.json 2> $o/${tag}_bench_dc2.log
for wl in fast3 interp4 interp1 img5dc img5fast img5interp; do
  python bench.py --workload $wl --steps 5 --warmup 3 > $o/${tag}_bench_$wl.json 2> $o/${tag}_bench_$wl.log
done
for wl in dc2 interp4 fast3; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $o/${tag}_launches_$wl.csv \
      python bench.py --workload $wl --steps 2 --warmup 3 --no-e2e --no-cpu --no-companions > $o/${tag}_ncu_launch_$wl.log 2>&1
done
bash tools/ncu_full.sh $tag dc2 interp4
echo done
