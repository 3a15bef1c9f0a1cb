#!/bin/bash
# GPU box: bench lines for every workload, the ncu launch list of the default
# bench command, and --set full captures of the top kernels (dc2, interp4).
#   bash tools/refresh_profiles.sh <tag>      -> gpurun_out/<tag>_*
tag=${1:-r01}
o=gpurun_out
python bench.py --steps 10 --warmup 3 > $o/${tag}_bench_dc2.json 2> $o/${tag}_bench_dc2.log
for wl in fast3 interp4 interp1 img5dc img5fast img5interp; do
  python bench.py --workload $wl --steps 5 --warmup 3 > $o/${tag}_bench_$wl.json 2> $o/${tag}_bench_$wl.log
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $o/${tag}_launches_dc2.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $o/${tag}_ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $o/${tag}_launches_interp4.csv \
    python bench.py --workload interp4 --steps 2 --warmup 3 --no-e2e --no-cpu > $o/${tag}_ncu_launch4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"lanczos|gram_piece|procrustes_fit|dc_stitch|points_piece" -c 5 \
    -o $o/${tag}_dc2_full python tools/profile_run.py dc2 > $o/${tag}_ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"gower_bulk|subtract_mean" -c 2 \
    -o $o/${tag}_interp4_full python tools/profile_run.py interp4 > $o/${tag}_ncu_full4.log 2>&1
echo done
