#!/bin/bash
# GPU box: --set full captures of the top kernels of the given workloads,
# exported to text on the box (the .ncu-rep files are too large to bring back).
#   bash tools/ncu_full.sh <tag> [workload ...]
#   -> gpurun_out/<tag>_ncu_full_<wl>.txt (details page), <tag>_ncu_src_<wl>_<kernel>.csv
tag=${1:-r02}; shift
o=gpurun_out
for wl in ${@:-dc2 interp4}; do
  case $wl in
    dc2|fast3) k='regex:lanczos|gram_piece|procrustes_fit|piece_out|rows_points|trk_points'; c=6 ;;
    interp4) k='regex:gower_bulk|subtract_mean'; c=2 ;;
    img5*) k='regex:bgemm|gram_tile|bk_'; c=6 ;;
  esac
  [ -n "$NCU_K" ] && k="regex:$NCU_K" && c=${NCU_C:-4}
  python tools/profile_run.py $wl > $o/${tag}_${wl}_plain.log 2>&1 || { echo "plain run failed: $wl"; tail -3 $o/${tag}_${wl}_plain.log; continue; }
  rep=/tmp/${tag}_${wl}_full
  ncu --set full --import-source on --clock-control none -k "$k" -c $c \
      -f -o $rep python tools/profile_run.py $wl > $o/${tag}_${wl}_full.log 2>&1
  ncu -i $rep.ncu-rep --page details > $o/${tag}_ncu_full_${wl}.txt 2>&1
  # per-launch DRAM traffic and duration (bench.py TRAFFIC / roofline.traffic)
  ncu -i $rep.ncu-rep --page raw --csv \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      > $o/${tag}_ncu_dram_${wl}.csv 2>/dev/null
  for kn in ${NCU_SRC:-gram_piece lanczos_smem piece_out gower_bulk}; do
    ncu -i $rep.ncu-rep --page source --csv -k regex:$kn -c 1 > $o/${tag}_ncu_src_${wl}_${kn}.csv 2>/dev/null
    [ -s $o/${tag}_ncu_src_${wl}_${kn}.csv ] || rm -f $o/${tag}_ncu_src_${wl}_${kn}.csv
  done
  tail -1 $o/${tag}_${wl}_full.log
done
