ncu --set full --import-source on --clock-control none -k regex:gower_bulk -s 22 -c 2 -f -o /tmp/gab python tools/gower_tiles_ab.py > gpurun_out/gab.log 2>&1
ncu -i /tmp/gab.ncu-rep --page details > gpurun_out/gab_details.txt 2>&1
ncu -i /tmp/gab.ncu-rep --page source --csv -k regex:gower_bulk -c 1 > gpurun_out/gab_src_plain.csv 2>/dev/null
ncu -i /tmp/gab.ncu-rep --page source --csv -k regex:gower_bulk -s 1 -c 1 > gpurun_out/gab_src_tiles.csv 2>/dev/null
ls -la gpurun_out/gab*
