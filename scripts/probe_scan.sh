#!/bin/bash
# ncu --set full of the grid-wide scan solve (N = 2^24, p_t = 1)
TAG=${1:-r02}
OUT=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:scan_solve_kernel --launch-skip 2 --launch-count 1 -o /tmp/${TAG}_scan -f python scripts/scan_target.py > $OUT/${TAG}_ncu_scan.log 2>&1
ncu -i /tmp/${TAG}_scan.ncu-rep --page raw --csv > $OUT/${TAG}_ncu_scan_raw.csv 2>/dev/null
ncu -i /tmp/${TAG}_scan.ncu-rep --page source --csv --print-source sass > $OUT/${TAG}_ncu_scan_sass.csv 2>/dev/null
