#!/bin/bash
# Grid-wide scan solve (N = 2^24, p_t = 1): throughput/error table, ncu launch
# list of the three passes, ncu --set full of the tile-map and replay passes
TAG=${1:-r02}
OUT=gpurun_out
python scripts/scan_bench.py $OUT/${TAG}_scan.json > $OUT/${TAG}_scan.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_scan_launches.csv python scripts/scan_target.py > /dev/null 2>&1
for K in agg replay; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:scan_${K}_kernel --launch-skip 2 \
      --launch-count 1 -o /tmp/${TAG}_scan_$K -f python scripts/scan_target.py > $OUT/${TAG}_ncu_scan_$K.log 2>&1
  ncu -i /tmp/${TAG}_scan_$K.ncu-rep --page raw --csv > $OUT/${TAG}_ncu_scan_${K}_raw.csv 2>/dev/null
done
