#!/bin/bash
# fp64 dependent-op latency and an ncu --set full capture of the config-1 tail kernel
set -u
TAG=${1:-r02}
OUT=gpurun_out
./scripts/micro/fp64_latency > $OUT/${TAG}_fp64_latency.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tail_kernel --launch-skip 2 \
    --launch-count 1 -o /tmp/${TAG}_tail -f python scripts/tail_target.py > $OUT/${TAG}_ncu_tail.log 2>&1
ncu -i /tmp/${TAG}_tail.ncu-rep --page raw --csv > $OUT/${TAG}_ncu_tail_raw.csv 2>/dev/null
ncu -i /tmp/${TAG}_tail.ncu-rep --page source --csv --print-source sass > $OUT/${TAG}_ncu_tail_sass.csv 2>/dev/null
echo "tail probe done"
