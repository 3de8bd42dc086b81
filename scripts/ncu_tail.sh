#!/bin/bash
# ncu --set full of the single-CTA engine running BASELINE config 1 whole (one launch = one solve)
TAG=${1:-r02}; OUT=gpurun_out
NT_B=1 NT_LOGN=10 NT_PT=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:tail_kernel \
  --launch-count 1 -o /tmp/${TAG}_tail -f python scripts/ncu_target.py > $OUT/${TAG}_ncu_tail.log 2>&1
ncu -i /tmp/${TAG}_tail.ncu-rep --page raw --csv > $OUT/${TAG}_ncu_tail_raw.csv 2>/dev/null
ncu -i /tmp/${TAG}_tail.ncu-rep --page source --csv --print-source sass > $OUT/${TAG}_ncu_tail_sass.csv 2>/dev/null
