#!/bin/bash
# A/B of the single-CTA tail threshold (slabs per problem) on config 2
OUT=${1:-gpurun_out/exp_tail.txt}
: > $OUT
for tm in 0 256 512 1024 4096; do
  for pt in 1 3; do
    echo "[tail_max=$tm] p_t=$pt $(TMG_TAIL_MAX=$tm timeout 120 python scripts/trace_solve.py 1 20 $pt 2>&1 | head -1)" >> $OUT
  done
done
echo "[tail_max=0] config1 $(timeout 120 python scripts/trace_solve.py 1 10 1 2>&1 | head -1)" >> $OUT
