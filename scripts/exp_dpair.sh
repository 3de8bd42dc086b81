#!/bin/bash
# A/B: coarse down-pass pairs (default) vs TMG_NO_DPAIR=1, same build
OUT=${1:-gpurun_out/exp_dpair.txt}
: > $OUT
for rep in 1 2; do
for env in "" "TMG_NO_DPAIR=1"; do
  echo "[$env] config3 $(env $env timeout 300 python scripts/trace_solve.py 64 22 1 2>&1 | head -1)" >> $OUT
  for pt in 1 0; do
    echo "[$env] config2 p_t=$pt $(env $env timeout 120 python scripts/trace_solve.py 1 20 $pt 2>&1 | head -1)" >> $OUT
  done
done
done
