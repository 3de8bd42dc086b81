#!/bin/bash
# A/B: stopping norm from the finest up pass (default, K_UP2NORM) vs from the
# next cycle's finest down pass (TMG_NORM_IN_DOWN=1, K_DOWNNORM)
OUT=${1:-gpurun_out/exp_norm.txt}
: > $OUT
for rep in 1 2; do
for env in "" "TMG_NORM_IN_DOWN=1"; do
  echo "[$env] config3 $(env $env timeout 300 python scripts/trace_solve.py 64 22 1 2>&1 | head -1)" >> $OUT
  for pt in 0 1 2 3; do
    echo "[$env] config2 p_t=$pt $(env $env timeout 120 python scripts/trace_solve.py 1 20 $pt 2>&1 | head -1)" >> $OUT
  done
done
done
