#!/bin/bash
# A/B: vertical fusion with one-slab lanes (n_t >= 3 fp64; default) vs TMG_NO_VFUSE=1
OUT=${1:-gpurun_out/exp_vfuse_p1.txt}
: > $OUT
for rep in 1 2; do
for env in "" "TMG_NO_VFUSE=1"; do
  for pt in 2 3; do
    echo "[$env] config2 p_t=$pt $(env $env timeout 120 python scripts/trace_solve.py 1 20 $pt 2>&1 | head -1)" >> $OUT
  done
  echo "[$env] B=16 2^22 p_t=2 $(env $env timeout 300 python scripts/trace_solve.py 16 22 2 2>&1 | head -1)" >> $OUT
done
done
