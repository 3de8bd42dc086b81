#!/bin/bash
# A/B: finest up pass fused with the next cycle's finest down pass (default)
# vs separate K_UP2 + K_DOWNNORM (TMG_NO_FUSE=1), same build
OUT=${1:-gpurun_out/exp_fuse.txt}
: > $OUT
for rep in 1 2; do
for env in "" "TMG_NO_FUSE=1"; do
  echo "[$env] config3 $(env $env timeout 300 python scripts/trace_solve.py 64 22 1 2>&1 | head -1)" >> $OUT
  for pt in 1 3; do
    echo "[$env] config2 p_t=$pt $(env $env timeout 120 python scripts/trace_solve.py 1 20 $pt 2>&1 | head -1)" >> $OUT
  done
done
done
