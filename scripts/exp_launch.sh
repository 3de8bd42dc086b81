#!/bin/bash
# A/B of launch-overhead settings on the latency-bound config 2 (N=2^20) and
# the headline: graph-mode solve times (first line of scripts/trace_solve.py)
OUT=${1:-gpurun_out/exp_launch.txt}
: > $OUT
for env in "" "TMG_NO_PDL=1" "TMG_CHUNK_WAVES=1" "TMG_CHUNK_WAVES=2" "TMG_CHUNK_WAVES=8" "TMG_CHUNK_MIN=4" "TMG_CHUNK_MIN=1"; do
  for pt in 1 3; do
    echo "[$env] p_t=$pt $(env $env timeout 120 python scripts/trace_solve.py 1 20 $pt 2>&1 | head -1)" >> $OUT
  done
done
for env in "" "TMG_NO_PDL=1"; do
  echo "[$env] config3 $(env $env timeout 300 python scripts/trace_solve.py 64 22 1 2>&1 | head -1)" >> $OUT
done
