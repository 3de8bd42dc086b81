#!/bin/bash
# Same-box A/B of library variants (scripts/ab_build.sh): graph-mode solve
# times of config 3 (B=64, 2^22, p_t=1) and config 2 (2^20, p_t=1, 3)
#   bash scripts/ab_run.sh out.txt default stage64 ...
OUT=$1; shift
: > $OUT
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = default ]; then LIB=""; else LIB="TMG_LIB=$PWD/build/$v/libtimemg_b200.so"; fi
    echo "[$v] config3 $(env $LIB timeout 300 python scripts/trace_solve.py 64 22 1 2>&1 | grep "graph solve")" >> $OUT
    for pt in 1 3; do
      echo "[$v] config2 p_t=$pt $(env $LIB timeout 120 python scripts/trace_solve.py 1 20 $pt 2>&1 | grep "graph solve")" >> $OUT
    done
  done
done
