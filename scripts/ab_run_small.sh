#!/bin/bash
# Same-box A/B of library variants on the latency-bound configurations:
# config 1 (2^10), config 2 (2^20, p_t = 1), config 4 (2^20, p_t = 2 needs the n_t = 3 units)
#   bash scripts/ab_run_small.sh out.txt default v5 ...
OUT=$1; shift
: > $OUT
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = default ]; then LIB=""; else LIB="TMG_LIB=$PWD/build/$v/libtimemg_b200.so"; fi
    echo "[$v] config1 $(env $LIB timeout 120 python scripts/trace_solve.py 1 10 1 2>&1 | grep "graph solve")" >> $OUT
    echo "[$v] config2 p_t=1 $(env $LIB timeout 120 python scripts/trace_solve.py 1 20 1 2>&1 | grep "graph solve\|tail_kernel" | tr '\n' ' ')" >> $OUT
    echo "[$v] 2^14 p_t=1 $(env $LIB timeout 120 python scripts/trace_solve.py 1 14 1 2>&1 | grep "graph solve")" >> $OUT
  done
done
