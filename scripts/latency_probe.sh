#!/bin/bash
# Latency-bound configurations: per-phase tail trace (config 1), per-kernel
# live trace of config 2 p_t=1 and p_t=3, and the whole BASELINE suite.
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
timeout 300 python scripts/tail_trace.py 1024 > $OUT/${TAG}_tail_trace_config1.txt 2>&1
timeout 300 python scripts/trace_solve.py 1 20 1 1 > $OUT/${TAG}_trace_config2_p1.txt 2>&1
timeout 300 python scripts/trace_solve.py 1 20 3 1 > $OUT/${TAG}_trace_config2_p3.txt 2>&1
timeout 900 python scripts/bench_suite.py --out $OUT/${TAG}_suite.json > $OUT/${TAG}_suite.log 2>&1
echo "latency probe done"
