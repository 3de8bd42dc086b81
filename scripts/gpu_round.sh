#!/bin/bash
# One GPU-box validation round (run from the repo root under gpurun):
#   host probe (CPU, numpy BLAS trees), pytest -m gpu, smoke, bench config 3
#   and config 5, then the profiling recipe (launch lists + ncu --set full of
#   the dominant kernels).   Usage: bash scripts/gpu_round.sh TAG [noprof]
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
{ lscpu | head -20; nproc; python -c "import numpy; numpy.show_config()" 2>&1 | head -40;
  python -c "from paper_1409_5254_b200 import blas_tree as b; print('dgemv trees', b.probe())"; } \
  > $OUT/${TAG}_host.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/${TAG}_smi.txt
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?"
tail -3 $OUT/${TAG}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --workload config5 --steps 10 --warmup 3 > $OUT/${TAG}_bench_c5.json 2> $OUT/${TAG}_bench_c5.err
echo "bench c5 rc=$?"
if [ "${2:-}" != "noprof" ]; then bash scripts/profile_round.sh $TAG; fi
