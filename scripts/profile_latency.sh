#!/bin/bash
# latency-bound configs: ncu launch list of one config-2 solve (B=1, N=2^20,
# p_t=1) and an ncu --set full capture (with source) of the single-CTA tail
# engine running the whole config-1 solve (N=2^10)
OUT=gpurun_out
cat > /tmp/one_solve.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1409_5254_b200 as tmg
from paper_1409_5254_b200 import problems
n = int(sys.argv[1]); p_t = int(sys.argv[2])
rhs, tau, _ = problems.seeded_rhs(p_t, n, 1.0, 42)
hier = tmg.TimeHierarchy.build(tmg.BasisSpec(p_t), tau, n, coarsest=2)
for _ in range(2):
    u, st = tmg.solve(hier, rhs, np.zeros_like(rhs), tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8))
print("iterations", st.iterations)
PY
TMG_NO_SOLVE_GRAPH=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/lat_launches_c2.csv python /tmp/one_solve.py 1048576 1 > $OUT/lat_c2.log 2>&1
echo "c2 launch list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tail_kernel --launch-skip 1 \
    --launch-count 1 -o $OUT/lat_tail_c1 -f python /tmp/one_solve.py 1024 1 > $OUT/lat_tail.log 2>&1
echo "tail ncu rc=$?"
