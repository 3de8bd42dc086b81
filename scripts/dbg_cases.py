"""Run solve cases one per subprocess (a fault in one does not hide the rest)."""
import os, subprocess, sys
CASES = [(2, 1 << 16), (1, 1 << 16), (2, 1 << 12), (1, 1 << 12), (3, 1 << 14), (0, 1 << 16)]
code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
import paper_1409_5254_b200 as tmg
from paper_1409_5254_b200 import problems
p_t, n = int(sys.argv[1]), int(sys.argv[2])
rhs, tau, _ = problems.seeded_rhs(p_t, n, 1.0, 42)
hier = tmg.TimeHierarchy.build(tmg.BasisSpec(p_t), tau, n, coarsest=2)
u, st = tmg.solve(hier, rhs, np.zeros_like(rhs), tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8))
print("ok", p_t, n, st.iterations, st.residual_norms[-1])
'''
for p_t, n in CASES:
    r = subprocess.run([sys.executable, "-c", code, str(p_t), str(n)], capture_output=True, text=True,
                       env={**os.environ, "TMG_SYNC_DEBUG": "1"}, timeout=300)
    print(p_t, n, "rc", r.returncode, r.stdout.strip()[-300:], r.stderr.strip()[-600:], flush=True)
