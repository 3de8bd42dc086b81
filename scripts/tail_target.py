"""Config 1 (p_t=1, N=2^10, V(1,1) to 1e-8): the whole solve is one tail_kernel
launch -- the ncu target for the latency-bound single-CTA engine."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1409_5254_b200 as tmg  # noqa: E402
from paper_1409_5254_b200 import problems  # noqa: E402

n = int(os.environ.get("TT_N", 1024))
rhs, tau, _ = problems.seeded_rhs(1, n, 1.0, 42)
hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), tau, n, coarsest=2)
cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8)
for _ in range(3):
    u, st = tmg.solve(hier, rhs, np.zeros_like(rhs), cfg)
print("iterations", st.iterations)
