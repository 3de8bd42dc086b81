import os, sys
os.environ["TMG_TAIL_TRACE"] = "1"
sys.path.insert(0, ".")
import numpy as np
import paper_1409_5254_b200 as tmg
from paper_1409_5254_b200 import problems
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
rhs, tau, _ = problems.seeded_rhs(1, n, 1.0, 42)
hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), tau, n, coarsest=2)
u, st = tmg.solve(hier, rhs, np.zeros_like(rhs), tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8))
print("iterations", st.iterations, flush=True)
hier.__dict__.pop("_tmg_plans")   # destroy the plan -> trace printed
import gc; gc.collect()
