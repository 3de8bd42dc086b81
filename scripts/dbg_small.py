"""Small batched solve for compute-sanitizer runs: B problems, n slabs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1409_5254_b200 as tmg
from paper_1409_5254_b200 import problems
n = 1 << int(os.environ.get("LOGN", 16)); B = int(os.environ.get("B", 2))
F = problems.seeded_rhs_batch_device(1, n, 1.0, 42, list(range(B)))
hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), 1.0 / n, n, coarsest=2)
cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8)
res = []
for rep in range(int(os.environ.get("REPS", 1))):
    U = torch.zeros_like(F)
    U, st = tmg.solve_batched(hier, F, U, cfg, inplace=True)
    torch.cuda.synchronize()
    res.append((U.cpu().numpy().copy(), [s.residual_norms for s in st]))
    print(rep, [s.iterations for s in st], flush=True)
print("all reps identical:", all(np.array_equal(r[0], res[0][0]) and r[1] == res[0][1] for r in res))
