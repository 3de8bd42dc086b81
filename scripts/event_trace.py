import os, sys
os.environ["TMG_EVENT_TRACE"] = "1"
sys.path.insert(0, ".")
import torch
import paper_1409_5254_b200 as tmg
from paper_1409_5254_b200 import problems
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 22
F = problems.seeded_rhs_batch_device(1, n, 1.0, 42, list(range(B)) if B > 1 else (None,))
hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), 1.0 / n, n, coarsest=2)
cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8)
U = torch.zeros_like(F)
for rep in range(2):
    U.zero_()
    _, st = tmg.solve_batched(hier, F, U, cfg, inplace=True)
    print("iterations", st[0].iterations, file=sys.stderr, flush=True)
