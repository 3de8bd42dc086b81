"""Determinism probe: repeat one V-cycle (plan.cycles, no norms) and the
single-level entry points on identical inputs; report bitwise differences."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1409_5254_b200 as tmg
from paper_1409_5254_b200 import problems, solver, _native as nat
n = 1 << int(os.environ.get("LOGN", 22)); B = int(os.environ.get("B", 2)); R = int(os.environ.get("REPS", 8))
F = problems.seeded_rhs_batch_device(1, n, 1.0, 42, list(range(B)))
hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), 1.0 / n, n, coarsest=2)
cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8)
depth = len(hier.levels)
plan = solver.get_plan(hier, 0, depth, solver.omegas_for(hier, cfg, depth), cfg, B)
g = torch.Generator(device="cuda").manual_seed(1)
U0 = torch.randn(F.shape, generator=g, device="cuda", dtype=torch.float64)
outs = []
for r in range(R):
    U = U0.clone()
    plan.cycles(F, U, 1)
    torch.cuda.synchronize()
    outs.append(U)
for r in range(1, R):
    d = (outs[r] != outs[0])
    if d.any():
        idx = d.nonzero()
        print("cycle rep", r, "differs at", idx.shape[0], "entries; first", idx[:3].tolist(), "problems", sorted(set(idx[:, 0].tolist())))
print("cycles done")
# solve repeated from U0 (norms)
res = []
for r in range(R // 2):
    U = U0.clone()
    _, st = tmg.solve_batched(hier, F, U, cfg, inplace=True)
    res.append((U.clone(), [s.residual_norms for s in st]))
for r in range(1, len(res)):
    same_u = torch.equal(res[r][0], res[0][0]); same_n = res[r][1] == res[0][1]
    if not (same_u and same_n):
        k = [next((i for i, (a, b) in enumerate(zip(x, y)) if a != b), None) for x, y in zip(res[r][1], res[0][1])]
        print("solve rep", r, "u same", same_u, "norms same", same_n, "first differing norm index per problem", k)
print("solves done")
