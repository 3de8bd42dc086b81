"""fp32 plan solve diagnostics: iterations and residual history vs fp64."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1409_5254_b200 as tmg
from paper_1409_5254_b200 import _native as nat, problems, solver
p_t = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = 1 << int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 16
rhs, tau, _ = problems.seeded_rhs(p_t, n, 1.0, 42)
hier = tmg.TimeHierarchy.build(tmg.BasisSpec(p_t), tau, n, coarsest=2)
cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-5)
u64, st64 = tmg.solve(hier, rhs, np.zeros_like(rhs), cfg)
depth = len(hier.levels)
plan = solver.get_plan(hier, 0, depth, solver.omegas_for(hier, cfg, depth), cfg, 1, nat.F32)
F = torch.from_numpy(rhs).float().cuda()[None]
U = torch.zeros_like(F)
it, norms, conv = plan.solve(F, U, [1e-12 * float(np.linalg.norm(rhs))], cfg.eps, 30)
print("fp64", st64.iterations, [f"{v:.3e}" for v in st64.residual_norms[:6]])
print("fp32", int(it[0]), bool(conv[0]), [f"{v:.3e}" for v in norms[0][:8]])
u32 = U[0].double().cpu().numpy()
print("rel diff", np.linalg.norm(u32 - u64) / np.linalg.norm(u64), "info", plan.info())
