"""Host-buffer (e2e) solve time of the config-3 batch through the C ABI's
tmg_plan_solve_host, pinned buffers: python scripts/e2e_ab.py [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1409_5254_b200 as tmg  # noqa: E402
from paper_1409_5254_b200 import problems, solver  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
B, n = 64, 1 << 22
F = problems.seeded_rhs_batch_device(1, n, 1.0, 42, list(range(B)))
floors = [1e-12 * float(v) for v in torch.linalg.norm(F.reshape(B, -1), dim=1).cpu()]
hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), 1.0 / n, n, coarsest=2)
cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8)
depth = len(hier.levels)
plan = solver.get_plan(hier, 0, depth, solver.omegas_for(hier, cfg, depth), cfg, B)
Fh = F.cpu().pin_memory()
Uh = torch.empty_like(Fh).pin_memory()
del F
torch.cuda.empty_cache()
plan.solve_host(Fh, None, Uh, floors, cfg.eps, cfg.max_iters)
ts = []
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    it, _, _ = plan.solve_host(Fh, None, Uh, floors, cfg.eps, cfg.max_iters)
    ts.append(time.perf_counter() - t0)
dof = B * n * 2 * float(it.sum()) / B
print(f"chunks={os.environ.get('TMG_HOST_CHUNKS', 'default')} e2e {min(ts) * 1e3:.1f} ms "
      f"(median {sorted(ts)[len(ts) // 2] * 1e3:.1f}), {B * n * 2 * int(it[0]) / min(ts):.3e} time-DoF/s")
