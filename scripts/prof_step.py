"""Break one batched config-3 solve into host overhead, plan.solve and kernels."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1409_5254_b200 as tmg
from paper_1409_5254_b200 import problems, solver

B, n = 64, 1 << 22
F = problems.seeded_rhs_batch_device(1, n, 1.0, 42, list(range(B)))
floors = [1e-12 * float(v) for v in torch.linalg.norm(F.reshape(B, -1), dim=1).cpu()]
hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), 1.0 / n, n, coarsest=2)
cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8)
U = torch.zeros_like(F)
for _ in range(3):
    U.zero_()
    tmg.solve_batched(hier, F, U, cfg, floors=floors, inplace=True)
torch.cuda.synchronize()
plan = solver.get_plan(hier, 0, len(hier.levels), solver.omegas_for(hier, cfg, len(hier.levels)), cfg, B)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for rep in range(3):
    t0 = time.perf_counter()
    ev[0].record()
    U.zero_()
    ev[1].record()
    it, norms, conv = plan.solve(F, U, floors, 1e-8, 250)
    ev[2].record()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"zero {ev[0].elapsed_time(ev[1]):.3f} ms  plan.solve {ev[1].elapsed_time(ev[2]):.3f} ms  "
          f"wall {1e3*(t1-t0):.3f} ms  iters {set(it.tolist())}", flush=True)
for rep in range(3):
    t0 = time.perf_counter()
    ev[0].record()
    U.zero_()
    tmg.solve_batched(hier, F, U, cfg, floors=floors, inplace=True)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"solve_batched step {ev[0].elapsed_time(ev[1]):.3f} ms wall {1e3*(time.perf_counter()-t0):.3f}")
# one cycle alone (no norms) via cycles()
ev[0].record()
plan.cycles(F, U, 5)
ev[1].record()
torch.cuda.synchronize()
print(f"5 cycles (graph, no norms): {ev[0].elapsed_time(ev[1]):.3f} ms")
import os
os.environ["TMG_NO_SOLVE_GRAPH"] = "1"
for rep in range(3):
    ev[0].record()
    it, norms, conv = plan.solve(F, U, floors, 1e-8, 250)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"host-loop solve (per-cycle graph + sync): {ev[0].elapsed_time(ev[1]):.3f} ms")
