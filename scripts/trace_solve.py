"""Live per-kernel device times of one solve (the plan's own launches, CUDA
events on the launch stream; tmg_trace_enable) plus the graph-launched time
of the same solve:   python scripts/trace_solve.py [B] [log2 N] [p_t] [nu]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1409_5254_b200 as tmg  # noqa: E402
from paper_1409_5254_b200 import _native as nat, problems, solver  # noqa: E402

solver.TAIL_MAX = int(os.environ.get("TMG_TAIL_MAX", "0"))  # 0 = library default
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 20)
p_t = int(sys.argv[3]) if len(sys.argv) > 3 else 1
nu = int(sys.argv[4]) if len(sys.argv) > 4 else 1
F = problems.seeded_rhs_batch_device(p_t, n, 1.0, 42, list(range(B)))
floors = [1e-12 * float(v) for v in torch.linalg.norm(F.reshape(B, -1), dim=1).cpu()]
hier = tmg.TimeHierarchy.build(tmg.BasisSpec(p_t), 1.0 / n, n, coarsest=2)
cfg = tmg.CycleConfig(nu1=nu, nu2=nu, eps=1e-8)
depth = len(hier.levels)
plan = solver.get_plan(hier, 0, depth, solver.omegas_for(hier, cfg, depth), cfg, B)
U = torch.zeros_like(F)
for _ in range(3):
    U.zero_()
    plan.solve(F, U, floors, cfg.eps, cfg.max_iters)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
U.zero_()
torch.cuda.synchronize()
e0.record()
it, _, _ = plan.solve(F, U, floors, cfg.eps, cfg.max_iters)
e1.record()
torch.cuda.synchronize()
print(f"graph solve: {e0.elapsed_time(e1):.3f} ms, {int(it.max())} cycles, "
      f"{plan.info()['kernels_per_cycle']} kernels per cycle")
L = nat.load()
U.zero_()
L.tmg_trace_enable(1)
plan.solve(F, U, floors, cfg.eps, cfg.max_iters)
buf = ctypes.create_string_buffer(1 << 20)
L.tmg_trace_read(buf, len(buf))
L.tmg_trace_enable(0)
rows = [ln.split("\t") for ln in buf.value.decode().splitlines()]
tot = sum(float(r[2]) for r in rows)
print(f"traced (direct launches): {tot:.3f} ms")
for name, cnt, ms in sorted(rows, key=lambda r: -float(r[2])):
    print(f"{float(ms):9.3f} ms {100 * float(ms) / tot:5.1f}% {int(cnt):5d} {1e3 * float(ms) / int(cnt):9.1f} us/launch  {name}")
