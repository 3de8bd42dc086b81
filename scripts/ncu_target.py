"""One batched config-3 solve (no solve graph, so ncu sees every kernel):
the target for `ncu -k regex:... --launch-skip` captures of single passes."""
import os
import sys

os.environ.setdefault("TMG_NO_SOLVE_GRAPH", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1409_5254_b200 as tmg  # noqa: E402
from paper_1409_5254_b200 import problems  # noqa: E402

B, n = int(os.environ.get("NT_B", 64)), 1 << int(os.environ.get("NT_LOGN", 22))
p_t = int(os.environ.get("NT_PT", 1))
F = problems.seeded_rhs_batch_device(p_t, n, 1.0, 42, list(range(B)))
floors = [1e-12 * float(v) for v in torch.linalg.norm(F.reshape(B, -1), dim=1).cpu()]
hier = tmg.TimeHierarchy.build(tmg.BasisSpec(p_t), 1.0 / n, n, coarsest=2)
cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8)
U = torch.zeros_like(F)
st = tmg.solve_batched(hier, F, U, cfg, floors=floors, inplace=True)[1]
torch.cuda.synchronize()
print("iterations", sorted({s.iterations for s in st}))
