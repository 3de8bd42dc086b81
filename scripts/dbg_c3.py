import sys, hashlib, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_1409_5254_b200 as tmg
from paper_1409_5254_b200 import problems
from conftest import *  # noqa
import json
man = json.load(open("tests/golden/golden.json"))
cases = [x for x in man["big_solves"] if x["name"].startswith("config3_b")]
n = cases[0]["n"]; print("n", n, "B", len(cases))
rhs = [problems.seeded_rhs(1, n, 1.0, 42, c["batch_index"])[0] for c in cases]
hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), 1.0 / n, n, coarsest=2)
cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8)
for mode in ("host", "dev"):
    if mode == "host":
        U, stats = tmg.solve_batched(hier, np.stack(rhs), None, cfg)
    else:
        F = torch.from_numpy(np.stack(rhs)).cuda(); U = torch.zeros_like(F)
        U, stats = tmg.solve_batched(hier, F, U, cfg, inplace=True); U = U.cpu().numpy()
    for b, c in enumerate(cases):
        a = np.array(stats[b].residual_norms); g = np.array(c["residual_norms"])
        d = np.nonzero(a != g)[0] if len(a) == len(g) else "len"
        print(mode, b, stats[b].iterations, c["iterations"], "diff idx", d, (a[d] / g[d] - 1) if len(a) == len(g) and len(d) else "",
              hashlib.sha256(np.ascontiguousarray(U[b]).tobytes()).hexdigest() == c["sha_u"])
