"""One grid-wide scan solve at N = 2^24, p_t = 1 (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1409_5254_b200 as tmg  # noqa: E402

n = 1 << 24
ops = tmg.assemble_local(tmg.BasisSpec(1), 2.0 ** -24)
rd = torch.from_numpy(np.random.default_rng(0).standard_normal((n, 2))).cuda()
for _ in range(3):
    u = tmg.forward_solve(tmg.GlobalSystem(ops, n), rd, method="scan")
torch.cuda.synchronize()
print("done")
