"""Right-hand-side kernels (tmg_rhs.cu) at the headline size: moments of given
samples (tmg_rhs_samples: HBM-bound, reads s and writes n_t doubles per slab)
and of the seeded 8-term sine forcing (tmg_rhs_sines: fp64-sin bound).
    python scripts/rhs_bench.py [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1409_5254_b200 as tmg  # noqa: E402
from paper_1409_5254_b200 import problems, rhs  # noqa: E402

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6546.6


def best(fn, reps=5, inner=5):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(inner):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3 / inner)
    return min(ts)


rows = []
for p_t, B, lg in ((1, 64, 22), (3, 16, 22), (0, 64, 22)):
    n, nt = 1 << lg, p_t + 1
    basis = tmg.BasisSpec(p_t)
    fv = torch.randn((B, n, nt), dtype=torch.float64, device="cuda")
    rhs.rhs_moments_samples(fv, basis, 1.0 / n)
    t_s = best(lambda: rhs.rhs_moments_samples(fv, basis, 1.0 / n))
    nbytes = 2 * nt * 8 * n * B
    ids = list(range(B))
    problems.seeded_rhs_batch_device(p_t, n, 1.0, 42, ids)
    t_q = best(lambda: problems.seeded_rhs_batch_device(p_t, n, 1.0, 42, ids), reps=3, inner=2)
    row = {"p_t": p_t, "batch": B, "n": n,
           "samples_s": t_s, "samples_GBps": nbytes / t_s / 1e9, "samples_frac_of_peak": nbytes / t_s / 1e9 / peak,
           "sines_s": t_q, "sines_write_GBps": nt * 8 * n * B / t_q / 1e9,
           "sines_per_s": 8 * nt * n * B / t_q}
    rows.append(row)
    print(row, flush=True)
    del fv
if len(sys.argv) > 1:
    json.dump(rows, open(sys.argv[1], "w"), indent=1)
