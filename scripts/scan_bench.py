"""Grid-wide scan solve (forward_solve(method="scan"), tmg_coarse_solve method 1):
HBM throughput at N = 2^24 and its error against the extended-precision
solution of the same system (oracle/, test infrastructure) next to the
reference-order serial substitution's own error.
    python scripts/scan_bench.py [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1409_5254_b200 as tmg  # noqa: E402
from oracle import oracle as O  # noqa: E402

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6546.6
rows = []
for p_t, tau, n, B in ((1, 2.0 ** -24, 1 << 24, 1), (1, 1e-6, 1 << 20, 64), (3, 1e-3, 1 << 22, 4),
                       (0, 2.0 ** -10, 1 << 24, 4), (2, 0.5, 1 << 22, 4)):
    ops = tmg.assemble_local(tmg.BasisSpec(p_t), tau)
    nt = p_t + 1
    rhs = np.random.default_rng(n).standard_normal((B, n, nt)) if B > 1 else \
        np.random.default_rng(n).standard_normal((n, nt))
    rd = torch.from_numpy(rhs).cuda()
    sysm = tmg.GlobalSystem(ops, n)
    for _ in range(3):
        got = tmg.forward_solve(sysm, rd, method="scan")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    ts = []
    for _ in range(5):      # best of 5 groups of 10 back-to-back calls
        e0.record()
        for _ in range(reps):
            got = tmg.forward_solve(sysm, rd, method="scan")
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3 / reps)
    t = min(ts)
    gbs = 2 * nt * 8 * n * B / t / 1e9
    # the same through the C ABI directly (tmg_coarse_solve method 1): no
    # per-call Python work (descriptor, output allocation) between the launches
    import ctypes
    from paper_1409_5254_b200 import _native as nat, blas_tree
    d = nat.level_desc(ops, n)
    out = torch.empty_like(rd)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    args = (nat.F64, ctypes.byref(d), ctypes.c_void_p(rd.data_ptr()), ctypes.c_void_p(out.data_ptr()), B, 1,
            blas_tree.resolve(None), st)
    L = nat.load()
    for _ in range(3):
        nat.check(L.tmg_coarse_solve(*args), "tmg_coarse_solve")
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0.record()
        for _ in range(reps):
            L.tmg_coarse_solve(*args)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3 / reps)
    t_abi = min(ts)
    assert torch.equal(out, got)
    x = rhs if B == 1 else rhs[0]
    g = got.cpu().numpy() if B == 1 else got[0].cpu().numpy()
    exact = O.forward_solve_extended(ops, x)
    serial = O.forward_substitute(ops, x)
    nrm = np.linalg.norm(exact)
    row = {"p_t": p_t, "tau": tau, "n": n, "batch": B, "seconds": t, "GBps": gbs, "frac_of_peak": gbs / peak,
           "abi_seconds": t_abi, "abi_GBps": 2 * nt * 8 * n * B / t_abi / 1e9,
           "abi_frac_of_peak": 2 * nt * 8 * n * B / t_abi / 1e9 / peak,
           "scan_vs_exact": float(np.linalg.norm(g - exact) / nrm),
           "serial_vs_exact": float(np.linalg.norm(serial - exact) / nrm),
           "scan_vs_serial": float(np.linalg.norm(g - serial) / nrm)}
    rows.append(row)
    print(row, flush=True)
if len(sys.argv) > 1:
    json.dump(rows, open(sys.argv[1], "w"), indent=1)
