"""BASELINE config 5 alone: one fused pass (2 sweeps + residual + restriction)
over N=2^26 slabs, p_t=3, fp64 and fp32, CUDA-event timed: GB/s algorithmic."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1409_5254_b200 as tmg  # noqa: E402
from paper_1409_5254_b200 import _native as nat  # noqa: E402

n, nt = 1 << 26, 4
tau = 2.0 ** -26
basis = tmg.BasisSpec(3)
ops = tmg.assemble_local(basis, tau)
r1, r2 = tmg.build_transfers(basis, tau)
d = nat.level_desc(ops, n, tmg.optimal_omega(tmg.alpha(basis, tau)), r1, r2)
L = nat.load()
g = torch.Generator(device="cuda").manual_seed(0)
P = lambda t: ctypes.c_void_p(t.data_ptr())
for code, tdt, s in ((0, torch.float64, 8), (1, torch.float32, 4)):
    u = torch.randn((n, nt), generator=g, device="cuda", dtype=torch.float64).to(tdt)
    f = torch.randn((n, nt), generator=g, device="cuda", dtype=torch.float64).to(tdt)
    uo, fc = torch.empty_like(u), torch.empty((n // 2, nt), dtype=tdt, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    run = lambda: nat.check(L.tmg_down(code, ctypes.byref(d), P(f), P(u), P(uo), P(fc), 1, 2, None, st))
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        e0.record(); run(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    t = sorted(ts)[len(ts) // 2]
    print(json.dumps({"dtype": "f64" if code == 0 else "f32", "median_s": t, "GBps": 3.5 * nt * s * n / t / 1e9}))
    del u, f, uo, fc
    torch.cuda.empty_cache()
