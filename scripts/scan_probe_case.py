"""Timing of one scan-solve case through the C ABI: python scripts/scan_probe_case.py p_t log2n B"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1409_5254_b200 as tmg
from paper_1409_5254_b200 import _native as nat, blas_tree
p_t, lg, B = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
n = 1 << lg; nt = p_t + 1
ops = tmg.assemble_local(tmg.BasisSpec(p_t), 1e-3)
rd = torch.randn((B, n, nt), dtype=torch.float64, device="cuda")
out = torch.empty_like(rd)
d = nat.level_desc(ops, n)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
args = (nat.F64, ctypes.byref(d), ctypes.c_void_p(rd.data_ptr()), ctypes.c_void_p(out.data_ptr()), B, 1, blas_tree.resolve(None), st)
L = nat.load()
for _ in range(3): nat.check(L.tmg_coarse_solve(*args), "x")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(5):
    e0.record()
    for _ in range(5): L.tmg_coarse_solve(*args)
    e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 5)
t = min(ts) * 1e-3
print(f"p_t={p_t} n=2^{lg} B={B} run={os.environ.get('TMG_SCAN_RUN','auto')}: {t*1e6:.1f} us (all {[round(x*1e3) for x in ts]}), {2*nt*8*n*B/t/1e9:.0f} GB/s")
