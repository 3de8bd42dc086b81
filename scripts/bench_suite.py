"""All BASELINE configurations on one GPU (evidence for DESIGN.md / profiles).

    python scripts/bench_suite.py [--out profiles/r01_suite.json] [--quick]

config 1: p_t=1, N=2^10, V(1,1) to 1e-8 (latency: wall time per solve)
config 2: N=2^20, p_t=0..3, V(1,1) to 1e-8
config 3: see bench.py (the headline)
config 4: N=2^20, p_t=2, T in {1e-2, 1, 1e2}, nu in {1, 2}, V- and W-cycles
config 5: one fused pass (2 sweeps + residual + restriction), N=2^26, p_t=3,
          fp64 and fp32; the first 2^16 slabs are the seeded numpy inputs of
          the golden vector and the output prefix is checked against it
All solves: seeded problems, zero initial guess, coarsest 2.
Times are CUDA-event device times of the public API calls with the inputs
already on the GPU; small working sets get an L2 flush before each timed solve.
"""

import argparse
import ctypes
import hashlib
import json
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1409_5254_b200 as tmg  # noqa: E402
from paper_1409_5254_b200 import _native as nat, problems, solver  # noqa: E402

FLUSH = None


def flush_l2():
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    FLUSH.zero_()


def timed(fn, reps, flush=True):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    out = None
    for _ in range(reps):
        if flush:
            flush_l2()
        torch.cuda.synchronize()
        ev0.record()
        out = fn()
        ev1.record()
        torch.cuda.synchronize()
        ts.append(ev0.elapsed_time(ev1) * 1e-3)
    return min(ts), sorted(ts)[len(ts) // 2], out


def solve_case(p_t, n, T, nu, cycle="V", reps=5, coarsest=2, coarse="auto"):
    rhs = problems.seeded_rhs_batch_device(p_t, n, T, 42, (None,))[0]
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(p_t), T / n, n, coarsest=coarsest)
    cfg = tmg.CycleConfig(nu1=nu, nu2=nu, eps=1e-8, cycle=cycle, coarse=coarse)
    u = torch.zeros_like(rhs)
    floor = 1e-12 * float(torch.linalg.norm(rhs))

    def run():
        u.zero_()
        return tmg.solve_batched(hier, rhs[None], u[None], cfg, floors=[floor], inplace=True)[1][0]

    run()
    best, med, st = timed(run, reps)
    dofs = n * (p_t + 1) * st.iterations
    return {"p_t": p_t, "n": n, "T": T, "nu": nu, "cycle": cycle, "coarsest": hier.levels[-1].n_steps,
            "coarse_solver": coarse, "iterations": st.iterations,
            "best_s": best, "median_s": med, "time_dof_per_s": dofs / med,
            "final_norm": st.residual_norms[-1]}


def config5(reps=10):
    n, nt = 1 << 26, 4
    tau = 2.0 ** -26
    basis = tmg.BasisSpec(3)
    ops = tmg.assemble_local(basis, tau)
    r1, r2 = tmg.build_transfers(basis, tau)
    om = tmg.optimal_omega(tmg.alpha(basis, tau))
    d = nat.level_desc(ops, n, om, r1, r2)
    L = nat.load()
    g = torch.Generator(device="cuda").manual_seed(0)
    res = {}
    up, fp = problems.kernel_inputs(1 << 16, nt, 0)
    golden = json.load(open(os.path.join(REPO, "tests", "golden", "golden.json")))["config5"]
    for dtype, tdt, code in (("f64", torch.float64, 0), ("f32", torch.float32, 1)):
        u = torch.randn((n, nt), generator=g, device="cuda", dtype=torch.float64)
        f = torch.randn((n, nt), generator=g, device="cuda", dtype=torch.float64)
        u[: 1 << 16] = torch.from_numpy(up).cuda()
        f[: 1 << 16] = torch.from_numpy(fp).cuda()
        u, f = u.to(tdt), f.to(tdt)
        uo = torch.empty_like(u)
        fc = torch.empty((n // 2, nt), dtype=tdt, device="cuda")
        P = lambda t: ctypes.c_void_p(t.data_ptr())

        def run():
            nat.check(L.tmg_down(code, ctypes.byref(d), P(f), P(u), P(uo), P(fc), 1, 2, None,
                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))

        run()
        best, med, _ = timed(run, reps, flush=False)  # 7.5 GB per pass >> L2
        s = 8 if dtype == "f64" else 4
        algo = 3.5 * nt * s * n
        entry = {"bytes": algo, "best_s": best, "median_s": med, "GBps": algo / med / 1e9}
        head_u = uo[: 1 << 16].double().cpu().numpy()
        head_fc = fc[: 1 << 15].double().cpu().numpy()
        if dtype == "f64":
            entry["prefix_u_sha_match"] = hashlib.sha256(head_u.tobytes()).hexdigest() == golden["sha_u"]
            entry["prefix_fc_sha_match"] = hashlib.sha256(head_fc.tobytes()).hexdigest() == golden["sha_fc"]
        else:
            from oracle import oracle as O  # checker only
            ru, rfc = O.down_pass(ops, r1, r2, om, up, fp, 2)
            entry["prefix_u_rel"] = float(np.linalg.norm(head_u - ru) / np.linalg.norm(ru))
            entry["prefix_fc_rel"] = float(np.linalg.norm(head_fc - rfc) / np.linalg.norm(rfc))
        res[dtype] = entry
        del u, f, uo, fc
        torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(REPO, "MEASURED_PEAKS.json")) else 6650.0
    out = {"gpu": torch.cuda.get_device_name(0), "peak_hbm_gbs": peak}
    out["config1"] = solve_case(1, 1 << 10, 1.0, 1, reps=20)
    print("config1", out["config1"], flush=True)
    out["config2"] = [solve_case(p, 1 << 20, 1.0, 1) for p in range(4)]
    for r in out["config2"]:
        print("config2", r, flush=True)
    if not args.quick:
        # V and F down to 2 slabs (the reference setting); V and W over a 1024-slab
        # coarsest level solved by the parallel scan (a deep W-cycle visits the
        # 2-slab level 2^19 times per cycle -- inherently sequential, see DESIGN)
        out["config4"] = []
        for T in (1e-2, 1.0, 1e2):
            for nu in (1, 2):
                out["config4"].append(solve_case(2, 1 << 20, T, nu, "V"))
                out["config4"].append(solve_case(2, 1 << 20, T, nu, "V", coarsest=1024, coarse="scan"))
                out["config4"].append(solve_case(2, 1 << 20, T, nu, "W", coarsest=1024, coarse="scan",
                                                 reps=3))
                out["config4"].append(solve_case(2, 1 << 20, T, nu, "F"))
        out["config4_deepW"] = [solve_case(2, 1 << 14, 1.0, 1, "W", reps=2)]
        for r in out["config4"] + out["config4_deepW"]:
            print("config4", r, flush=True)
    out["config5"] = config5()
    for k, v in out["config5"].items():
        v["frac_of_peak"] = v["GBps"] / peak
        print("config5", k, v, flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
