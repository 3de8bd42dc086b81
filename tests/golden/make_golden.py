"""Generate golden vectors by running the REFERENCE itself (arxiv/paper_1409_5254,
``timemg`` at /root/reference/pkg/src).  Runs only in the build container
(the reference is not present on GPU boxes); the outputs are committed under
tests/golden/ and consumed by the CPU and GPU parity tests.

    python tests/golden/make_golden.py            # all cases (~3 min on 8 cores)
    python tests/golden/make_golden.py --quick    # skip the 2^20/2^22 solves

Inputs follow SURVEY.md §8(d): seeded problems from
paper_1409_5254_b200.problems (our input definition, not reference code),
zero initial guess unless stated, CycleConfig as listed per case.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import timemg  # noqa: E402  (the reference)
from timemg import multigrid as ref_mg  # noqa: E402
from paper_1409_5254_b200 import problems  # noqa: E402

WORKERS = os.cpu_count() or 1


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def omegas_of(hier, cfg):
    depth = ref_mg._depth(hier, cfg)
    return [float(w) for w in ref_mg._resolve_omegas(hier, cfg, depth)]


def assembly_cases(arrays, manifest):
    taus = [1e-8, 2.0**-26, 1e-6, 2.0**-20, 1e-3, 2.0**-10, 0.01, 0.1, 0.25, 0.5, 0.8,
            1.0, 3.0, 10.0, 1e3, 1e6]
    rows = []
    for rule in ("radau_lagrange", "scaled_legendre"):
        for p_t in range(6):
            basis = timemg.BasisSpec(p_t, rule)
            for ti, tau in enumerate(taus):
                key = f"asm_{rule[:5]}_p{p_t}_t{ti}"
                ops = timemg.assemble_local(basis, tau)
                r1, r2 = timemg.build_transfers(basis, tau)
                for name, val in (("K", ops.stiffness), ("M", ops.mass), ("C", ops.coupling),
                                  ("A", ops.minus_step_matrix), ("lu", ops.lu.lu),
                                  ("perm", ops.lu.perm), ("es", ops.eval_start),
                                  ("ee", ops.eval_end), ("r1", r1), ("r2", r2)):
                    arrays[f"{key}_{name}"] = np.asarray(val)
                a = timemg.alpha(basis, tau)
                rows.append({"key": key, "rule": rule, "p_t": p_t, "tau": tau, "alpha": a,
                             "omega": timemg.optimal_omega(a)})
    manifest["assembly"] = rows


def sweep_cases(arrays, manifest):
    cases = []
    spec = [(0, 1.0, 2, 1.0, 1, 0), (1, 0.2, 16, 0.8, 3, 1), (1, 3.0, 128, 1.0, 2, 2),
            (2, 0.5, 10, 0.9, 1, 3), (3, 1e-3, 257, 0.6, 2, 4), (3, 2.0**-26, 1000, None, 2, 5),
            (2, 1e2, 64, 1.3, 4, 6), (0, 1e-6, 96, None, 3, 7), (1, 0.01, 1, 0.5, 2, 8)]
    for i, (p_t, tau, n, omega, nu, seed) in enumerate(spec):
        basis = timemg.BasisSpec(p_t)
        ops = timemg.assemble_local(basis, tau)
        if omega is None:
            omega = timemg.optimal_omega(timemg.alpha(basis, tau))
        rng = np.random.default_rng(100 + seed)
        u = rng.standard_normal((n, p_t + 1))
        f = rng.standard_normal((n, p_t + 1))
        out = timemg.block_jacobi_sweep(ops, u, f, omega, nu)
        key = f"sweep{i}"
        arrays[f"{key}_u"], arrays[f"{key}_f"], arrays[f"{key}_out"] = u, f, out
        cases.append({"key": key, "p_t": p_t, "tau": tau, "n": n, "omega": omega, "nu": nu})
    # residual / restriction / prolongation primitives
    for i, (p_t, tau, n) in enumerate([(0, 0.3, 64), (1, 1e-4, 96), (2, 5.0, 32), (3, 2.0**-20, 256)]):
        basis = timemg.BasisSpec(p_t)
        ops = timemg.assemble_local(basis, tau)
        r1, r2 = timemg.build_transfers(basis, tau)
        rng = np.random.default_rng(200 + i)
        u = rng.standard_normal((n, p_t + 1))
        f = rng.standard_normal((n, p_t + 1))
        uc = rng.standard_normal((n // 2, p_t + 1))
        r = np.zeros_like(u)
        ref_mg._residual_slab(ops, f, u, r, 0, n)
        fc = np.zeros((n // 2, p_t + 1))
        ref_mg._restrict_slab(r1, r2, r, fc, 0, n // 2)
        up = u.copy()
        ref_mg._prolong_add_slab(r1, r2, uc, up, 0, n // 2)
        key = f"prim{i}"
        for nm, v in (("u", u), ("f", f), ("uc", uc), ("r", r), ("fc", fc), ("up", up)):
            arrays[f"{key}_{nm}"] = v
        cases.append({"key": key, "p_t": p_t, "tau": tau, "n": n, "kind": "primitives"})
    # forward substitution (the coarse solve, numpy matmul -> OpenBLAS dgemv)
    for i, (p_t, tau, n) in enumerate([(0, 0.5, 8), (1, 2.0**-9, 8), (2, 0.1, 16), (3, 1e-2, 15),
                                       (1, 1.0, 512), (3, 7.0, 2)]):
        ops = timemg.assemble_local(timemg.BasisSpec(p_t), tau)
        rng = np.random.default_rng(300 + i)
        rhs = rng.standard_normal((n, p_t + 1))
        out = np.empty_like(rhs)
        ref_mg._forward_substitute(ops, rhs, out)
        key = f"fsub{i}"
        arrays[f"{key}_rhs"], arrays[f"{key}_out"] = rhs, out
        cases.append({"key": key, "p_t": p_t, "tau": tau, "n": n, "kind": "forward_substitute"})
    manifest["sweeps"] = cases


def cycle_cases(arrays, manifest):
    cases = []
    spec = [
        # kind, p_t, tau, n, n_levels, coarsest, nu1, nu2, damping, level, seed
        ("v", 1, 0.5, 32, 2, 8, 2, 1, "optimal", 0, 5),
        ("two", 1, 0.5, 32, 2, 8, 2, 1, "optimal", 0, 5),
        ("two", 0, 0.8, 8, 2, 2, 1, 1, "optimal", 0, 7),
        ("two", 1, 0.8, 8, 2, 2, 1, 1, "optimal", 0, 7),
        ("v", 0, 1e-3, 64, 4, 8, 2, 2, "optimal", 0, 11),
        ("v", 2, 1e-2, 1024, "max", 2, 1, 1, "optimal", 0, 12),
        ("v", 3, 2.0**-10, 512, "max", 8, 2, 2, "optimal", 0, 13),
        ("v", 1, 1e-6, 4096, "max", 8, 2, 2, 0.7, 0, 14),
        ("v", 0, 1.0, 1000, "max", 2, 1, 1, "optimal", 0, 15),
        ("v", 2, 3.0, 96, "max", 2, 0, 1, "optimal", 0, 16),
        ("v", 1, 0.1, 96, "max", 2, 1, 0, "optimal", 0, 17),
        ("two", 2, 1e-4, 256, "max", 2, 1, 2, "optimal", 2, 18),
    ]
    for i, (kind, p_t, tau, n, nl, coarsest, nu1, nu2, damping, level, seed) in enumerate(spec):
        basis = timemg.BasisSpec(p_t)
        hier = timemg.TimeHierarchy.build(basis, tau, n, n_levels=nl, coarsest=coarsest)
        cfg = timemg.CycleConfig(nu1=nu1, nu2=nu2, damping=damping)
        rng = np.random.default_rng(seed)
        nn = hier.levels[level].n_steps
        u = rng.random((nn, p_t + 1))
        f = rng.random((nn, p_t + 1))
        if kind == "v":
            out = timemg.v_cycle(hier, u, f, cfg)
        else:
            out = timemg.two_grid_cycle(hier, level, u, f, cfg)
        key = f"cyc{i}"
        arrays[f"{key}_u"], arrays[f"{key}_f"], arrays[f"{key}_out"] = u, f, out
        cases.append({"key": key, "kind": kind, "p_t": p_t, "tau": tau, "n": n, "n_levels": nl,
                      "coarsest": coarsest, "nu1": nu1, "nu2": nu2, "damping": damping,
                      "level": level, "omegas": omegas_of(hier, cfg),
                      "sizes": [l.n_steps for l in hier.levels]})
    manifest["cycles"] = cases


def solve_record(hier, rhs, u_init, cfg):
    t0 = time.perf_counter()
    u, st = timemg.solve(hier, rhs, u_init, cfg)
    return u, st, time.perf_counter() - t0


def small_solve_cases(arrays, manifest):
    cases = []
    spec = [
        # name, p_t, n, T, coarsest, nu1, nu2, n_levels, damping, eps, max_iters, init, rule
        ("config1", 1, 1024, 1.0, 2, 1, 1, "max", "optimal", 1e-8, 250, "zero", "radau_lagrange"),
        ("p0_n256", 0, 256, 1.0, 2, 1, 1, "max", "optimal", 1e-8, 250, "zero", "radau_lagrange"),
        ("p2_n512_c8", 2, 512, 10.0, 8, 2, 2, "max", "optimal", 1e-10, 250, "zero", "radau_lagrange"),
        ("p3_n2048", 3, 2048, 0.01, 2, 1, 1, "max", "optimal", 1e-8, 250, "zero", "radau_lagrange"),
        ("p1_n1000", 1, 1000, 1.0, 2, 1, 1, "max", "optimal", 1e-8, 250, "zero", "radau_lagrange"),
        ("p1_lev3", 1, 512, 1.0, 2, 2, 1, 3, "optimal", 1e-8, 250, "zero", "radau_lagrange"),
        ("p2_fixed_w", 2, 256, 1.0, 2, 1, 1, "max", 0.8, 1e-8, 250, "zero", "radau_lagrange"),
        ("p1_maxit", 1, 1024, 1.0, 2, 1, 1, "max", "optimal", 1e-12, 3, "zero", "radau_lagrange"),
        ("p1_rand", 1, 4096, 1e-3, 8, 2, 2, "max", "optimal", 1e-8, 250, "random", "radau_lagrange"),
        ("legendre_p2", 2, 256, 1.0, 2, 1, 1, "max", "optimal", 1e-8, 250, "zero", "scaled_legendre"),
        ("p0_nu21", 0, 2048, 100.0, 2, 2, 1, "max", "optimal", 1e-9, 250, "zero", "radau_lagrange"),
    ]
    for name, p_t, n, T, coarsest, nu1, nu2, nl, damping, eps, mi, init, rule in spec:
        basis = timemg.BasisSpec(p_t, rule)
        a, phi, u0 = problems.forcing_params(42)
        tau = T / n
        rhs = timemg.rhs_moments(problems.make_forcing(a, phi, T), basis, tau, n, u0=u0)
        hier = timemg.TimeHierarchy.build(basis, tau, n, n_levels=nl, coarsest=coarsest)
        cfg = timemg.CycleConfig(nu1=nu1, nu2=nu2, damping=damping, levels=nl, eps=eps,
                                 max_iters=mi, workers=1)
        u_init = np.zeros_like(rhs) if init == "zero" else timemg.random_initial_guess(hier, 42)
        u, st, dt = solve_record(hier, rhs, u_init, cfg)
        arrays[f"solve_{name}_rhs"] = rhs
        arrays[f"solve_{name}_u"] = u
        cases.append({"name": name, "p_t": p_t, "n": n, "T": T, "coarsest": coarsest,
                      "nu1": nu1, "nu2": nu2, "n_levels": nl, "damping": damping, "eps": eps,
                      "max_iters": mi, "init": init, "rule": rule,
                      "iterations": st.iterations, "residual_norms": st.residual_norms,
                      "factor": st.factor, "converged": bool(st.converged),
                      "sha_rhs": sha(rhs), "sha_u": sha(u), "ref_seconds": dt,
                      "omegas": omegas_of(hier, cfg),
                      "sizes": [l.n_steps for l in hier.levels]})
    manifest["small_solves"] = cases


def factor_cases(manifest):
    cases = []
    for p_t, tau, nu in [(0, 1.0, 1), (1, 1e-2, 2), (3, 1e2, 1), (2, 1e-6, 1)]:
        hier = timemg.TimeHierarchy.build(timemg.BasisSpec(p_t), tau, 1024, n_levels=2)
        cfg = timemg.CycleConfig(nu1=nu, nu2=nu, eps=1e-100, seed=42, max_iters=150)
        got = timemg.measure_convergence_factor(hier, cfg)
        cases.append({"p_t": p_t, "tau": tau, "nu": nu, "factor": got,
                      "omegas": omegas_of(hier, timemg.CycleConfig())})
    manifest["factors"] = cases


def big_solve_cases(manifest, quick):
    cases = []
    # acceptance criterion 9 (tests/test_acceptance.py:179-192)
    basis = timemg.BasisSpec(1)
    n = 1 << 16
    hier = timemg.TimeHierarchy.build(basis, 1e-6, n)
    f = np.zeros((n, 2))
    u_init = timemg.random_initial_guess(hier, 42)
    u, st, dt = solve_record(hier, f, u_init, timemg.CycleConfig(eps=1e-8, seed=42,
                                                                 workers=WORKERS))
    cases.append({"name": "crit9", "p_t": 1, "n": n, "tau": 1e-6, "coarsest": 8, "nu1": 2,
                  "nu2": 2, "init": "random42", "f": "zero", "eps": 1e-8,
                  "iterations": st.iterations, "residual_norms": st.residual_norms,
                  "sha_u": sha(u), "ref_seconds": dt, "ref_workers": WORKERS})
    spec = []
    if not quick:
        for p_t in range(4):
            spec.append((f"config2_p{p_t}", p_t, 1 << 20, 1.0, 1, None))
        for T in (1e-2, 1.0, 1e2):
            for nu in (1, 2):
                spec.append((f"config4_T{T:g}_nu{nu}", 2, 1 << 20, T, nu, None))
        for b in (0, 1):
            spec.append((f"config3_b{b}", 1, 1 << 22, 1.0, 1, b))
    for name, p_t, n, T, nu, b in spec:
        rhs, tau, u0 = problems.seeded_rhs(p_t, n, T, 42, b)
        basis = timemg.BasisSpec(p_t)
        hier = timemg.TimeHierarchy.build(basis, tau, n, coarsest=2)
        cfg = timemg.CycleConfig(nu1=nu, nu2=nu, eps=1e-8, workers=WORKERS)
        u, st, dt = solve_record(hier, rhs, np.zeros_like(rhs), cfg)
        cases.append({"name": name, "p_t": p_t, "n": n, "T": T, "nu1": nu, "nu2": nu,
                      "coarsest": 2, "batch_index": b, "init": "zero", "eps": 1e-8,
                      "iterations": st.iterations, "residual_norms": st.residual_norms,
                      "sha_rhs": sha(rhs), "sha_u": sha(u), "ref_seconds": dt,
                      "ref_workers": WORKERS})
        print(f"  {name}: {st.iterations} iters, {dt:.2f} s", flush=True)
    manifest["big_solves"] = cases


def config5_case(arrays, manifest):
    n = 1 << 16
    p_t = 3
    tau = 2.0**-26
    basis = timemg.BasisSpec(p_t)
    ops = timemg.assemble_local(basis, tau)
    r1, r2 = timemg.build_transfers(basis, tau)
    omega = timemg.optimal_omega(timemg.alpha(basis, tau))
    u, f = problems.kernel_inputs(n, p_t + 1, 0)
    t0 = time.perf_counter()
    us = timemg.block_jacobi_sweep(ops, u, f, omega, 2)
    r = np.zeros_like(us)
    ref_mg._residual_slab(ops, f, us, r, 0, n)
    fc = np.zeros((n // 2, p_t + 1))
    ref_mg._restrict_slab(r1, r2, r, fc, 0, n // 2)
    dt = time.perf_counter() - t0
    arrays["config5_u_head"] = us[:512]
    arrays["config5_fc_head"] = fc[:256]
    manifest["config5"] = {"n": n, "p_t": p_t, "tau": tau, "omega": omega, "nu": 2,
                           "sha_u_in": sha(u), "sha_f_in": sha(f), "sha_u": sha(us),
                           "sha_fc": sha(fc), "ref_seconds": dt}


def dgemv_calibration(arrays, manifest):
    rng = np.random.default_rng(77)
    for nt in range(1, 5):
        c = rng.standard_normal((nt, nt))
        x = rng.standard_normal((512, nt))
        y = np.stack([c @ x[k] for k in range(512)])
        arrays[f"dgemv{nt}_c"], arrays[f"dgemv{nt}_x"], arrays[f"dgemv{nt}_y"] = c, x, y
    cfg = np.__config__.get_info("blas_opt") if hasattr(np.__config__, "get_info") else None
    manifest["dgemv"] = {"numpy": np.__version__, "blas": str(cfg)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    arrays, manifest = {}, {"reference": "/root/reference/pkg/src/timemg",
                            "numpy": np.__version__, "host_cpus": WORKERS}
    for step in (assembly_cases, sweep_cases, cycle_cases, small_solve_cases, config5_case,
                 dgemv_calibration):
        t0 = time.perf_counter()
        step(arrays, manifest)
        print(f"{step.__name__}: {time.perf_counter() - t0:.1f} s", flush=True)
    t0 = time.perf_counter()
    factor_cases(manifest)
    print(f"factor_cases: {time.perf_counter() - t0:.1f} s", flush=True)
    big_solve_cases(manifest, args.quick)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
    print("wrote", os.path.join(HERE, "golden.npz"), os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
