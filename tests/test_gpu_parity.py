"""GPU parity: the sm_100a kernels (through the C ABI) against the reference's
golden vectors and the pinned CPU oracle.  fp64 comparisons are bitwise
(``tobytes``); iteration counts and residual-norm histories must be equal.
The fp32 path is checked normwise (tolerance 1e-5, BASELINE config 5).
"""

import ctypes
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1409_5254_b200 as tmg  # noqa: E402
from paper_1409_5254_b200 import _native as nat  # noqa: E402
from paper_1409_5254_b200 import problems, solver  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    nat.check(nat.load().tmg_device_check(0))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def same_bits(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def omegas(hier, damping="optimal"):
    return [tmg.resolve_damping(damping, tmg.alpha(hier.basis, l.tau)) for l in hier.levels]


def hier_of(c):
    tau = c["tau"] if "tau" in c else c["T"] / c["n"]
    return tmg.TimeHierarchy.build(tmg.BasisSpec(c["p_t"], c.get("rule", "radau_lagrange")), tau,
                                   c["n"], n_levels=c.get("n_levels", "max"),
                                   coarsest=c.get("coarsest", 8))


def dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def P(t):
    return ctypes.c_void_p(t.data_ptr())


# --------------------------------------------------------------------------- slab kernels

def test_block_jacobi_sweep_golden(golden):
    man, arr = golden
    for c in man["sweeps"]:
        if c.get("kind"):
            continue
        k = c["key"]
        ops = tmg.assemble_local(tmg.BasisSpec(c["p_t"]), c["tau"])
        out = tmg.block_jacobi_sweep(ops, arr[f"{k}_u"], arr[f"{k}_f"], c["omega"], c["nu"])
        assert same_bits(out, arr[f"{k}_out"]), k


def test_primitives_golden(golden):
    """residual, restriction (tmg_down nu1=0) and prolongation (tmg_up nu2=0)."""
    import torch
    man, arr = golden
    L = nat.load()
    for c in man["sweeps"]:
        if c.get("kind") != "primitives":
            continue
        k, n = c["key"], c["n"]
        basis = tmg.BasisSpec(c["p_t"])
        ops = tmg.assemble_local(basis, c["tau"])
        r1, r2 = tmg.build_transfers(basis, c["tau"])
        d = nat.level_desc(ops, n, 1.0, r1, r2)
        u, f, uc = dev(arr[f"{k}_u"]), dev(arr[f"{k}_f"]), dev(arr[f"{k}_uc"])
        r = torch.empty_like(u)
        nat.check(L.tmg_residual(0, ctypes.byref(d), P(f), P(u), P(r), 1, None))
        uo = torch.empty_like(u)
        fc = torch.empty((n // 2, c["p_t"] + 1), dtype=torch.float64, device="cuda")
        nat.check(L.tmg_down(0, ctypes.byref(d), P(f), P(u), P(uo), P(fc), 1, 0, None, None))
        up = torch.empty_like(u)
        nat.check(L.tmg_up(0, ctypes.byref(d), P(f), P(u), P(uc), P(up), None, 1, 0, None, None))
        torch.cuda.synchronize()
        assert same_bits(r.cpu().numpy(), arr[f"{k}_r"]), k
        assert same_bits(fc.cpu().numpy(), arr[f"{k}_fc"]), k
        assert same_bits(up.cpu().numpy(), arr[f"{k}_up"]), k
        assert same_bits(uo.cpu().numpy(), arr[f"{k}_u"]), k


def test_forward_substitute_golden(golden):
    import torch
    man, arr = golden
    L = nat.load()
    for c in man["sweeps"]:
        if c.get("kind") != "forward_substitute":
            continue
        k = c["key"]
        ops = tmg.assemble_local(tmg.BasisSpec(c["p_t"]), c["tau"])
        d = nat.level_desc(ops, c["n"])
        rhs = dev(arr[f"{k}_rhs"])
        out = torch.empty_like(rhs)
        nat.check(L.tmg_coarse_solve(0, ctypes.byref(d), P(rhs), P(out), 1, 0, 0, None))
        assert same_bits(out.cpu().numpy(), arr[f"{k}_out"]), k


def test_resid_norm_matches_numpy_order(oracle_mod):
    import torch
    L = nat.load()
    for n, p_t in [(1024, 1), (1000, 2), (1 << 16, 3), (96 * 64, 0), (12345, 1)]:
        ops = tmg.assemble_local(tmg.BasisSpec(p_t), 1e-3)
        rng = np.random.default_rng(n)
        u = rng.standard_normal((n, p_t + 1))
        f = rng.standard_normal((n, p_t + 1))
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        d = nat.level_desc(ops, n)
        fd, ud = dev(f), dev(u)  # keep both alive across the call
        nat.check(L.tmg_resid_norm(0, ctypes.byref(d), P(fd), P(ud), P(out), 1, None))
        r = oracle_mod.residual(ops, f, u)
        acc = r[:, 0] * r[:, 0]
        for j in range(1, p_t + 1):
            acc = acc + r[:, j] * r[:, j]
        want = float(np.sqrt(np.sum(acc)))
        assert float(out.item()) == want, (n, p_t)


# --------------------------------------------------------------------------- cycles

def test_cycles_golden(golden):
    man, arr = golden
    for c in man["cycles"]:
        k = c["key"]
        hier = hier_of(c)
        cfg = tmg.CycleConfig(nu1=c["nu1"], nu2=c["nu2"], damping=c["damping"])
        if c["kind"] == "v":
            out = tmg.v_cycle(hier, arr[f"{k}_u"], arr[f"{k}_f"], cfg)
        else:
            out = tmg.two_grid_cycle(hier, c["level"], arr[f"{k}_u"], arr[f"{k}_f"], cfg)
        assert same_bits(out, arr[f"{k}_out"]), k


def test_small_solves_golden(golden):
    man, arr = golden
    for c in man["small_solves"]:
        name = c["name"]
        hier = hier_of(c)
        cfg = tmg.CycleConfig(nu1=c["nu1"], nu2=c["nu2"], damping=c["damping"], levels=c["n_levels"],
                              eps=c["eps"], max_iters=c["max_iters"])
        rhs = arr[f"solve_{name}_rhs"]
        u0 = np.zeros_like(rhs) if c["init"] == "zero" else tmg.random_initial_guess(hier, 42)
        u, st = tmg.solve(hier, rhs, u0, cfg)
        assert st.iterations == c["iterations"], name
        assert st.residual_norms == c["residual_norms"], name
        assert st.converged == c["converged"], name
        assert same_bits(u, arr[f"solve_{name}_u"]), name


def test_acceptance_criterion9_digest(golden):
    man, _ = golden
    c = next(x for x in man["big_solves"] if x["name"] == "crit9")
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), 1e-6, c["n"])
    f = np.zeros((c["n"], 2))
    u, st = tmg.solve(hier, f, tmg.random_initial_guess(hier, 42), tmg.CycleConfig(eps=1e-8))
    assert st.iterations == 9
    assert st.residual_norms == c["residual_norms"]
    assert sha(u) == c["sha_u"]


@pytest.mark.parametrize("name", ["config2_p0", "config2_p1", "config2_p2", "config2_p3",
                                  "config4_T0.01_nu1", "config4_T0.01_nu2", "config4_T1_nu2",
                                  "config4_T100_nu1", "config4_T100_nu2"])
def test_big_solves_golden(golden, name):
    man, _ = golden
    c = next(x for x in man["big_solves"] if x["name"] == name)
    rhs, tau, _ = problems.seeded_rhs(c["p_t"], c["n"], c["T"], 42, c["batch_index"])
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(c["p_t"]), tau, c["n"], coarsest=2)
    cfg = tmg.CycleConfig(nu1=c["nu1"], nu2=c["nu2"], eps=1e-8)
    u, st = tmg.solve(hier, rhs, np.zeros_like(rhs), cfg)
    assert st.iterations == c["iterations"], name
    assert st.residual_norms == c["residual_norms"], name
    assert sha(u) == c["sha_u"], name


def test_config3_batched_golden(golden):
    """B problems in one batched solve equal the reference's separate solves."""
    man, _ = golden
    cases = [x for x in man["big_solves"] if x["name"].startswith("config3_b")]
    n = cases[0]["n"]
    rhs = [problems.seeded_rhs(1, n, 1.0, 42, c["batch_index"])[0] for c in cases]
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), 1.0 / n, n, coarsest=2)
    cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8)
    U, stats = tmg.solve_batched(hier, np.stack(rhs), None, cfg)
    for b, c in enumerate(cases):
        assert stats[b].iterations == c["iterations"]
        assert stats[b].residual_norms == c["residual_norms"]
        assert sha(U[b]) == c["sha_u"], c["name"]


def test_config5_prefix_fp64(golden):
    """fused down pass (2 sweeps + residual + restriction) on the 2^16 prefix."""
    import torch
    man, arr = golden
    c = man["config5"]
    basis = tmg.BasisSpec(c["p_t"])
    ops = tmg.assemble_local(basis, c["tau"])
    r1, r2 = tmg.build_transfers(basis, c["tau"])
    u, f = problems.kernel_inputs(c["n"], c["p_t"] + 1, 0)
    d = nat.level_desc(ops, c["n"], c["omega"], r1, r2)
    ud, fd = dev(u), dev(f)
    uo = torch.empty_like(ud)
    fc = torch.empty((c["n"] // 2, 4), dtype=torch.float64, device="cuda")
    nat.check(nat.load().tmg_down(0, ctypes.byref(d), P(fd), P(ud), P(uo), P(fc), 1, 2, None, None))
    torch.cuda.synchronize()
    assert sha(uo.cpu().numpy()) == c["sha_u"]
    assert sha(fc.cpu().numpy()) == c["sha_fc"]


def test_config5_fp32_normwise(golden):
    import torch
    man, arr = golden
    c = man["config5"]
    basis = tmg.BasisSpec(c["p_t"])
    ops = tmg.assemble_local(basis, c["tau"])
    r1, r2 = tmg.build_transfers(basis, c["tau"])
    u, f = problems.kernel_inputs(c["n"], c["p_t"] + 1, 0)
    d = nat.level_desc(ops, c["n"], c["omega"], r1, r2)
    ud = torch.from_numpy(u).float().cuda()
    fd = torch.from_numpy(f).float().cuda()
    uo = torch.empty_like(ud)
    fc = torch.empty((c["n"] // 2, 4), dtype=torch.float32, device="cuda")
    nat.check(nat.load().tmg_down(1, ctypes.byref(d), P(fd), P(ud), P(uo), P(fc), 1, 2, None, None))
    torch.cuda.synchronize()
    want_u = arr["config5_u_head"]
    want_fc = arr["config5_fc_head"]
    got_u = uo.double().cpu().numpy()[:512]
    got_fc = fc.double().cpu().numpy()[:256]
    assert np.linalg.norm(got_u - want_u) <= 1e-5 * np.linalg.norm(want_u)
    assert np.linalg.norm(got_fc - want_fc) <= 1e-5 * np.linalg.norm(want_fc)


# --------------------------------------------------------------------------- vs oracle

@pytest.mark.parametrize("p_t,n,rule,nu", [(1, 100000, "radau_lagrange", 1),
                                           (2, 1 << 14, "scaled_legendre", 2),
                                           (3, 96 * 256, "radau_lagrange", 1),
                                           (0, 3 * (1 << 15), "radau_lagrange", 3)])
def test_streaming_odd_sizes_vs_oracle(oracle_mod, p_t, n, rule, nu):
    T = 1.0
    a, phi, u0 = problems.forcing_params(7)
    basis = tmg.BasisSpec(p_t, rule)
    rhs = tmg.rhs_moments(problems.make_forcing(a, phi, T), basis, T / n, n, u0=u0)
    hier = tmg.TimeHierarchy.build(basis, T / n, n, coarsest=2)
    cfg = tmg.CycleConfig(nu1=nu, nu2=nu, eps=1e-9)
    u, st = tmg.solve(hier, rhs, np.zeros_like(rhs), cfg)
    ur, norms, iters = oracle_mod.iterate(hier, omegas(hier), rhs, np.zeros_like(rhs), nu, nu,
                                          1e-9, 250)
    assert st.iterations == iters
    assert st.residual_norms == norms
    assert same_bits(u, ur)


@pytest.mark.parametrize("cycle", ["W", "F"])
@pytest.mark.parametrize("n,p_t,nu", [(1024, 1, 1), (1 << 17, 2, 1), (1 << 15, 1, 2), (1 << 16, 3, 1)])
def test_w_f_cycle_vs_oracle(oracle_mod, n, p_t, nu, cycle):
    """W- and F-cycle solves (whole problem in the tail, and streamed levels
    above it) bitwise against the oracle's tmo_cycle_rec compositions"""
    rhs, tau, _ = problems.seeded_rhs(p_t, n, 1.0, 42)
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(p_t), tau, n, coarsest=2)
    cfg = tmg.CycleConfig(nu1=nu, nu2=nu, eps=1e-8, cycle=cycle)
    u, st = tmg.solve(hier, rhs, np.zeros_like(rhs), cfg)
    ur, norms, iters = oracle_mod.iterate(hier, omegas(hier), rhs, np.zeros_like(rhs), nu, nu,
                                          1e-8, 250, gamma=tmg.hierarchy.CYCLE_KIND[cycle])
    assert st.iterations == iters
    assert st.residual_norms == norms
    assert same_bits(u, ur)


@pytest.mark.parametrize("n,p_t", [(512, 1), (1 << 14, 2)])
def test_f_cycle_single_cycles(oracle_mod, n, p_t):
    """v_cycle(config.cycle="F") from a random iterate: one F-cycle, then a
    second on its output, bitwise against the oracle's cycle"""
    rhs, tau, _ = problems.seeded_rhs(p_t, n, 1.0, 42)
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(p_t), tau, n, coarsest=2)
    cfg = tmg.CycleConfig(nu1=1, nu2=1, cycle="F")
    u = tmg.random_initial_guess(hier, 5)
    for _ in range(2):
        out = tmg.v_cycle(hier, u, rhs, cfg)
        ref = oracle_mod.cycle(hier, omegas(hier), u, rhs, 1, 1, gamma=3)
        assert same_bits(out, ref)
        u = out


def test_batched_independent_stopping(oracle_mod):
    """problems that converge at different iteration counts in one batch"""
    n = 1 << 15
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), 1.0 / n, n, coarsest=2)
    F = np.stack([problems.seeded_rhs(1, n, 1.0, 42, b)[0] * (10.0 ** b) for b in range(3)])
    F[2] = 0.0  # zero rhs with random start: a different history
    U0 = np.zeros_like(F)
    U0[2] = tmg.random_initial_guess(hier, 3)
    cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-10)
    U, stats = tmg.solve_batched(hier, F, U0, cfg)
    om = omegas(hier)
    for b in range(3):
        ur, norms, iters = oracle_mod.iterate(hier, om, F[b], U0[b], 1, 1, 1e-10, 250)
        assert stats[b].iterations == iters, b
        assert stats[b].residual_norms == norms, b
        assert same_bits(U[b], ur), b


def test_tail_split_invariance():
    """the level where the single-CTA engine takes over does not change bits"""
    rhs, tau, _ = problems.seeded_rhs(2, 1 << 13, 1.0, 42)
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(2), tau, 1 << 13, coarsest=2)
    cfg = tmg.CycleConfig(nu1=1, nu2=2, eps=1e-8)
    outs = []
    for tail_max in (2, 64, 1024):
        solver.TAIL_MAX = tail_max
        try:
            u, st = tmg.solve(hier, rhs, np.zeros_like(rhs), cfg)
        finally:
            solver.TAIL_MAX = 0
        hier.__dict__.pop("_tmg_plans", None)
        outs.append((u.tobytes(), tuple(st.residual_norms)))
    assert len(set(outs)) == 1


def test_reference_semantics():
    ops = tmg.assemble_local(tmg.BasisSpec(0), 1.0)
    out = tmg.block_jacobi_sweep(ops, np.ones((2, 1)), np.zeros((2, 1)), omega=1.0)
    assert np.allclose(out.ravel(), [0.0, 0.5], atol=1e-15)
    ops = tmg.assemble_local(tmg.BasisSpec(1), 3.0)
    u = np.random.default_rng(0).random((128, 2))
    out = tmg.block_jacobi_sweep(ops, u, np.zeros_like(u), omega=1.0, nu=2)
    assert np.linalg.norm(out) <= 1e-12 * np.linalg.norm(u)
    with pytest.raises(ValueError):
        tmg.block_jacobi_sweep(ops, u, u, omega=2.5)
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(0), 1.0, 16, n_levels=2)
    z = tmg.two_grid_cycle(hier, 0, np.zeros((16, 1)), np.zeros((16, 1)))
    assert np.max(np.abs(z)) == 0.0
    with pytest.raises(ValueError):
        tmg.two_grid_cycle(hier, 1, np.zeros((8, 1)), np.zeros((8, 1)))
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(0), 1e-4, 64)
    _, st = tmg.solve(hier, np.zeros((64, 1)), config=tmg.CycleConfig(eps=1e-12, max_iters=2, seed=0))
    assert not st.converged and st.iterations == 2


def test_measure_convergence_factor_golden(golden):
    man, _ = golden
    for c in man["factors"]:
        hier = tmg.TimeHierarchy.build(tmg.BasisSpec(c["p_t"]), c["tau"], 1024, n_levels=2)
        cfg = tmg.CycleConfig(nu1=c["nu"], nu2=c["nu"], eps=1e-100, seed=42, max_iters=150)
        got = tmg.measure_convergence_factor(hier, cfg)
        assert got == c["factor"], c


def test_device_resident_torch_api():
    import torch
    rhs, tau, _ = problems.seeded_rhs(1, 1 << 14, 1.0, 42)
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), tau, 1 << 14, coarsest=2)
    cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8)
    u_np, st_np = tmg.solve(hier, rhs, np.zeros_like(rhs), cfg)
    f_t = torch.from_numpy(rhs).cuda()
    u_t, st_t = tmg.solve(hier, f_t, torch.zeros_like(f_t), cfg)
    assert torch.is_tensor(u_t) and u_t.is_cuda
    assert u_t.cpu().numpy().tobytes() == u_np.tobytes()
    assert st_t.residual_norms == st_np.residual_norms


def test_batched_host_pipeline_vs_oracle(oracle_mod):
    """B >= 8 host buffers go through the sub-batch pipeline (two streams)."""
    n = 1 << 13
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), 1.0 / n, n, coarsest=2)
    F = np.stack([problems.seeded_rhs(1, n, 1.0, 42, b)[0] for b in range(8)])
    cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8)
    om = omegas(hier)
    for U0 in (None, np.stack([tmg.random_initial_guess(hier, b) for b in range(8)])):
        U, stats = tmg.solve_batched(hier, F, U0, cfg)
        for b in range(8):
            u0 = np.zeros_like(F[b]) if U0 is None else U0[b]
            ur, norms, iters = oracle_mod.iterate(hier, om, F[b], u0, 1, 1, 1e-8, 250)
            assert stats[b].iterations == iters, b
            assert stats[b].residual_norms == norms, b
            assert same_bits(U[b], ur), b


@pytest.mark.parametrize("p_t,tau,n", [(1, 1e-6, 1 << 20), (2, 0.5, 4097), (3, 1e3, 1000),
                                       (0, 2.0 ** -10, 65536), (1, 2.0 ** -24, 1 << 24),
                                       (3, 1e-3, 3 * 100003), (2, 1.0, 1)])
def test_scan_forward_solve_vs_oracle(oracle_mod, p_t, tau, n):
    """grid-wide look-back scan solve: within 1e-12 relative of the exact
    (long-double) solution of the same system, and within 1e-12 of the
    reference-order forward substitution beyond that order's own error.  For
    small steps (alpha -> 1) the serial sweep itself drifts from the exact
    solution by ~sqrt(N) ulp (2.7e-12 relative at 2^20, 4.4e-11 at 2^24): the
    scan is compared with both, batched problems too."""
    ops = tmg.assemble_local(tmg.BasisSpec(p_t), tau)
    rhs = np.random.default_rng(n).standard_normal((n, p_t + 1))
    want = oracle_mod.forward_substitute(ops, rhs)
    exact = oracle_mod.forward_solve_extended(ops, rhs)
    got = tmg.forward_solve(tmg.GlobalSystem(ops, n), rhs, method="scan")
    nrm = np.linalg.norm(exact)
    assert np.linalg.norm(got - exact) <= 1e-12 * nrm
    assert np.linalg.norm(got - want) <= np.linalg.norm(want - exact) + 1e-12 * nrm
    if n <= 1 << 20:
        rhs3 = np.stack([rhs, 2.0 * rhs, -rhs])
        got3 = tmg.forward_solve(tmg.GlobalSystem(ops, n), rhs3, method="scan")
        for b, k in enumerate((1.0, 2.0, -1.0)):
            assert np.linalg.norm(got3[b] - k * exact) <= 1e-12 * abs(k) * nrm
    exact = tmg.forward_solve(tmg.GlobalSystem(ops, min(n, 4096)), rhs[:4096], method="serial")
    assert same_bits(exact, oracle_mod.forward_substitute(ops, rhs[:4096]))


def test_w_cycle_large_coarsest_scan(oracle_mod):
    """W-cycle with a 1024-slab coarsest level solved by the scan: iterates
    within 1e-12 of the oracle (which uses forward substitution)."""
    n = 1 << 16
    rhs, tau, _ = problems.seeded_rhs(2, n, 1.0, 42)
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(2), tau, n, coarsest=1024)
    cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8, cycle="W", coarse="scan")
    u, st = tmg.solve(hier, rhs, np.zeros_like(rhs), cfg)
    ur, norms, iters = oracle_mod.iterate(hier, omegas(hier), rhs, np.zeros_like(rhs), 1, 1, 1e-8,
                                          250, gamma=2)
    assert st.iterations == iters
    assert np.linalg.norm(u - ur) <= 1e-12 * np.linalg.norm(ur)
    assert np.allclose(st.residual_norms, norms, rtol=1e-9, atol=0)


def test_measure_convergence_factors_batched(golden):
    """many step sizes in one launch (one operator per problem) == one
    measure_convergence_factor call per step size, bit for bit"""
    man, _ = golden
    for c in man["factors"]:
        basis = tmg.BasisSpec(c["p_t"])
        taus = [c["tau"], 1e-3, 1.0, 1e3]
        got = tmg.measure_convergence_factors(basis, taus, nu=c["nu"], max_iters=150)
        assert got[0] == c["factor"], c
        for t, g in zip(taus[1:], got[1:]):
            hier = tmg.TimeHierarchy.build(basis, t, 1024, n_levels=2)
            one = tmg.measure_convergence_factor(
                hier, tmg.CycleConfig(nu1=c["nu"], nu2=c["nu"], eps=1e-100, seed=42, max_iters=150))
            assert g == one, (c, t)


def test_rhs_moments_device_close_to_host():
    """torch-evaluated forcing + the tmg_rhs_samples kernel vs the host quadrature."""
    import torch
    a, phi, u0 = problems.forcing_params(42)
    for p_t in range(4):
        basis = tmg.BasisSpec(p_t)
        n, T = 4096, 1.0
        host = tmg.rhs_moments(problems.make_forcing(a, phi, T), basis, T / n, n, u0=u0)

        def f(t):
            v = torch.zeros_like(t)
            for k in range(8):
                v += a[k] * torch.sin(2.0 * np.pi * (k + 1) * t / T + phi[k])
            return v

        dev = tmg.rhs_moments_device(f, basis, T / n, n, u0=u0).cpu().numpy()
        assert np.max(np.abs(dev - host)) <= 1e-14 * np.max(np.abs(host))


@pytest.mark.gpu
def test_solve_bitwise_repeatable():
    """Repeated batched solves from the same iterate are bit-identical (guards
    the shared-memory ring's reuse ordering: generic reads of a stage before
    the bulk copy that refills it)."""
    import torch
    n, B = 1 << 22, 2
    F = problems.seeded_rhs_batch_device(1, n, 1.0, 42, list(range(B)))
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), 1.0 / n, n, coarsest=2)
    cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8)
    U0 = torch.randn(F.shape, generator=torch.Generator(device="cuda").manual_seed(1), device="cuda",
                     dtype=torch.float64)
    ref = None
    for _ in range(4):
        U = U0.clone()
        _, st = tmg.solve_batched(hier, F, U, cfg, inplace=True)
        out = (U, [s.residual_norms for s in st])
        if ref is None:
            ref = out
        else:
            assert torch.equal(out[0], ref[0])
            assert out[1] == ref[1]


# the fused finest pass (level-1 up + finest up + next finest down), the coarse
# up/down pairs and their warm-up rows, for every sweep count and a batch
@pytest.mark.parametrize("p_t,n,nu,B", [(1, 1 << 15, 2, 1), (1, 1 << 15, 3, 2), (0, 1 << 16, 4, 1),
                                        (1, 3 << 13, 1, 2)])
def test_fused_passes_vs_oracle(oracle_mod, p_t, n, nu, B):
    T = 1.0
    basis = tmg.BasisSpec(p_t)
    hier = tmg.TimeHierarchy.build(basis, T / n, n, coarsest=2)
    cfg = tmg.CycleConfig(nu1=nu, nu2=nu, eps=1e-9)
    F = []
    for b in range(B):
        a, phi, u0 = problems.forcing_params(11 + b)
        F.append(tmg.rhs_moments(problems.make_forcing(a, phi, T), basis, T / n, n, u0=u0))
    F = np.stack(F)
    import torch
    floors = [1e-12 * float(np.linalg.norm(F[b])) for b in range(B)]
    U, stats = tmg.solve_batched(hier, torch.from_numpy(F).cuda(), None, cfg, floors=floors)
    U = U.cpu().numpy()
    for b in range(B):
        ur, norms, iters = oracle_mod.iterate(hier, omegas(hier), F[b], np.zeros_like(F[b]), nu, nu,
                                              1e-9, 250)
        assert stats[b].iterations == iters
        assert stats[b].residual_norms == norms
        assert same_bits(U[b], ur)


# fp32 plans (the throughput variant: FMA + precomputed damped inverse) through
# the same fused passes: converge to the fp64 solution within fp32 accuracy
@pytest.mark.parametrize("p_t", [1, 2])
def test_fp32_plan_solve_close_to_fp64(p_t):
    import torch
    n = 1 << 16
    rhs, tau, _ = problems.seeded_rhs(p_t, n, 1.0, 42)
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(p_t), tau, n, coarsest=2)
    # fp32 residuals bottom out near 1e-5 relative at this size: stop at 1e-4
    cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-4)
    u64, st64 = tmg.solve(hier, rhs, np.zeros_like(rhs), cfg)
    depth = len(hier.levels)
    plan = solver.get_plan(hier, 0, depth, solver.omegas_for(hier, cfg, depth), cfg, 1, nat.F32)
    F = torch.from_numpy(rhs).float().cuda()[None]
    U = torch.zeros_like(F)
    it, norms, conv = plan.solve(F, U, [1e-12 * float(np.linalg.norm(rhs))], cfg.eps, cfg.max_iters)
    u32 = U[0].double().cpu().numpy()
    assert conv[0] and abs(int(it[0]) - st64.iterations) <= 1
    # same iterates up to fp32 rounding: the first residual norms agree to 1e-4;
    # the final solutions differ by at most the algebraic error at eps = 1e-4
    # (the two may stop one cycle apart)
    assert np.allclose(norms[0][:3], st64.residual_norms[:3], rtol=1e-4)
    assert np.linalg.norm(u32 - u64) <= 1e-3 * np.linalg.norm(u64)
