"""GPU parity at the measured sizes and on the edge cases of the drop-in API.

* BASELINE config 5 at its full size (N = 2^26, p_t = 3, nu1 = 2): the
  reference's own config-5 inputs on the first 2^16 slabs must hash to the
  reference's outputs (tests/golden, make_golden.py:config5_case), and the
  whole 2^26-slab pass must equal the oracle bit for bit (fp64) / within 1e-5
  normwise (fp32).
* Signed zeros of the sparse coupling (multigrid.py:158-165 adds the exact
  products 0 * u_prev of rows >= 1): right-hand sides with -0 entries take the
  kernels' exact sign-tracking path; everything stays bitwise.
* The host-BLAS tree of the coarse solve measured on THIS host (blas_tree.py)
  reproduces numpy's own `coupling @ x` inside the reference's forward
  substitution (dg.py:290-303), restated here with numpy.
* Input validation (solve / solve_batched broadcast like the reference's
  assignments, ValueError otherwise) and the host-buffer pipeline's sub-plan
  reuse (B = 32).
"""

import ctypes
import hashlib
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1409_5254_b200 as tmg  # noqa: E402
from paper_1409_5254_b200 import _native as nat  # noqa: E402
from paper_1409_5254_b200 import blas_tree, problems  # noqa: E402


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


def P(t):
    return ctypes.c_void_p(t.data_ptr())


def omegas(hier):
    return [tmg.optimal_omega(tmg.alpha(hier.basis, lev.tau)) for lev in hier.levels]


# --------------------------------------------------------------------------- config 5, full size

def test_config5_full_size(golden, oracle_mod):
    import torch
    man, _ = golden
    c = man["config5"]
    n, nt = 1 << 26, 4
    tau = 2.0 ** -26
    assert c["tau"] == tau and c["p_t"] == 3 and c["nu"] == 2
    basis = tmg.BasisSpec(3)
    ops = tmg.assemble_local(basis, tau)
    r1, r2 = tmg.build_transfers(basis, tau)
    om = tmg.optimal_omega(tmg.alpha(basis, tau))
    assert om == c["omega"]
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    u = torch.randn((n, nt), generator=gen, device="cuda", dtype=torch.float64)
    f = torch.randn((n, nt), generator=gen, device="cuda", dtype=torch.float64)
    up, fp = problems.kernel_inputs(c["n"], nt, 0)
    assert sha(up) == c["sha_u_in"] and sha(fp) == c["sha_f_in"]
    u[:c["n"]].copy_(torch.from_numpy(up))
    f[:c["n"]].copy_(torch.from_numpy(fp))
    d = nat.level_desc(ops, n, om, r1, r2)
    uo = torch.empty_like(u)
    fc = torch.empty((n // 2, nt), dtype=torch.float64, device="cuda")
    nat.check(nat.load().tmg_down(nat.F64, ctypes.byref(d), P(f), P(u), P(uo), P(fc), 1, 2, None, None))
    torch.cuda.synchronize()
    uo_h, fc_h = uo.cpu().numpy(), fc.cpu().numpy()
    # the reference's own outputs on the 2^16-slab prefix
    assert sha(uo_h[:c["n"]]) == c["sha_u"]
    assert sha(fc_h[:c["n"] // 2]) == c["sha_fc"]
    # the whole pass against the oracle
    uh, fh = u.cpu().numpy(), f.cpu().numpy()
    ur, fcr = oracle_mod.down_pass(ops, r1, r2, om, uh, fh, nu=2)
    assert same_bits(uo_h, ur)
    assert same_bits(fc_h, fcr)
    # fp32 variant: normwise 1e-5 against the fp64 result (BASELINE config 5)
    u32, f32 = u.float(), f.float()
    uo32 = torch.empty_like(u32)
    fc32 = torch.empty((n // 2, nt), dtype=torch.float32, device="cuda")
    nat.check(nat.load().tmg_down(nat.F32, ctypes.byref(d), P(f32), P(u32), P(uo32), P(fc32), 1, 2,
                                  None, None))
    torch.cuda.synchronize()
    eu = float(torch.linalg.norm(uo32.double() - uo) / torch.linalg.norm(uo))
    ef = float(torch.linalg.norm(fc32.double() - fc) / torch.linalg.norm(fc))
    assert eu <= 1e-5 and ef <= 1e-5, (eu, ef)


# --------------------------------------------------------------------------- signed zeros

def _neg_zero_inputs(n, nt, seed):
    rng = np.random.default_rng(seed)
    f = rng.standard_normal((n, nt))
    u = rng.standard_normal((n, nt))
    # -0 in rows >= 1 of f at random slabs, and at every row start / chunk
    # edge pattern (slab % 64 in {0, 63}); zero slabs of u with random signs
    pick = rng.random(n) < 0.05
    pick[::64] = True
    pick[63::64] = True
    for i in range(1, nt):
        f[pick, i] = -0.0
    z = rng.random(n) < 0.2
    u[z] = np.where(rng.random((int(z.sum()), nt)) < 0.5, -0.0, 0.0)
    return u, f


@pytest.mark.parametrize("p_t,n,nu", [(1, 1 << 14, 1), (1, 3 * 4096 + 64, 2), (2, 1 << 13, 2),
                                      (3, 5000, 1)])
def test_signed_zero_down_pass(oracle_mod, p_t, n, nu):
    import torch
    nt = p_t + 1
    tau = 1.0 / n
    basis = tmg.BasisSpec(p_t)
    ops = tmg.assemble_local(basis, tau)
    r1, r2 = tmg.build_transfers(basis, tau)
    om = tmg.optimal_omega(tmg.alpha(basis, tau))
    u, f = _neg_zero_inputs(n, nt, n + p_t)
    d = nat.level_desc(ops, n, om, r1, r2)
    ud, fd = torch.from_numpy(u).cuda(), torch.from_numpy(f).cuda()
    uo = torch.empty_like(ud)
    fc = torch.empty((n // 2, nt), dtype=torch.float64, device="cuda")
    nat.check(nat.load().tmg_down(nat.F64, ctypes.byref(d), P(fd), P(ud), P(uo), P(fc), 1, nu, None, None))
    torch.cuda.synchronize()
    ur, fcr = oracle_mod.down_pass(ops, r1, r2, om, u, f, nu=nu)
    got = uo.cpu().numpy()
    assert same_bits(got, ur)
    assert np.array_equal(np.signbit(got), np.signbit(ur))
    assert same_bits(fc.cpu().numpy(), fcr)


@pytest.mark.parametrize("p_t,n", [(1, 1 << 15), (2, 1 << 14)])
def test_signed_zero_solve(oracle_mod, p_t, n):
    """f = -0 nearly everywhere (a few nonzero slabs) from the zero initial
    guess: residual rows of exact -0 all through the first cycles."""
    nt = p_t + 1
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(p_t), 1.0 / n, n, coarsest=2)
    f = np.full((n, nt), -0.0)
    rng = np.random.default_rng(7)
    idx = rng.integers(0, n, 40)
    f[idx] = rng.standard_normal((40, nt))
    cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8)
    u, st = tmg.solve(hier, f, np.zeros_like(f), cfg)
    ur, norms, iters = oracle_mod.iterate(hier, omegas(hier), f, np.zeros_like(f), 1, 1, 1e-8, 250)
    assert st.iterations == iters and st.residual_norms == norms
    assert same_bits(u, ur)
    assert np.array_equal(np.signbit(u), np.signbit(ur))


# --------------------------------------------------------------------------- host BLAS tree

def _solve_rows_ref(lu, perm, b):
    """BlockLU.solve_rows (dg.py:153-168) for one row vector b, numpy order."""
    n = lu.shape[0]
    if n == 1:
        return b / lu[0, 0]
    y = b[perm].copy()
    for i in range(1, n):
        for j in range(i):
            y[i] -= lu[i, j] * y[j]
    for i in range(n - 1, -1, -1):
        for j in range(i + 1, n):
            y[i] -= lu[i, j] * y[j]
        y[i] /= lu[i, i]
    return y


def test_blas_tree_calibrated_on_this_host():
    """The variant measured on the executing host reproduces the reference's
    forward substitution computed with THIS host's numpy (its dgemv)."""
    res = blas_tree.probe()
    v = blas_tree.calibrated_variant()
    assert all(v in res[nt] for nt in res), res
    for p_t, tau, n in ((1, 0.01, 300), (2, 0.3, 200), (3, 2.0, 150), (0, 0.5, 100)):
        ops = tmg.assemble_local(tmg.BasisSpec(p_t), tau)
        rhs = np.random.default_rng(p_t).standard_normal((n, p_t + 1))
        want = np.empty_like(rhs)
        want[0] = _solve_rows_ref(ops.lu.lu, np.asarray(ops.lu.perm), rhs[0])
        for k in range(1, n):
            want[k] = _solve_rows_ref(ops.lu.lu, np.asarray(ops.lu.perm),
                                      rhs[k] + ops.coupling @ want[k - 1])
        got = tmg.forward_solve(tmg.GlobalSystem(ops, n), rhs)  # default: serial, calibrated tree
        assert same_bits(got, want), (p_t, v)


# --------------------------------------------------------------------------- drop-in edges

def test_solve_broadcast_and_validation():
    import torch
    n = 1 << 12
    rhs, tau, _ = problems.seeded_rhs(1, n, 1.0, 42)
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), tau, n, coarsest=2)
    cfg = tmg.CycleConfig(nu1=1, nu2=1)
    u_ref, st_ref = tmg.solve(hier, rhs, np.zeros_like(rhs), cfg)
    # scalar and row-broadcast initial guesses, as `ws.u[0][0][:] = u_init`
    u_s, st_s = tmg.solve(hier, rhs, 0.0, cfg)
    assert same_bits(u_s, u_ref) and st_s.residual_norms == st_ref.residual_norms
    u_r, _ = tmg.solve(hier, rhs, np.zeros(2), cfg)
    assert same_bits(u_r, u_ref)
    # a CUDA initial guess with a host f
    u_c, _ = tmg.solve(hier, rhs, torch.zeros((n, 2), dtype=torch.float64, device="cuda"), cfg)
    assert isinstance(u_c, np.ndarray) and same_bits(u_c, u_ref)
    # device f, host scalar guess
    u_d, _ = tmg.solve(hier, torch.from_numpy(rhs).cuda(), 0.0, cfg)
    assert same_bits(u_d.cpu().numpy(), u_ref)
    with pytest.raises(ValueError):
        tmg.solve(hier, rhs[:-1], 0.0, cfg)
    with pytest.raises(ValueError):
        tmg.solve(hier, rhs, np.zeros((n, 3)), cfg)
    with pytest.raises(ValueError):
        tmg.solve(hier, torch.from_numpy(rhs[:, :1]).cuda().expand(n, 3), 0.0, cfg)
    F = np.stack([rhs, rhs])
    with pytest.raises(ValueError):
        tmg.solve_batched(hier, F[:, :-2], None, cfg)
    with pytest.raises(ValueError):
        tmg.solve_batched(hier, F, np.zeros((3, n, 2)), cfg)
    with pytest.raises(ValueError):
        tmg.solve_batched(hier, F, None, cfg, floors=[1.0, 2.0, 3.0])
    U, stats = tmg.solve_batched(hier, F, 0.0, cfg)
    assert same_bits(U[0], u_ref) and same_bits(U[1], u_ref)
    with pytest.raises(NotImplementedError):
        nat.level_desc(tmg.assemble_local(tmg.BasisSpec(7), 0.1), 8)


def test_host_pipeline_subplan_reuse(oracle_mod):
    """B = 32 host buffers: more sub-batches than compute sub-plans, so
    sub-plans (their buffers, graphs and pinned staging) are reused."""
    import torch
    n = 1 << 12
    B = 32
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), 1.0 / n, n, coarsest=2)
    F = np.stack([problems.seeded_rhs(1, n, 1.0, 42, b)[0] for b in range(B)])
    cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8)
    os.environ["TMG_HOST_CHUNKS"] = "16"
    try:
        U, stats = tmg.solve_batched(hier, F, None, cfg)
    finally:
        del os.environ["TMG_HOST_CHUNKS"]
    Ud, stats_d = tmg.solve_batched(hier, torch.from_numpy(F).cuda(), None, cfg)
    assert same_bits(U, Ud.cpu().numpy())
    om = omegas(hier)
    for b in (0, 7, 17, 31):
        ur, norms, iters = oracle_mod.iterate(hier, om, F[b], np.zeros_like(F[b]), 1, 1, 1e-8, 250)
        assert stats[b].iterations == iters and stats[b].residual_norms == norms
        assert same_bits(U[b], ur)


# --------------------------------------------------------------------------- GPU right-hand side

@pytest.mark.parametrize("p_t,T", [(0, 1.0), (1, 1.0), (2, 0.01), (3, 100.0)])
def test_rhs_samples_bitwise_with_host(p_t, T):
    """host samples of the forcing -> the kernel's moments == rhs_moments on
    the host bit for bit (numpy's small-K dgemm is a fused multiply-add chain)."""
    from paper_1409_5254_b200 import rhs as rhs_mod
    n = 5000
    a, phi, u0 = problems.forcing_params(42, p_t)
    f = problems.make_forcing(a, phi, T)
    basis = tmg.BasisSpec(p_t)
    host = tmg.rhs_moments(f, basis, T / n, n, u0=u0)
    c, _, _ = rhs_mod.quadrature(basis, T / n)
    times = (np.arange(n)[:, None] + c[None, :]) * (T / n)
    got = tmg.rhs_moments_samples(f(times), basis, T / n, u0).cpu().numpy()
    assert same_bits(got, host)
    # zero forcing: signed zeros of the moments as numpy makes them
    z = tmg.rhs_moments(lambda t: 0.0 * t, basis, T / n, n, u0=0.0)
    gz = tmg.rhs_moments_samples(np.zeros((n, basis.n_t)), basis, T / n, 0.0).cpu().numpy()
    assert same_bits(gz, z) and np.array_equal(np.signbit(gz), np.signbit(z))


@pytest.mark.parametrize("p_t,T", [(0, 1.0), (1, 1.0), (2, 0.01), (2, 100.0), (3, 1.0)])
def test_rhs_sines_kernel_close_to_host(p_t, T):
    n = 1 << 14
    basis = tmg.BasisSpec(p_t)
    ids = [0, 1, 5]
    dev = problems.seeded_rhs_batch_device(p_t, n, T, 42, ids).cpu().numpy()
    for i, b in enumerate(ids):
        host, _, _ = problems.seeded_rhs(p_t, n, T, 42, b)
        err = np.max(np.abs(dev[i] - host)) / np.max(np.abs(host))
        assert err <= 1e-14, (b, err)


def test_rhs_device_callable_and_solve():
    """rhs_moments_device (torch forcing) feeds the solver; iteration counts
    equal those of the host-assembled problem."""
    import torch
    n = 1 << 14
    a, phi, u0 = problems.forcing_params(42)
    basis = tmg.BasisSpec(1)

    def f(t):
        v = torch.zeros_like(t)
        for k in range(8):
            v += a[k] * torch.sin(2.0 * np.pi * (k + 1) * t + phi[k])
        return v

    dev = tmg.rhs_moments_device(f, basis, 1.0 / n, n, u0=u0)
    host, _, _ = problems.seeded_rhs(1, n, 1.0, 42)
    assert np.max(np.abs(dev.cpu().numpy() - host)) <= 1e-14 * np.max(np.abs(host))
    hier = tmg.TimeHierarchy.build(basis, 1.0 / n, n, coarsest=2)
    cfg = tmg.CycleConfig(nu1=1, nu2=1)
    _, st_d = tmg.solve(hier, dev, 0.0, cfg)
    _, st_h = tmg.solve(hier, host, 0.0, cfg)
    assert st_d.iterations == st_h.iterations


# --------------------------------------------------------------------------- single-CTA engine

@pytest.mark.parametrize("p_t", [0, 1, 2, 3])
@pytest.mark.parametrize("n", [4, 8, 16, 64, 512])
def test_tail_cycle_sparse_forcing(oracle_mod, p_t, n):
    """One V-cycle of a problem that lives in the single-CTA engine, with
    zero slabs in f (exact zeros and the IEEE-division fallback of the LU
    solves): bitwise the oracle's cycle (multigrid.py:263-330)."""
    nt = p_t + 1
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(p_t), 1.0 / n, n, coarsest=2)
    rng = np.random.default_rng(n + p_t)
    f = np.zeros((n, nt))
    idx = rng.integers(0, n, max(1, n // 8))
    f[idx] = rng.standard_normal((len(idx), nt))
    for u0 in (np.zeros_like(f), rng.standard_normal((n, nt))):
        cfg = tmg.CycleConfig(nu1=1, nu2=2)
        got = tmg.v_cycle(hier, u0, f, cfg)
        want = oracle_mod.cycle(hier, omegas(hier), u0, f, 1, 2)
        assert same_bits(got, want)


def test_solve_batched_stream_matches_batched(oracle_mod):
    """Batches through the cross-batch pipeline (tmg_plan_solve_host_stream)
    equal separate solves: iterates, norms and counts."""
    import torch
    n, B, nb = 1 << 13, 4, 5
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), 1.0 / n, n, coarsest=2)
    cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8)
    batches = [np.stack([problems.seeded_rhs(1, n, 1.0, 42, k * B + b)[0] for b in range(B)])
               for k in range(nb)]
    outs, stats = tmg.solve_batched_stream(hier, batches, None, cfg)
    assert len(outs) == nb and len(stats) == nb
    for k in range(nb):
        Ud, st_d = tmg.solve_batched(hier, torch.from_numpy(batches[k]).cuda(), None, cfg)
        assert same_bits(outs[k], Ud.cpu().numpy())
        for b in range(B):
            assert stats[k][b].iterations == st_d[b].iterations
            assert stats[k][b].residual_norms == st_d[b].residual_norms
    ur, norms, iters = oracle_mod.iterate(hier, omegas(hier), batches[3][1], np.zeros((n, 2)), 1, 1, 1e-8, 250)
    assert same_bits(outs[3][1], ur) and stats[3][1].residual_norms == norms
    # the same host output buffer reused across batches (written in stream order)
    U = np.empty((B, n, 2))
    outs2, _ = tmg.solve_batched_stream(hier, batches[:2], [U, U], cfg)
    assert same_bits(outs2[1], outs[1])
    with pytest.raises(ValueError):
        tmg.solve_batched_stream(hier, [batches[0][:, :-1]], None, cfg)


def test_phase_times_split(oracle_mod):
    """SolveStats.times with PHASE_TIMES: the traced solve (kernels launched
    one by one) gives the same bits as the graph-launched one and splits the
    device time over the reference's phase keys (multigrid.py:227-241)."""
    from paper_1409_5254_b200 import solver
    n = 1 << 15
    rhs, tau, _ = problems.seeded_rhs(1, n, 1.0, 42)
    hier = tmg.TimeHierarchy.build(tmg.BasisSpec(1), tau, n, coarsest=2)
    cfg = tmg.CycleConfig(nu1=1, nu2=1, eps=1e-8)
    u0, st0 = tmg.solve(hier, rhs, np.zeros_like(rhs), cfg)
    assert set(st0.times) == {"smoothing", "transfer", "coarse", "residual"}
    solver.PHASE_TIMES = True
    try:
        u1, st1 = tmg.solve(hier, rhs, np.zeros_like(rhs), cfg)
    finally:
        solver.PHASE_TIMES = False
    assert u1.tobytes() == u0.tobytes() and st1.residual_norms == st0.residual_norms
    assert set(st1.times) == {"smoothing", "transfer", "coarse", "residual"}
    assert st1.times["smoothing"] > 0 and st1.times["coarse"] > 0 and st1.times["residual"] > 0
    assert st1.times["transfer"] == 0.0


@pytest.mark.parametrize("p_t", [0, 1, 2, 3])
def test_scan_edges_guards_and_alignment(oracle_mod, p_t):
    """grid-wide scan solve through the C ABI at sizes around the tile and run
    boundaries (a tile is 256 slabs for n_t <= 2, 128 above), batched with
    ragged ends, with the output inside guard regions (nothing outside u is
    written) and with a right-hand side that is NOT 16-byte aligned (the
    synchronous fetch path instead of cp.async)."""
    import torch
    nt = p_t + 1
    L = nat.load()
    ops = tmg.assemble_local(tmg.BasisSpec(p_t), 1e-3)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    guard = 64
    for n, B in [(1, 1), (2, 3), (127, 2), (128, 1), (129, 2), (255, 1), (256, 2), (257, 3), (2047, 1),
                 (2049, 2), (256 * 7 + 1, 2), (128 * 33 - 1, 3), (40000, 2)]:
        rng = np.random.default_rng(1000 * p_t + n)
        rhs = rng.standard_normal((B, n, nt))
        d = nat.level_desc(ops, n)
        for shift in (0, 1):   # shift = 1: f starts 8 bytes into its buffer
            fbuf = torch.zeros(B * n * nt + 2, dtype=torch.float64, device="cuda")
            fv = fbuf[shift:shift + B * n * nt]
            fv.copy_(torch.from_numpy(rhs.reshape(-1)))
            ubuf = torch.full((B * n * nt + 2 * guard,), float("nan"), dtype=torch.float64, device="cuda")
            uv = ubuf[guard:guard + B * n * nt]
            nat.check(L.tmg_coarse_solve(nat.F64, ctypes.byref(d), ctypes.c_void_p(fv.data_ptr()),
                                         ctypes.c_void_p(uv.data_ptr()), B, 1, blas_tree.resolve(None), st),
                      "tmg_coarse_solve")
            torch.cuda.synchronize()
            host = ubuf.cpu().numpy()
            assert np.all(np.isnan(host[:guard])) and np.all(np.isnan(host[-guard:])), (n, B, shift)
            got = host[guard:-guard].reshape(B, n, nt)
            assert np.all(np.isfinite(got)), (n, B, shift)
            for b in range(B):
                exact = oracle_mod.forward_solve_extended(ops, rhs[b])
                want = oracle_mod.forward_substitute(ops, rhs[b])
                nrm = max(np.linalg.norm(exact), 1e-300)
                assert np.linalg.norm(got[b] - exact) <= 1e-12 * nrm, (n, B, b, shift)
                assert np.linalg.norm(got[b] - want) <= np.linalg.norm(want - exact) + 1e-12 * nrm


@pytest.mark.parametrize("p_t", [0, 1, 2, 3])
def test_scan_fp32_through_abi(oracle_mod, p_t):
    """the fp32 instantiation of the scan solve (throughput variant: cp.async
    pieces of 4 / 8 / 16 bytes, FMA arithmetic) against the extended-precision
    solution, normwise 1e-4, aligned and unaligned right-hand sides"""
    import torch
    nt = p_t + 1
    L = nat.load()
    ops = tmg.assemble_local(tmg.BasisSpec(p_t), 1e-2)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for n, B in [(5000, 2), (257, 1), (128 * 9, 3)]:
        rhs = np.random.default_rng(77 + n).standard_normal((B, n, nt)).astype(np.float32)
        d = nat.level_desc(ops, n)
        for shift in (0, 1):
            fbuf = torch.zeros(B * n * nt + 4, dtype=torch.float32, device="cuda")
            fv = fbuf[shift:shift + B * n * nt]
            fv.copy_(torch.from_numpy(rhs.reshape(-1)))
            u = torch.full((B * n * nt,), float("nan"), dtype=torch.float32, device="cuda")
            nat.check(L.tmg_coarse_solve(nat.F32, ctypes.byref(d), ctypes.c_void_p(fv.data_ptr()),
                                         ctypes.c_void_p(u.data_ptr()), B, 1, blas_tree.resolve(None), st),
                      "tmg_coarse_solve fp32")
            torch.cuda.synchronize()
            got = u.cpu().numpy().reshape(B, n, nt).astype(np.float64)
            for b in range(B):
                exact = oracle_mod.forward_solve_extended(ops, rhs[b].astype(np.float64))
                assert np.linalg.norm(got[b] - exact) <= 1e-4 * np.linalg.norm(exact), (n, B, b, shift)
