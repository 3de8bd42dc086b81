"""Pin the CPU oracle (oracle/tmg_oracle.c) to the reference's own outputs.

Every comparison here is bitwise (``tobytes`` equality): the golden vectors in
tests/golden were produced by running the reference (make_golden.py).  Only
then is the oracle trusted as the checker for the GPU path.
"""

import hashlib

import numpy as np
import pytest

from paper_1409_5254_b200 import problems
from paper_1409_5254_b200.assembly import BasisSpec, alpha, assemble_local, build_transfers, \
    optimal_omega
from paper_1409_5254_b200.hierarchy import TimeHierarchy


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def same_bits(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


@pytest.mark.parametrize("n", list(range(0, 140)) + [255, 256, 257, 1000, 1024, 4096, 8191,
                                                    65536, 100003, 1 << 20])
def test_pairwise_sum_matches_numpy(oracle_mod, n):
    rng = np.random.default_rng(n)
    a = rng.random(n) * 10.0 ** rng.uniform(-8, 8, n)
    assert oracle_mod.pairwise_sum(a) == np.sum(a)


def test_sweeps_bitwise(golden, oracle_mod):
    man, arr = golden
    for c in man["sweeps"]:
        k = c["key"]
        ops = assemble_local(BasisSpec(c["p_t"]), c["tau"])
        if c.get("kind") == "primitives":
            r1, r2 = build_transfers(BasisSpec(c["p_t"]), c["tau"])
            r = oracle_mod.residual(ops, arr[f"{k}_f"], arr[f"{k}_u"])
            assert same_bits(r, arr[f"{k}_r"]), k
            fc = oracle_mod.restrict(ops, r1, r2, arr[f"{k}_r"])
            assert same_bits(fc, arr[f"{k}_fc"]), k
            up = oracle_mod.prolong_add(ops, r1, r2, arr[f"{k}_uc"], arr[f"{k}_u"])
            assert same_bits(up, arr[f"{k}_up"]), k
        elif c.get("kind") == "forward_substitute":
            out = oracle_mod.forward_substitute(ops, arr[f"{k}_rhs"])
            assert same_bits(out, arr[f"{k}_out"]), k
        else:
            out = oracle_mod.block_jacobi(ops, arr[f"{k}_u"], arr[f"{k}_f"], c["omega"], c["nu"])
            assert same_bits(out, arr[f"{k}_out"]), k


def _hier(c):
    return TimeHierarchy.build(BasisSpec(c["p_t"], c.get("rule", "radau_lagrange")),
                               c["tau"] if "tau" in c else c["T"] / c["n"], c["n"],
                               n_levels=c["n_levels"], coarsest=c["coarsest"])


def test_cycles_bitwise(golden, oracle_mod):
    man, arr = golden
    for c in man["cycles"]:
        k = c["key"]
        hier = _hier(c)
        assert [l.n_steps for l in hier.levels] == c["sizes"]
        if c["kind"] == "v":
            depth = len(hier.levels)
            out = oracle_mod.cycle(hier, c["omegas"], arr[f"{k}_u"], arr[f"{k}_f"], c["nu1"],
                                   c["nu2"], depth=depth)
        else:
            out = oracle_mod.cycle(hier, c["omegas"], arr[f"{k}_u"], arr[f"{k}_f"], c["nu1"],
                                   c["nu2"], depth=2, level=c["level"])
        assert same_bits(out, arr[f"{k}_out"]), k


def test_small_solves_bitwise(golden, oracle_mod):
    man, arr = golden
    for c in man["small_solves"]:
        name = c["name"]
        hier = _hier(c)
        rhs = arr[f"solve_{name}_rhs"]
        if c["init"] == "zero":
            u0 = np.zeros_like(rhs)
        else:
            u0 = np.random.default_rng(42).random(rhs.shape)
        depth = len(c["omegas"])
        u, norms, iters = oracle_mod.iterate(hier, c["omegas"], rhs, u0, c["nu1"], c["nu2"],
                                             c["eps"], c["max_iters"], depth=depth)
        assert iters == c["iterations"], name
        assert norms == c["residual_norms"], name
        assert same_bits(u, arr[f"solve_{name}_u"]), name


def test_acceptance_criterion9_digest(golden, oracle_mod):
    man, _ = golden
    c = next(x for x in man["big_solves"] if x["name"] == "crit9")
    hier = TimeHierarchy.build(BasisSpec(1), 1e-6, c["n"])
    omegas = [optimal_omega(alpha(hier.basis, l.tau)) for l in hier.levels]
    f = np.zeros((c["n"], 2))
    u0 = np.random.default_rng(42).random((c["n"], 2))
    u, norms, iters = oracle_mod.iterate(hier, omegas, f, u0, 2, 2, 1e-8, 250)
    assert iters == c["iterations"] == 9
    assert norms == c["residual_norms"]
    assert sha(u) == c["sha_u"]
    assert c["sha_u"].startswith("f561263f11d1a65a")  # pkg/test_output.txt:388


def test_config5_prefix(golden, oracle_mod):
    man, arr = golden
    c = man["config5"]
    basis = BasisSpec(c["p_t"])
    ops = assemble_local(basis, c["tau"])
    r1, r2 = build_transfers(basis, c["tau"])
    u, f = problems.kernel_inputs(c["n"], c["p_t"] + 1, 0)
    assert sha(u) == c["sha_u_in"] and sha(f) == c["sha_f_in"]
    us, fc = oracle_mod.down_pass(ops, r1, r2, c["omega"], u, f, c["nu"])
    assert sha(us) == c["sha_u"]
    assert sha(fc) == c["sha_fc"]


@pytest.mark.slow
@pytest.mark.parametrize("name", ["config2_p1", "config2_p3", "config4_T0.01_nu2"])
def test_big_solves(golden, oracle_mod, name):
    man, _ = golden
    found = [x for x in man["big_solves"] if x["name"] == name]
    if not found:
        pytest.skip("golden generated with --quick")
    c = found[0]
    rhs, tau, _ = problems.seeded_rhs(c["p_t"], c["n"], c["T"], 42, c["batch_index"])
    assert sha(rhs) == c["sha_rhs"]
    hier = TimeHierarchy.build(BasisSpec(c["p_t"]), tau, c["n"], coarsest=2)
    omegas = [optimal_omega(alpha(hier.basis, l.tau)) for l in hier.levels]
    u, norms, iters = oracle_mod.iterate(hier, omegas, rhs, np.zeros_like(rhs), c["nu1"],
                                         c["nu2"], 1e-8, 250)
    assert iters == c["iterations"]
    assert norms == c["residual_norms"]
    assert sha(u) == c["sha_u"]


def test_dgemv_tree_calibration(golden):
    """The coarse solve's `coupling @ x` tree (variant 0) reproduces the golden
    host's numpy/OpenBLAS results bit for bit."""
    from math import fsum  # noqa: F401
    from fractions import Fraction

    def fma(a, b, c):
        return float(Fraction(a) * Fraction(b) + Fraction(c))

    trees = {1: lambda a, x: a[0] * x[0],
             2: lambda a, x: fma(a[0], x[0], a[1] * x[1]),
             3: lambda a, x: fma(a[2], x[2], fma(a[0], x[0], a[1] * x[1])),
             4: lambda a, x: (a[0] * x[0] + a[2] * x[2]) + (a[1] * x[1] + a[3] * x[3])}
    _, arr = golden
    for nt in range(1, 5):
        c, x, y = arr[f"dgemv{nt}_c"], arr[f"dgemv{nt}_x"], arr[f"dgemv{nt}_y"]
        for k in range(0, 512, 7):
            for i in range(nt):
                assert trees[nt](c[i], x[k]) + 0.0 == y[k, i]


def test_cycle_kinds_compose(oracle_mod):
    """The W (gamma 2) and F (kind 3) cycles are compositions of the reference's
    own steps: on two levels every kind is the two-grid cycle; on
    three levels F == W (the coarser level's two visits are both two-grid
    cycles); on four levels F differs from both (its second visit of level 1
    is a V-cycle, the W's a W-cycle)."""
    n, p_t = 256, 1
    rhs, tau, _ = problems.seeded_rhs(p_t, n, 1.0, 42)
    hier = TimeHierarchy.build(BasisSpec(p_t), tau, n, coarsest=2)
    from paper_1409_5254_b200.hierarchy import CycleConfig, level_omegas
    om = level_omegas(hier, CycleConfig(), len(hier.levels))
    u0 = np.random.default_rng(1).standard_normal(rhs.shape)
    cyc = lambda g, d: oracle_mod.cycle(hier, om, u0, rhs, 1, 1, depth=d, gamma=g)
    assert same_bits(cyc(3, 2), cyc(1, 2)) and same_bits(cyc(2, 2), cyc(1, 2))
    assert same_bits(cyc(3, 3), cyc(2, 3))
    f4, w4, v4 = cyc(3, 4), cyc(2, 4), cyc(1, 4)
    assert not same_bits(f4, w4) and not same_bits(f4, v4)
    with pytest.raises(AssertionError):
        oracle_mod.cycle(hier, om, u0, rhs, 1, 1, depth=4, gamma=4)
