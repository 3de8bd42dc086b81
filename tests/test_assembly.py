"""Host assembly reproduces the reference's per-level constants bit for bit
(golden vectors from the reference, tests/golden/make_golden.py)."""

import numpy as np
import pytest

from paper_1409_5254_b200 import problems
from paper_1409_5254_b200.assembly import BasisSpec, alpha, assemble_local, build_transfers, \
    optimal_omega, resolve_damping
from paper_1409_5254_b200.hierarchy import CycleConfig, TimeHierarchy, max_ratio


def test_assembly_bitwise(golden):
    man, arr = golden
    for row in man["assembly"]:
        key = row["key"]
        basis = BasisSpec(row["p_t"], row["rule"])
        ops = assemble_local(basis, row["tau"])
        r1, r2 = build_transfers(basis, row["tau"])
        got = {"K": ops.stiffness, "M": ops.mass, "C": ops.coupling, "A": ops.minus_step_matrix,
               "lu": ops.lu.lu, "perm": ops.lu.perm, "es": ops.eval_start, "ee": ops.eval_end,
               "r1": r1, "r2": r2}
        for name, val in got.items():
            want = arr[f"{key}_{name}"]
            assert np.asarray(val).tobytes() == want.tobytes(), (key, name)
        a = alpha(basis, row["tau"])
        assert a == row["alpha"], key
        assert optimal_omega(a) == row["omega"], key


def test_seeded_rhs_matches_golden(golden):
    man, arr = golden
    c = next(x for x in man["small_solves"] if x["name"] == "config1")
    rhs, tau, _ = problems.seeded_rhs(1, 1024, 1.0, 42)
    assert rhs.tobytes() == arr["solve_config1_rhs"].tobytes()


def test_hierarchy_sizes(golden):
    man, _ = golden
    for c in man["small_solves"]:
        hier = TimeHierarchy.build(BasisSpec(c["p_t"], c["rule"]), c["T"] / c["n"], c["n"],
                                   n_levels=c["n_levels"], coarsest=c["coarsest"])
        assert [l.n_steps for l in hier.levels] == c["sizes"]
        cfg = CycleConfig(damping=c["damping"])
        om = [resolve_damping(cfg.damping, alpha(hier.basis, l.tau)) for l in hier.levels]
        assert om == c["omegas"]


def test_hierarchy_nesting_and_caps():
    hier = TimeHierarchy.build(BasisSpec(1), 0.25, 64, coarsest=4)
    assert [l.n_steps for l in hier.levels] == [64, 32, 16, 8, 4]
    for fine, coarse in zip(hier.levels, hier.levels[1:]):
        assert coarse.tau == 2.0 * fine.tau
    assert hier.levels[-1].r1 is None
    assert len(TimeHierarchy.build(BasisSpec(0), 1.0, 64, n_levels=2)) == 2
    assert TimeHierarchy.build(BasisSpec(0), 1.0, 8, coarsest=2).levels[-1].n_steps >= 2
    with pytest.raises(ValueError):
        TimeHierarchy.build(BasisSpec(0), 1.0, 1)
    with pytest.raises(ValueError):
        TimeHierarchy.build(BasisSpec(0), -1.0, 8)


def test_config_validation():
    for bad in (dict(nu1=0, nu2=0), dict(eps=1.5), dict(workers=0), dict(max_iters=0),
                dict(levels=0), dict(cycle="X"), dict(coarse="lu")):
        with pytest.raises(ValueError):
            CycleConfig(**bad)
    with pytest.raises(ValueError):
        resolve_damping(2.5, 0.5)
    with pytest.raises(ValueError):
        resolve_damping("fast", 0.5)


def test_max_ratio():
    assert np.isnan(max_ratio([1.0]))
    assert max_ratio([1.0, 0.5]) == 0.5
    assert max_ratio([1.0, 0.1, 0.05, 0.04]) == 0.04 / 0.05
