"""The host-BLAS summation-tree calibration (blas_tree.py) on this host: the
emulations reproduce numpy's `c @ x` for the tree they name, and the golden
host's tree (variant 0) is what this image's numpy/OpenBLAS computes."""

import numpy as np
import pytest

from paper_1409_5254_b200 import CycleConfig, blas_tree


def test_emulations_are_exact_trees():
    a = np.array([1.0, 2.0 ** -60, -1.0, 3.0])
    x = np.array([1.0, 1.0, 1.0, 2.0 ** -55])
    # sequential: ((1 + 2^-60) - 1) + 3 * 2^-55 rounds the tiny term away
    assert blas_tree.emulate(1, a[:3], x[:3]) == 0.0
    for v in blas_tree.VARIANTS:
        assert blas_tree.emulate(v, [2.0], [3.0]) == 6.0
        assert not np.signbit(blas_tree.emulate(v, [-0.0], [1.0]))  # "+ 0.0" of the zeroed y


def test_probe_finds_this_hosts_tree():
    res = blas_tree.probe(n_samples=64)
    assert set(res) == {1, 2, 3, 4}
    v = blas_tree.calibrated_variant()
    assert all(v in res[nt] for nt in res)
    assert blas_tree.resolve(None) == v
    assert blas_tree.resolve(1) == 1
    with pytest.raises(ValueError):
        blas_tree.resolve(7)


def test_config_accepts_none_and_rejects_unknown_variant():
    assert CycleConfig().dot_variant is None and CycleConfig().coarse == "serial"
    with pytest.raises(ValueError):
        CycleConfig(dot_variant=5)
