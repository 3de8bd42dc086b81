"""Calibration of the host-BLAS summation tree the reference's coarse solve inherits.

The reference's exact coarsest-level solve computes ``coupling @ out[n-1]``
with numpy matmul (multigrid.py:205, and dg.py:302 in ``forward_solve``),
i.e. through the host's BLAS dgemv.  The dgemv micro-kernel fixes how the
n_t products of a row are rounded and summed (with or without FMA, in which
tree), and that differs between BLAS builds and CPU kernels.  For bitwise
parity the GPU coarse solve must use the tree of the host the reference runs
on, so the tree is measured here, on the executing host, by running numpy on
random operands and comparing every row with exact emulations of the trees
the kernels implement (``blas_dot`` in csrc/tmg_slab.cuh, ``tmo_blas_dot_row``
in the oracle):

  variant 0  OpenBLAS 0.3.30 dgemv_t small-n trees (Haswell kernels; measured
             on the golden host):  n=1 a0x0;  n=2 fma(a0,x0,a1x1);
             n=3 fma(a2,x2,fma(a0,x0,a1x1));  n=4 (a0x0+a2x2)+(a1x1+a3x3)
  variant 1  sequential, separately rounded: ((a0x0 + a1x1) + a2x2) + ...
  variant 2  sequential FMA chain: t = a0x0; t = fma(aj, xj, t), j = 1..

every result then "+ 0.0" (dgemv accumulates into a zeroed y).  No match
raises: the solve would otherwise silently differ from the reference on this
host (CycleConfig.dot_variant can still force a variant explicitly).
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

VARIANTS = (0, 1, 2)
NAMES = {0: "openblas-haswell-small-n", 1: "sequential", 2: "fma-chain"}


def _fma(a: float, b: float, c: float) -> float:
    # exact a*b + c, rounded once (int true division is correctly rounded)
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def emulate(variant: int, a, x) -> float:
    n = len(a)
    a = [float(v) for v in a]
    x = [float(v) for v in x]
    if variant == 1 or (variant == 0 and n > 4):
        t = a[0] * x[0]
        for j in range(1, n):
            t = t + a[j] * x[j]
    elif variant == 2:
        t = a[0] * x[0]
        for j in range(1, n):
            t = _fma(a[j], x[j], t)
    elif n == 1:
        t = a[0] * x[0]
    elif n == 2:
        t = _fma(a[0], x[0], a[1] * x[1])
    elif n == 3:
        t = _fma(a[2], x[2], _fma(a[0], x[0], a[1] * x[1]))
    else:
        t = (a[0] * x[0] + a[2] * x[2]) + (a[1] * x[1] + a[3] * x[3])
    return t + 0.0


def probe(n_samples: int = 256, seed: int = 20260101, max_nt: int = 4) -> dict:
    """{n_t: [variants whose every row equals numpy's `c @ x` bit for bit]}."""
    rng = np.random.default_rng(seed)
    out = {}
    for nt in range(1, max_nt + 1):
        ok = {v: True for v in VARIANTS}
        for k in range(n_samples):
            # mixed magnitudes make the trees distinguishable
            c = rng.standard_normal((nt, nt)) * np.exp2(rng.integers(-20, 20, (nt, nt)))
            x = rng.standard_normal(nt) * np.exp2(rng.integers(-20, 20, nt))
            y = c @ x
            for v in VARIANTS:
                if ok[v] and any(emulate(v, c[i], x) != y[i] or
                                 np.signbit(emulate(v, c[i], x)) != np.signbit(y[i])
                                 for i in range(nt)):
                    ok[v] = False
        out[nt] = [v for v in VARIANTS if ok[v]]
    return out


_CACHE: dict = {}


def calibrated_variant(max_nt: int = 4) -> int:
    """The tree variant that reproduces this host's numpy matmul for every
    n_t <= max_nt (measured once per process).  Raises RuntimeError when none
    of the implemented trees matches."""
    if max_nt not in _CACHE:
        res = probe(max_nt=max_nt)
        common = [v for v in VARIANTS if all(v in res[nt] for nt in res)]
        if not common:
            raise RuntimeError(
                "no implemented dgemv summation tree reproduces this host's numpy "
                f"`c @ x` (matches per n_t: {res}); the coarse solve cannot be bitwise "
                "with the reference here. Pass CycleConfig(dot_variant=...) to force one.")
        # prefer the tree the golden vectors were measured with
        _CACHE[max_nt] = 0 if 0 in common else common[0]
    return _CACHE[max_nt]


def resolve(dot_variant) -> int:
    """CycleConfig.dot_variant -> the variant passed to the kernels."""
    if dot_variant is None:
        return calibrated_variant()
    v = int(dot_variant)
    if v not in VARIANTS:
        raise ValueError(f"dot_variant must be None or one of {VARIANTS}, got {dot_variant!r}")
    return v
