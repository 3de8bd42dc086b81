"""Time-grid hierarchy, cycle configuration and solve statistics (host side).

Mirrors the reference's data types so code written against ``timemg`` works
unchanged (reference: pkg/src/timemg/multigrid.py):
  Level             multigrid.py:28-37
  TimeHierarchy     multigrid.py:40-80   (build: halve N, double tau while N
                                          is even and N/2 >= max(2, coarsest))
  CycleConfig       multigrid.py:83-116  (+ ``cycle`` = "V" | "W" | "F", ``coarse``)
  SolveStats        multigrid.py:119-134
  _max_ratio        multigrid.py:418-424
Nothing here touches the GPU.
"""

from __future__ import annotations

import dataclasses
from typing import Optional, Sequence

import numpy as np

from .assembly import BasisSpec, LocalOperators, alpha, assemble_local, build_transfers, \
    resolve_damping


@dataclasses.dataclass(frozen=True)
class Level:
    index: int
    n_steps: int
    tau: float
    ops: LocalOperators
    r1: Optional[np.ndarray] = None
    r2: Optional[np.ndarray] = None


class TimeHierarchy:
    """Nested uniform time grids (coarser = half the slabs, twice the step)."""

    def __init__(self, basis: BasisSpec, levels: Sequence[Level]):
        self.basis = basis
        self.levels = list(levels)

    def __len__(self) -> int:
        return len(self.levels)

    @property
    def finest(self) -> Level:
        return self.levels[0]

    @classmethod
    def build(cls, basis: BasisSpec, tau: float, n_steps: int, n_levels="max",
              coarsest: int = 8) -> "TimeHierarchy":
        if n_steps < 2:
            raise ValueError(f"need at least 2 steps, got {n_steps}")
        if tau <= 0:
            raise ValueError(f"time step must be positive, got {tau}")
        cap = np.inf if n_levels == "max" else int(n_levels)
        if cap < 1:
            raise ValueError(f"need at least one level, got {n_levels}")
        out = []
        n, t = n_steps, tau
        while True:
            ops = assemble_local(basis, t)
            if len(out) + 1 < cap and n % 2 == 0 and n // 2 >= max(2, coarsest):
                r1, r2 = build_transfers(basis, t)
                out.append(Level(len(out), n, t, ops, r1, r2))
                n, t = n // 2, 2.0 * t
            else:
                out.append(Level(len(out), n, t, ops))
                return cls(basis, out)


CYCLES = ("V", "W", "F")
# cycle kind codes of the C ABI (TmgPlanOpts.gamma): V 1, W 2 (gamma = 2), F 3
CYCLE_KIND = {"V": 1, "W": 2, "F": 3}
COARSE_SOLVERS = ("auto", "serial", "scan")


@dataclasses.dataclass
class CycleConfig:
    """Solver parameters; the reference fields keep their meaning and defaults.

    Additions (not in the reference): ``cycle`` ("V"; "W" = gamma 2; "F" = an
    F-cycle then a V-cycle on the coarser level), ``coarse`` ("serial", the default: block forward substitution,
    bitwise with the reference; "scan": parallel affine scan, ~1e-15 relative,
    opt-in; "auto": serial unless the coarsest level has > 16384 slabs) and
    ``dot_variant`` (the host-BLAS summation tree the reference's coarse solve
    inherits; None = measured on this host by
    blas_tree.py).  ``workers`` and ``min_slab`` are accepted for
    compatibility; the GPU ignores them.
    """

    nu1: int = 2
    nu2: int = 2
    damping: object = "optimal"
    levels: object = "max"
    eps: float = 1e-8
    max_iters: int = 250
    seed: int = 42
    workers: int = 1
    min_slab: int = 32768
    cycle: str = "V"
    coarse: str = "serial"
    dot_variant: object = None

    def __post_init__(self):
        if self.nu1 < 0 or self.nu2 < 0 or self.nu1 + self.nu2 < 1:
            raise ValueError(f"need nu1, nu2 >= 0 with nu1 + nu2 >= 1, got {self.nu1}, {self.nu2}")
        if not 0.0 < self.eps < 1.0:
            raise ValueError(f"eps must lie in (0, 1), got {self.eps}")
        if self.max_iters < 1:
            raise ValueError(f"max_iters must be >= 1, got {self.max_iters}")
        if self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")
        if self.levels != "max" and int(self.levels) < 1:
            raise ValueError(f"levels must be 'max' or >= 1, got {self.levels}")
        if self.cycle not in CYCLES:
            raise ValueError(f"cycle must be one of {CYCLES}, got {self.cycle!r}")
        if self.coarse not in COARSE_SOLVERS:
            raise ValueError(f"coarse must be one of {COARSE_SOLVERS}, got {self.coarse!r}")
        if self.dot_variant is not None and self.dot_variant not in (0, 1, 2):
            raise ValueError(f"dot_variant must be None, 0, 1 or 2, got {self.dot_variant!r}")


@dataclasses.dataclass
class SolveStats:
    iterations: int
    residual_norms: list
    factor: float
    times: dict
    converged: bool
    seed: int
    workers: int

    def to_dict(self) -> dict:
        return dataclasses.asdict(self)


def max_ratio(norms: Sequence[float]) -> float:
    """Worst ratio of consecutive norms, skipping the first when possible."""
    if len(norms) < 2:
        return float("nan")
    ratios = [norms[k + 1] / norms[k] for k in range(len(norms) - 1) if norms[k] > 0]
    if not ratios:
        return 0.0
    return float(max(ratios[1:])) if len(ratios) > 1 else float(ratios[0])


def depth_of(hier, config: CycleConfig) -> int:
    if config.levels == "max":
        return len(hier.levels)
    return min(len(hier.levels), int(config.levels))


def level_omegas(hier, config: CycleConfig, depth: int) -> list:
    """Per-level damping (multigrid.py:339-341)."""
    return [resolve_damping(config.damping, alpha(hier.basis, lev.tau))
            for lev in hier.levels[:depth]]
