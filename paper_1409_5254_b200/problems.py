"""Seeded synthetic inputs for the BASELINE configurations.

The model problem is u' + u = f on (0, T) with
    f(t) = sum_{k=1..8} a_k sin(2 pi k t / T + phi_k),
a_k ~ N(0, 1), phi_k ~ U(0, 2 pi), u0 ~ N(0, 1), drawn in that order from
``numpy.random.default_rng(seed)`` (seed 42 = the reference's default seed,
multigrid.py:102); problem b of a batch uses ``default_rng([seed, b])``.
The right-hand side is the reference quadrature ``rhs_moments``
(dg.py:265-287).  No public dataset is involved.
"""

from __future__ import annotations

import numpy as np

from .assembly import BasisSpec, rhs_moments


def forcing_params(seed=42, batch_index=None):
    rng = np.random.default_rng(seed if batch_index is None else [seed, batch_index])
    a = rng.standard_normal(8)
    phi = rng.uniform(0.0, 2.0 * np.pi, 8)
    u0 = float(rng.standard_normal())
    return a, phi, u0


def make_forcing(a, phi, T: float):
    a = np.asarray(a, dtype=float)
    phi = np.asarray(phi, dtype=float)

    def f(t):
        t = np.asarray(t, dtype=float)
        out = np.zeros_like(t)
        for k in range(8):
            out += a[k] * np.sin(2.0 * np.pi * (k + 1) * t / T + phi[k])
        return out

    return f


def seeded_rhs(p_t: int, n_steps: int, T: float = 1.0, seed=42, batch_index=None):
    """(rhs, tau, u0) for one seeded problem: rhs shape (n_steps, p_t + 1)."""
    a, phi, u0 = forcing_params(seed, batch_index)
    tau = T / n_steps
    rhs = rhs_moments(make_forcing(a, phi, T), BasisSpec(p_t), tau, n_steps, u0=u0)
    return rhs, tau, u0


def kernel_inputs(n_steps: int, n_t: int, seed: int = 0):
    """Config 5: u and f iid N(0, 1), u drawn first (default_rng(0))."""
    rng = np.random.default_rng(seed)
    u = rng.standard_normal((n_steps, n_t))
    f = rng.standard_normal((n_steps, n_t))
    return u, f


def seeded_rhs_batch_device(p_t: int, n_steps: int, T: float = 1.0, seed=42, batch_indices=(0,),
                            device="cuda"):
    """The seeded problems of ``seeded_rhs`` assembled on the GPU in ONE launch
    of the tmg_rhs_sines kernel (rhs.py): the forcing is evaluated in the
    kernel, nothing but the 17 parameters per problem crosses PCIe.  Values
    agree with the host assembly to a few ulp (CUDA's sin; the parity tests
    and the bench's parity pins use host inputs).  Returns a
    (B, n_steps, p_t + 1) float64 tensor."""
    from .rhs import rhs_moments_sines

    params = [forcing_params(seed, b) for b in batch_indices]
    amp = np.stack([a for a, _, _ in params])
    phase = np.stack([p for _, p, _ in params])
    u0 = np.array([u for _, _, u in params])
    return rhs_moments_sines(BasisSpec(p_t), T / n_steps, n_steps, amp, phase, T, u0)
