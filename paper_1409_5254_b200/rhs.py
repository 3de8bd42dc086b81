"""Right-hand-side moments on the GPU (rhs_moments, reference dg.py:265-287).

Two forms, both one launch of a hand-written kernel (csrc/tmg_rhs.cu) for a
whole batch:

* ``rhs_moments_samples`` -- forcing values at the quadrature times given
  (any callable evaluated by torch, or host samples): the moments are the
  fused multiply-add chain numpy's matmul performs (``fvals @ weights.T``,
  dg.py:284), so host samples give the reference's rhs bit for bit;
* ``rhs_moments_sines`` -- f(t) = sum_q amp_q sin(2 pi (q+1) t / T + phase_q)
  (the BASELINE problems, problems.py) evaluated inside the kernel: no f
  samples in memory at all; a few ulp from the host assembly (CUDA's sin).

``rhs_moments_device`` keeps the earlier signature (a torch-callable f).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .assembly import basis_values, radau_rule


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("timemg_b200 needs a CUDA device (B200, sm_100a); there is no CPU path")
    return torch


def quadrature(basis, tau: float):
    """(nodes c_k, weights (n_t, s) = tau * basis_values(c) * b, start values)
    exactly as rhs_moments forms them (dg.py:276-278, 286)."""
    rule = radau_rule(basis.n_t)
    weights = tau * basis_values(basis, rule.c) * rule.b
    start = basis_values(basis, np.array([0.0]))[:, 0]
    return (np.ascontiguousarray(rule.c, dtype=np.float64),
            np.ascontiguousarray(weights, dtype=np.float64),
            np.ascontiguousarray(start, dtype=np.float64))


def quadrature_times(basis, tau: float, n_steps: int, t0: float = 0.0, device="cuda"):
    """t0 + (n + c_k) tau as a (n_steps, s) float64 CUDA tensor (dg.py:279)."""
    torch = _torch()
    c, _, _ = quadrature(basis, tau)
    n = torch.arange(n_steps, device=device, dtype=torch.float64)[:, None]
    return t0 + (n + torch.from_numpy(c).to(device)[None, :]) * tau


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _check(rc, what):
    if rc:
        msg = nat.load().tmg_rhs_last_error().decode(errors="replace")
        if rc == nat.E_ARG:
            raise ValueError(f"{what}: {msg}")
        if rc == nat.E_UNSUPPORTED:
            raise NotImplementedError(f"{what}: {msg}")
        raise RuntimeError(f"{what}: CUDA error {rc}: {msg}")


def rhs_moments_samples(fvals, basis, tau: float, u0=0.0):
    """Moments of sampled forcing values: fvals (n, s) or (B, n, s) float64
    (CUDA tensor or host array); u0 a scalar or one value per problem.
    Returns a float64 CUDA tensor (n, n_t) or (B, n, n_t)."""
    torch = _torch()
    fv = fvals.to(device="cuda", dtype=torch.float64) if torch.is_tensor(fvals) else \
        torch.from_numpy(np.ascontiguousarray(fvals, dtype=np.float64)).cuda()
    squeeze = fv.dim() == 2
    if squeeze:
        fv = fv[None]
    fv = fv.contiguous()
    B, n, s = fv.shape
    c, w, start = quadrature(basis, tau)
    if s != len(c):
        raise ValueError(f"fvals has {s} samples per step, the rule has {len(c)} nodes")
    u0s = np.array(np.broadcast_to(np.asarray(u0, dtype=np.float64), (B,)))  # writable copy for torch
    u0d = torch.from_numpy(np.ascontiguousarray(u0s)).cuda() if np.any(u0s != 0.0) else None
    out = torch.empty((B, n, basis.n_t), dtype=torch.float64, device="cuda")
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _check(nat.load().tmg_rhs_samples(ctypes.c_void_p(fv.data_ptr()),
                                      ctypes.c_void_p(u0d.data_ptr() if u0d is not None else 0),
                                      _dptr(c), _dptr(w), _dptr(start), basis.n_t, s,
                                      ctypes.c_void_p(out.data_ptr()), n, B, stream), "tmg_rhs_samples")
    return out[0] if squeeze else out


def sine_frequencies(n_terms: int) -> np.ndarray:
    """2.0 * np.pi * (k + 1) as Python forms it in the forcing (problems.py)."""
    return np.array([2.0 * np.pi * (k + 1) for k in range(n_terms)], dtype=np.float64)


def rhs_moments_sines(basis, tau: float, n_steps: int, amp, phase, T: float = 1.0, u0=0.0,
                      t0: float = 0.0):
    """Moments of f_b(t) = sum_q amp[b, q] sin(2 pi (q+1) t / T + phase[b, q])
    for every problem b in one launch.  amp, phase: (B, K) or (K,); u0: scalar
    or (B,).  Returns (B, n, n_t) (or (n, n_t) for 1-D amp) float64 CUDA."""
    torch = _torch()
    amp = np.asarray(amp, dtype=np.float64)
    phase = np.asarray(phase, dtype=np.float64)
    squeeze = amp.ndim == 1
    amp2, ph2 = np.atleast_2d(amp), np.atleast_2d(phase)
    if amp2.shape != ph2.shape:
        raise ValueError(f"amp {amp2.shape} and phase {ph2.shape} differ")
    B, K = amp2.shape
    c, w, start = quadrature(basis, tau)
    freq = sine_frequencies(K)
    u0s = np.array(np.broadcast_to(np.asarray(u0, dtype=np.float64), (B,)))  # writable copy for torch
    ad = torch.from_numpy(np.ascontiguousarray(amp2)).cuda()
    pd = torch.from_numpy(np.ascontiguousarray(ph2)).cuda()
    u0d = torch.from_numpy(np.ascontiguousarray(u0s)).cuda() if np.any(u0s != 0.0) else None
    out = torch.empty((B, n_steps, basis.n_t), dtype=torch.float64, device="cuda")
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _check(nat.load().tmg_rhs_sines(ctypes.c_void_p(ad.data_ptr()), ctypes.c_void_p(pd.data_ptr()),
                                    ctypes.c_void_p(u0d.data_ptr() if u0d is not None else 0),
                                    _dptr(freq), K, float(T), float(tau), float(t0), _dptr(c), _dptr(w),
                                    _dptr(start), basis.n_t, len(c), ctypes.c_void_p(out.data_ptr()),
                                    n_steps, B, stream), "tmg_rhs_sines")
    return out[0] if squeeze else out


def rhs_moments_device(f, basis, tau: float, n_steps: int, u0: float = 0.0, t0: float = 0.0,
                       device: str = "cuda"):
    """rhs_moments (dg.py:265-287) with the forcing evaluated on the GPU: ``f``
    maps a float64 CUDA tensor of times (n_steps, s) to values of the same
    shape (torch ops); the moments come from the tmg_rhs_samples kernel.
    Returns a (n_steps, n_t) float64 CUDA tensor."""
    torch = _torch()
    times = quadrature_times(basis, tau, n_steps, t0, device)
    fv = f(times)
    if not torch.is_tensor(fv) or fv.shape != times.shape:
        raise TypeError("f must map a (n_steps, s) float64 tensor to values of the same shape")
    return rhs_moments_samples(fv, basis, tau, u0)
