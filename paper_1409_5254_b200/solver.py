"""GPU-backed drop-in for the reference solver API (pkg/src/timemg/multigrid.py).

Same names, arguments, defaults, return values and errors as the reference:
  block_jacobi_sweep(ops, u, f, omega, nu=1)           multigrid.py:208-220
  two_grid_cycle(hier, level, u, f, config=None)       multigrid.py:355-363
  v_cycle(hier, u, f, config=None)                     multigrid.py:366-375
  solve(hier, f, u_init=None, config=None)             multigrid.py:509-531
  measure_convergence_factor(hier, config=None)        multigrid.py:534-544
  random_initial_guess(hier, seed)                     multigrid.py:503-506
plus ``solve_batched`` (B independent right-hand sides sharing one operator,
each stopping at its own iteration count) and the W- and F-cycles via
``CycleConfig(cycle="W" | "F")``.

Arrays may be numpy (host; results come back as numpy) or torch CUDA tensors
(device-resident; results stay on the device).  Every numeric step runs in the
sm_100a kernels behind the C ABI; there is no CPU fallback.  ``hier`` may be
this package's TimeHierarchy or the reference's own (duck-typed: ``levels``
with ``n_steps``, ``tau``, ``ops``, ``r1``, ``r2``; ``basis``).
"""

from __future__ import annotations

import ctypes
import os
import time

import numpy as np

from . import _native as nat
from . import blas_tree
from .hierarchy import CYCLE_KIND, CycleConfig, SolveStats, depth_of, level_omegas, max_ratio

_COARSE = {"serial": 0, "scan": 1, "auto": 2}
# levels with at most this many slabs per problem run in the single-CTA engine
# (0 = library default); exposed for tests of split invariance
TAIL_MAX = 0


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("timemg_b200 needs a CUDA device (B200, sm_100a); there is no CPU path")
    return torch


def _dev(x, dtype_np=np.float64):
    """(device tensor, was_torch).  numpy input is copied host->device."""
    torch = _torch()
    tdt = torch.float64 if dtype_np == np.float64 else torch.float32
    if torch.is_tensor(x):
        t = x.to(device="cuda", dtype=tdt).contiguous()
        return t, True
    return torch.from_numpy(np.ascontiguousarray(x, dtype=dtype_np)).to("cuda"), False


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _is_host(x) -> bool:
    if isinstance(x, np.ndarray):
        return True
    try:
        import torch
        return torch.is_tensor(x) and not x.is_cuda
    except ImportError:
        return False


def _is_torch_cuda(x) -> bool:
    try:
        import torch
        return torch.is_tensor(x) and x.is_cuda
    except ImportError:
        return False


def _host_ptr(x) -> int:
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def _host_array(x, copy: bool):
    """C-contiguous float64 host array (numpy, or a CPU torch tensor kept as is)."""
    if isinstance(x, np.ndarray):
        return np.array(x, dtype=np.float64, order="C", copy=True) if copy else \
            np.ascontiguousarray(x, dtype=np.float64)
    import torch
    if torch.is_tensor(x):
        t = x.to(torch.float64).contiguous()
        return t.clone() if copy and t.data_ptr() == x.data_ptr() else t
    return np.array(x, dtype=np.float64, order="C", copy=True)


def _check_device():
    nat.check(nat.load().tmg_device_check(0), "timemg_b200 needs a CUDA device (B200, sm_100a)")


def _to_numpy(x):
    """numpy view of a numpy array, scalar, list or (CPU or CUDA) torch tensor."""
    if isinstance(x, np.ndarray):
        return x
    try:
        import torch
        if torch.is_tensor(x):
            return x.detach().cpu().numpy()
    except ImportError:
        pass
    return np.asarray(x, dtype=np.float64)


def _host_block(x, shape, what: str, copy: bool):
    """C-contiguous float64 host array of exactly ``shape``.  Anything numpy
    broadcasts to that shape is accepted, as the reference's assignments
    ``ws.u[0][0][:] = u_init`` / ``ws.f[0][:] = f`` do (multigrid.py:437-438);
    anything else raises ValueError before a pointer reaches the C ABI."""
    if _is_host(x) and tuple(x.shape) == shape:
        return _host_array(x, copy)
    src = _to_numpy(x)
    out = np.empty(shape, dtype=np.float64)
    try:
        out[...] = src
    except ValueError as e:
        raise ValueError(f"{what} of shape {np.shape(src)} does not broadcast to {shape}") from e
    return out


def _dev_block(x, shape, what: str):
    """(float64 CUDA tensor of exactly ``shape``, was_torch); broadcasts like
    the reference's assignments, ValueError otherwise."""
    torch = _torch()
    was_t = torch.is_tensor(x)
    t = x.to(device="cuda", dtype=torch.float64) if was_t else \
        torch.from_numpy(np.ascontiguousarray(_to_numpy(x), dtype=np.float64)).to("cuda")
    if tuple(t.shape) != shape:
        try:
            t = t.expand(shape)
        except RuntimeError as e:
            raise ValueError(f"{what} of shape {tuple(t.shape)} does not broadcast to {shape}") from e
    return t.contiguous(), was_t


def _check_floors(floors, B):
    fl = np.ascontiguousarray(np.broadcast_to(np.asarray(floors, dtype=np.float64), (B,)))
    return fl


def _out(t, was_torch):
    if was_torch:
        return t
    return t.cpu().numpy()


def _level_descs(hier, level0, depth, omegas):
    levels = hier.levels[level0:level0 + depth]
    out = []
    for i, lev in enumerate(levels):
        last = i + 1 == depth
        out.append(nat.level_desc(lev.ops, lev.n_steps, omegas[i],
                                  None if last else lev.r1, None if last else lev.r2))
    return out


class DevicePlan:
    """A tmg_plan: level constants, per-level device buffers, launch schedule.
    ``multi`` (a list of (hier, omegas) pairs): one operator per problem."""

    def __init__(self, hier, level0: int, depth: int, omegas, config: CycleConfig, batch: int,
                 dtype: int = nat.F64, use_graph: bool = True, multi=None):
        lib = nat.load()
        if multi is None:
            flat = _level_descs(hier, level0, depth, omegas)
        else:
            flat = [d for h, om in multi for d in _level_descs(h, level0, depth, om)]
        descs = (nat.LevelDesc * len(flat))(*flat)
        self.depth = depth
        self.batch = batch
        self.n0 = flat[0].n_slabs
        self.n_t = flat[0].n_t
        self.dtype = dtype
        opts = nat.PlanOpts(dtype, config.nu1, config.nu2, CYCLE_KIND[config.cycle],
                            _COARSE[config.coarse], blas_tree.resolve(config.dot_variant), int(use_graph),
                            int(TAIL_MAX))
        self._h = ctypes.c_void_p()
        create = lib.tmg_plan_create if multi is None else lib.tmg_plan_create_multi
        nat.check(create(ctypes.byref(self._h), descs, depth, batch, ctypes.byref(opts)),
                  "tmg_plan_create")

    def __del__(self):
        h = getattr(self, "_h", None)
        lib = getattr(nat, "_lib", None) if nat is not None else None
        if h is not None and h.value and lib is not None:
            lib.tmg_plan_destroy(h)
            self._h = None

    def cycles(self, f_dev, u_dev, n_cycles: int = 1):
        nat.check(nat.load().tmg_plan_cycles(self._h, _ptr(f_dev), _ptr(u_dev), int(n_cycles),
                                             _stream()), "tmg_plan_cycles")

    def solve(self, f_dev, u_dev, floors, eps: float, max_iters: int):
        floors = np.ascontiguousarray(floors, dtype=np.float64)
        nat.check(nat.load().tmg_plan_solve(
            self._h, _ptr(f_dev), _ptr(u_dev),
            floors.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), float(eps), int(max_iters),
            _stream()), "tmg_plan_solve")
        return self._stats(max_iters)

    def solve_host(self, f_host, u_init, u_out, floors, eps: float, max_iters: int):
        """Host buffers (numpy or CPU torch, ideally pinned) in and out: the
        C ABI copies in (u_init None = zero guess), solves and copies the
        solution into u_out."""
        floors = np.ascontiguousarray(floors, dtype=np.float64)
        uin = None if u_init is None else ctypes.c_void_p(_host_ptr(u_init))
        nat.check(nat.load().tmg_plan_solve_host(
            self._h, ctypes.c_void_p(_host_ptr(f_host)), uin, ctypes.c_void_p(_host_ptr(u_out)),
            floors.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), float(eps), int(max_iters)),
            "tmg_plan_solve_host")
        return self._stats(max_iters)

    def solve_host_stream(self, F_hosts, U_hosts, floors, eps: float, max_iters: int):
        """Batches of host buffers (pinned for full PCIe speed) from the zero
        guess, pipelined across batches (tmg_plan_solve_host_stream).
        Returns per batch (iterations[B], norms[B, max_iters+1], converged[B])."""
        nb = len(F_hosts)
        fl = np.ascontiguousarray(np.broadcast_to(np.asarray(floors, dtype=np.float64), (nb, self.batch)))
        fp = (ctypes.c_void_p * nb)(*[_host_ptr(x) for x in F_hosts])
        up = (ctypes.c_void_p * nb)(*[_host_ptr(x) for x in U_hosts])
        it = np.zeros((nb, self.batch), dtype=np.int32)
        conv = np.zeros((nb, self.batch), dtype=np.int32)
        norms = np.zeros((nb, self.batch, max_iters + 1))
        nat.check(nat.load().tmg_plan_solve_host_stream(
            self._h, nb, fp, up, fl.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), float(eps),
            int(max_iters), it.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            norms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            conv.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))), "tmg_plan_solve_host_stream")
        return [(it[k], norms[k], conv[k]) for k in range(nb)]

    def _stats(self, max_iters):
        it = np.zeros(self.batch, dtype=np.int32)
        conv = np.zeros(self.batch, dtype=np.int32)
        norms = np.zeros(self.batch * (max_iters + 1))
        nat.check(nat.load().tmg_plan_stats(
            self._h, it.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            norms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            conv.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))), "tmg_plan_stats")
        return it, norms.reshape(self.batch, max_iters + 1), conv

    def info(self):
        k = ctypes.c_int32()
        s = ctypes.c_int32()
        t = ctypes.c_int32()
        nat.check(nat.load().tmg_plan_info(self._h, ctypes.byref(k), ctypes.byref(s),
                                           ctypes.byref(t)))
        return {"kernels_per_cycle": k.value, "tail_level": t.value}


def omegas_for(hier, config, depth):
    """Per-level damping, cached on the hierarchy (alpha needs a small complex
    solve per level; multigrid.py:339-341)."""
    cache = hier.__dict__.setdefault("_tmg_omegas", {})
    key = (repr(config.damping), depth)
    if key not in cache:
        cache[key] = level_omegas(hier, config, depth)
    return cache[key]


def get_plan(hier, level0, depth, omegas, config, batch, dtype=nat.F64):
    key = (level0, depth, tuple(omegas), config.nu1, config.nu2, config.cycle, config.coarse,
           blas_tree.resolve(config.dot_variant), batch, dtype, TAIL_MAX)
    cache = hier.__dict__.setdefault("_tmg_plans", {})
    plan = cache.get(key)
    if plan is None:
        if len(cache) > 8:
            cache.clear()
        plan = DevicePlan(hier, level0, depth, omegas, config, batch, dtype)
        cache[key] = plan
    return plan


# ---------------------------------------------------------------------------
# reference API


def random_initial_guess(hier, seed: int) -> np.ndarray:
    """Uniform [0, 1) coefficients (multigrid.py:503-506)."""
    rng = np.random.default_rng(seed)
    return rng.random((hier.finest.n_steps, hier.finest.ops.n_t))


def block_jacobi_sweep(ops, u, f, omega: float, nu: int = 1):
    """nu damped block-Jacobi sweeps on the GPU (multigrid.py:208-220)."""
    if not 0.0 < omega < 2.0:
        raise ValueError(f"damping must lie in (0, 2), got {omega}")
    if nu < 0:
        raise ValueError(f"sweep count must be >= 0, got {nu}")
    ud, was_t = _dev(u)
    fd, _ = _dev(f)
    out = _torch().empty_like(ud)
    n = ud.shape[0]
    d = nat.level_desc(ops, n, omega)
    nat.check(nat.load().tmg_sweep(nat.F64, ctypes.byref(d), _ptr(fd), _ptr(ud), _ptr(out), 1,
                                   int(nu), None, _stream()), "tmg_sweep")
    return _out(out, was_t)


def _cycle_api(hier, level, depth_total, u, f, config):
    ud, was_t = _dev(u)
    fd, _ = _dev(f)
    omegas = omegas_for(hier, config, depth_total)[level:]
    plan = get_plan(hier, level, depth_total - level, omegas, config, 1)
    out = ud.clone()
    plan.cycles(fd, out, 1)
    return _out(out, was_t)


def two_grid_cycle(hier, level: int, u, f, config: CycleConfig = None):
    """Pre-smooth, restrict, exact coarse solve, prolongate, post-smooth
    (multigrid.py:355-363)."""
    config = config or CycleConfig()
    if level + 1 >= len(hier.levels):
        raise ValueError(f"level {level} has no coarser neighbor")
    return _cycle_api(hier, level, level + 2, u, f, config)


def v_cycle(hier, u, f, config: CycleConfig = None):
    """One V-cycle (or W-/F-cycle with config.cycle == "W"/"F") from the finest level
    (multigrid.py:366-375)."""
    config = config or CycleConfig()
    depth = depth_of(hier, config)
    if depth < 2:
        raise ValueError("v_cycle needs a hierarchy with at least 2 levels")
    return _cycle_api(hier, 0, depth, u, f, config)


SCAN_AUTO_MIN = 16384  # "auto": longer coarse solves use the parallel scan


def _forward_solve_dev(ops, n, fd, config, batch=1):
    torch = _torch()
    u = torch.empty_like(fd)
    d = nat.level_desc(ops, n)
    method = {"serial": 0, "scan": 1}.get(config.coarse, 1 if n > SCAN_AUTO_MIN else 0)
    nat.check(nat.load().tmg_coarse_solve(nat.F64, ctypes.byref(d), _ptr(fd), _ptr(u), batch, method,
                                          blas_tree.resolve(config.dot_variant), _stream()),
              "tmg_coarse_solve")
    return u


def forward_solve(system, rhs, method: str = "serial"):
    """Exact solve of the block lower-bidiagonal system on the GPU
    (dg.py:290-303).  method "serial" (default): block forward substitution,
    bitwise with the reference; "scan" (opt-in): the parallel associative scan
    of the rank-1 slab recurrence (~1e-15 relative, not bitwise).
    rhs: (n_steps, n_t) or (B, n_steps, n_t); numpy in -> numpy out."""
    if getattr(system, "periodic", False):
        raise ValueError("forward substitution requires a non-periodic system")
    rd, was_t = _dev(rhs)
    batch = rd.shape[0] if rd.dim() == 3 else 1
    n = rd.shape[-2]
    if n != system.n_steps or rd.shape[-1] != system.ops.n_t:
        raise ValueError(f"rhs shape {tuple(rd.shape)} does not match ({system.n_steps}, {system.ops.n_t})")
    u = _forward_solve_dev(system.ops, n, rd, CycleConfig(coarse=method), batch)
    return _out(u, was_t)


def _floor_of(f) -> float:
    torch = _torch()
    if torch.is_tensor(f):
        return 1e-12 * float(torch.linalg.norm(f.double()))
    return 1e-12 * float(np.linalg.norm(f))


# SolveStats.times (multigrid.py:227-241 splits smoothing / transfer / coarse /
# residual).  The fused kernels run several of the reference's phases in one
# launch, so by default the device solve's wall time is reported under
# "smoothing".  With PHASE_TIMES (or TMG_PHASE_TIMES=1) the solve runs under
# the library's kernel trace (every kernel launched separately and timed with
# CUDA events: slower than the graph-launched solve) and the kernel times are
# split as
#   "smoothing": the streaming level passes (sweeps fused with the residual,
#                restriction and prolongation of the same pass: "transfer" is
#                part of them and stays 0),
#   "coarse":    the single-CTA engine (every level <= 1024 slabs and the
#                coarsest-level solve),
#   "residual":  norm finalisation, stopping test and its host round trip.
PHASE_TIMES = os.environ.get("TMG_PHASE_TIMES", "") not in ("", "0")


def _times(total: float) -> dict:
    return {"smoothing": total, "transfer": 0.0, "coarse": 0.0, "residual": 0.0}


def _phase_bucket(kernel_name: str) -> str:
    if "tail" in kernel_name or "coarse" in kernel_name:
        return "coarse"
    if kernel_name.startswith("stream_kernel"):
        return "smoothing"
    return "residual"


def _traced(call):
    """Run call() under the kernel trace; returns (result, times dict)."""
    L = nat.load()
    L.tmg_trace_enable(1)
    try:
        out = call()
        buf = ctypes.create_string_buffer(1 << 20)
        L.tmg_trace_read(buf, len(buf))
    finally:
        L.tmg_trace_enable(0)
    times = _times(0.0)
    for line in buf.value.decode().splitlines():
        name, _, ms = line.split("\t")
        if name != "start":
            times[_phase_bucket(name)] += 1e-3 * float(ms)
    return out, times


def solve(hier, f, u_init=None, config: CycleConfig = None):
    """Cycle until ||r|| <= max(eps ||r0||, 1e-12 ||f||) (multigrid.py:509-531).
    Returns (u, SolveStats); non-convergence is a flag, not an exception."""
    config = config or CycleConfig()
    depth = depth_of(hier, config)
    shape = (hier.finest.n_steps, hier.finest.ops.n_t)
    if u_init is None:
        u_init = random_initial_guess(hier, config.seed)
    if depth >= 2 and (_is_host(f) or not _is_torch_cuda(f)):
        # host arrays (numpy, CPU torch, scalars): the C ABI's host-buffer
        # entry point, no torch.  floor = 1e-12 ||f|| of f as given
        # (multigrid.py:445), before broadcasting.
        _check_device()
        fh = _host_block(f, shape, "f", copy=False)
        uh = _host_block(u_init, shape, "u_init", copy=True)
        floor = 1e-12 * float(np.linalg.norm(_to_numpy(f).astype(np.float64, copy=False)))
        plan = get_plan(hier, 0, depth, omegas_for(hier, config, depth), config, 1)
        t0 = time.perf_counter()
        if PHASE_TIMES:
            (it, norms, conv), times = _traced(
                lambda: plan.solve_host(fh, uh, uh, [floor], config.eps, config.max_iters))
        else:
            it, norms, conv = plan.solve_host(fh, uh, uh, [floor], config.eps, config.max_iters)
            times = _times(time.perf_counter() - t0)
        k = int(it[0])
        hist = [float(v) for v in norms[0, :k + 1]]
        return uh, SolveStats(iterations=k, residual_norms=hist, factor=max_ratio(hist),
                              times=times, converged=bool(conv[0]), seed=config.seed,
                              workers=config.workers)
    torch = _torch()
    fd, was_t = _dev_block(f, shape, "f")
    if depth < 2:
        u = _forward_solve_dev(hier.finest.ops, hier.finest.n_steps, fd, config)
        stats = SolveStats(iterations=0, residual_norms=[0.0], factor=float("nan"),
                           times=_times(0.0), converged=True, seed=config.seed,
                           workers=config.workers)
        return _out(u, was_t), stats
    ud, _ = _dev_block(u_init, shape, "u_init")
    if torch.is_tensor(u_init) and ud.data_ptr() == u_init.data_ptr():
        ud = ud.clone()
    floor = _floor_of(f if torch.is_tensor(f) else _to_numpy(f))
    omegas = omegas_for(hier, config, depth)
    plan = get_plan(hier, 0, depth, omegas, config, 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if PHASE_TIMES:
        (it, norms, conv), times = _traced(lambda: plan.solve(fd, ud, [floor], config.eps, config.max_iters))
    else:
        it, norms, conv = plan.solve(fd, ud, [floor], config.eps, config.max_iters)
        times = _times(time.perf_counter() - t0)
    k = int(it[0])
    hist = [float(v) for v in norms[0, :k + 1]]
    stats = SolveStats(iterations=k, residual_norms=hist, factor=max_ratio(hist),
                       times=times, converged=bool(conv[0]), seed=config.seed,
                       workers=config.workers)
    return _out(ud, was_t), stats


def solve_batched(hier, F, U0=None, config: CycleConfig = None, floors=None, inplace=False):
    """B independent problems sharing hier's operator: F, U0 of shape
    (B, N, n_t).  Each problem follows the reference stopping rule on its own
    (exactly as B separate ``solve`` calls).  Returns (U, [SolveStats]).
    ``inplace=True`` (device tensors only) overwrites U0 with the solution."""
    config = config or CycleConfig()
    depth = depth_of(hier, config)
    if depth < 2:
        raise ValueError("solve_batched needs at least 2 levels")
    N, nt = hier.finest.n_steps, hier.finest.ops.n_t
    if len(getattr(F, "shape", ())) != 3 or tuple(F.shape[1:]) != (N, nt):
        raise ValueError(f"F must have shape (B, {N}, {nt}), got {tuple(getattr(F, 'shape', ()))}")
    B = int(F.shape[0])
    shape = (B, N, nt)
    if B < 1:
        raise ValueError("solve_batched needs at least one problem")
    if not _is_torch_cuda(F):
        # host buffers (numpy / CPU torch, ideally pinned): copies inside the C ABI
        _check_device()
        Fh = _host_block(F, shape, "F", copy=False)
        if U0 is None:
            Uin, Uh = None, np.empty(shape)
        else:
            host_u0 = _is_host(U0) and tuple(U0.shape) == shape
            Uh = _host_block(U0, shape, "U0", copy=not (inplace and host_u0))
            Uin = Uh
        if floors is None:
            floors = [1e-12 * float(np.linalg.norm(np.asarray(Fh[b], dtype=np.float64)))
                      for b in range(B)]
        floors = _check_floors(floors, B)
        plan = get_plan(hier, 0, depth, omegas_for(hier, config, depth), config, B)
        t0 = time.perf_counter()
        it, norms, conv = plan.solve_host(Fh, Uin, Uh, floors, config.eps, config.max_iters)
        elapsed = time.perf_counter() - t0
        return Uh, _batched_stats(it, norms, conv, elapsed, config)
    torch = _torch()
    Fd, was_t = _dev_block(F, shape, "F")
    if U0 is None:
        Ud = torch.zeros_like(Fd)
    else:
        Ud, _ = _dev_block(U0, shape, "U0")
        if not (inplace and torch.is_tensor(U0) and Ud.data_ptr() == U0.data_ptr()):
            Ud = Ud.clone()
    if floors is None:
        floors = [1e-12 * float(v) for v in torch.linalg.norm(Fd.reshape(B, -1), dim=1).cpu()]
    floors = _check_floors(floors, B)
    omegas = omegas_for(hier, config, depth)
    plan = get_plan(hier, 0, depth, omegas, config, B)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    it, norms, conv = plan.solve(Fd, Ud, floors, config.eps, config.max_iters)
    elapsed = time.perf_counter() - t0
    return _out(Ud, was_t), _batched_stats(it, norms, conv, elapsed, config)


def _stream_split(B: int) -> int:
    """Sub-batches per batch in solve_batched_stream: the pipeline's fill (first
    copy-in) and drain (last copy-out) are one sub-batch long, so finer is
    better until the per-solve latency of the small levels shows.  B = 64 x 2^22,
    time-DoF/s at 5 / 10 batches per call: split 1: 6.6e10 / 7.4e10, 2: 7.4e10 /
    7.8e10, 4: 7.6e10 / 7.6e10, 8: 7.2e10 / 7.4e10 -- halves are the default
    (TMG_STREAM_SPLIT overrides)."""
    env = os.environ.get("TMG_STREAM_SPLIT", "")
    if env:
        s = max(1, int(env))
        return s if B % s == 0 else 1
    return 2 if B % 2 == 0 and B // 2 >= 16 else 1


def solve_batched_stream(hier, F_batches, U_outs=None, config: CycleConfig = None, floors=None):
    """Many independent batches (host arrays (B, N, n_t), ideally pinned), each
    solved from the zero guess exactly like ``solve_batched``, with the PCIe
    copies of neighbouring (sub-)batches overlapping each solve.  Returns
    (U_outs, [[SolveStats] per batch])."""
    config = config or CycleConfig()
    depth = depth_of(hier, config)
    if depth < 2:
        raise ValueError("solve_batched_stream needs at least 2 levels")
    N, nt = hier.finest.n_steps, hier.finest.ops.n_t
    F_batches = list(F_batches)
    if not F_batches:
        raise ValueError("no batches")
    B = int(F_batches[0].shape[0])
    shape = (B, N, nt)
    for F in F_batches:
        if not _is_host(F) or tuple(F.shape) != shape:
            raise ValueError(f"every batch must be a host array of shape {shape}")
    Fh = [_host_array(F, copy=False) for F in F_batches]
    if U_outs is None:
        U_outs = [np.empty(shape) for _ in Fh]
    elif len(U_outs) != len(Fh) or any(not _is_host(U) or tuple(U.shape) != shape for U in U_outs):
        raise ValueError(f"U_outs must be {len(Fh)} host arrays of shape {shape}")
    if floors is None:
        floors = [[1e-12 * float(np.linalg.norm(np.asarray(F[b], dtype=np.float64))) for b in range(B)]
                  for F in Fh]
    _check_device()
    split = _stream_split(B)
    Bs = B // split
    if split > 1:
        # problems are independent: a batch is `split` consecutive sub-batches
        # (contiguous views of the same host arrays) in the same pipeline
        Fs = [F[i * Bs:(i + 1) * Bs] for F in Fh for i in range(split)]
        Us = [U[i * Bs:(i + 1) * Bs] for U in U_outs for i in range(split)]
        fl = [list(fb[i * Bs:(i + 1) * Bs]) for fb in floors for i in range(split)]
    else:
        Fs, Us, fl = Fh, U_outs, floors
    plan = get_plan(hier, 0, depth, omegas_for(hier, config, depth), config, Bs)
    t0 = time.perf_counter()
    res = plan.solve_host_stream(Fs, Us, fl, config.eps, config.max_iters)
    elapsed = time.perf_counter() - t0
    if split > 1:
        res = [tuple(np.concatenate([res[k * split + i][j] for i in range(split)]) for j in range(3))
               for k in range(len(Fh))]
    return U_outs, [_batched_stats(it, norms, conv, elapsed / len(Fh), config) for it, norms, conv in res]


def _batched_stats(it, norms, conv, elapsed, config):
    stats = []
    for b in range(len(it)):
        k = int(it[b])
        hist = [float(v) for v in norms[b, :k + 1]]
        stats.append(SolveStats(iterations=k, residual_norms=hist, factor=max_ratio(hist),
                                times=_times(elapsed), converged=bool(conv[b]), seed=config.seed,
                                workers=config.workers))
    return stats


def measure_convergence_factor(hier, config: CycleConfig = None) -> float:
    """Two-grid factor on f = 0 from the seeded random start
    (multigrid.py:534-544)."""
    config = config or CycleConfig(eps=1e-100)
    if len(hier.levels) < 2:
        raise ValueError("measuring the two-grid factor needs 2 levels")
    n, nt = hier.finest.n_steps, hier.finest.ops.n_t
    f = np.zeros((n, nt))
    torch = _torch()
    fd, _ = _dev(f)
    ud, _ = _dev(random_initial_guess(hier, config.seed))
    omegas = omegas_for(hier, config, 2)
    plan = get_plan(hier, 0, 2, omegas, config, 1)
    it, norms, conv = plan.solve(fd, ud, [0.0], config.eps, min(config.max_iters, 250))
    k = int(it[0])
    return max_ratio([float(v) for v in norms[0, :k + 1]])


def measure_convergence_factors(basis, taus, nu=1, n_steps: int = 1024, damping="optimal",
                                seed: int = 42, eps: float = 1e-100, max_iters: int = 250):
    """Two-grid convergence factors for many step sizes in ONE launch:
    factor[i] == measure_convergence_factor(TimeHierarchy.build(basis, taus[i],
    n_steps, n_levels=2), CycleConfig(nu1=nu, nu2=nu, damping=damping,
    eps=eps, seed=seed, max_iters=max_iters)) bit for bit (multigrid.py:534-544;
    the paper's measured-vs-predicted experiment, tests/test_acceptance.py:45-59).
    Each problem carries its own operator; one CTA per problem."""
    from .hierarchy import TimeHierarchy
    taus = list(taus)
    cfg = CycleConfig(nu1=nu, nu2=nu, damping=damping, eps=eps, seed=seed, max_iters=max_iters)
    hiers = [TimeHierarchy.build(basis, float(t), n_steps, n_levels=2) for t in taus]
    multi = [(h, omegas_for(h, cfg, 2)) for h in hiers]
    plan = DevicePlan(hiers[0], 0, 2, multi[0][1], cfg, len(hiers), multi=multi)
    u0 = random_initial_guess(hiers[0], seed)
    U = np.ascontiguousarray(np.broadcast_to(u0, (len(hiers),) + u0.shape))
    F = np.zeros_like(U)
    _check_device()
    it, norms, conv = plan.solve_host(F, U, U, np.zeros(len(hiers)), eps, min(max_iters, 250))
    return [max_ratio([float(v) for v in norms[b, :int(it[b]) + 1]]) for b in range(len(hiers))]
