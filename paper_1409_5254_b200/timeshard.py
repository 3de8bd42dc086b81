"""Time-axis sharding of ONE problem across ranks.

The reference parallelises a solve by giving every worker thread a contiguous,
even-aligned slab range per level (``_make_slab_table``, multigrid.py:382-415)
and letting worker 0 run the levels too short to split (``_cycle``'s ``None``
levels, :291-305); its worker count never changes the iterates
(test_multigrid.py:241-259).  Here ranks (one process per GPU) take the
workers' place:

* level l is *sharded* while every rank's range has at least ``min_local``
  slabs; rank g owns slabs [g m_l, (g+1) m_l) with m_l = N_l / R even, so
  restriction pairs and prolongation never straddle two ranks;
* a rank's level buffers hold a left halo of H slabs (the left neighbour's last
  H slabs) in front of its own range.  Jacobi couples slab n to slab n-1 only
  (``N = outer(eval_start, eval_end)``, dg.py:231-236), so after k sweeps of a
  buffer whose first slab has no predecessor every slab >= k is exact: with
  H >= nu + 1 the fused down pass (nu1 sweeps + residual + restriction) and up
  pass (prolong-add + nu2 sweeps) of the whole buffer give the rank's own slabs
  bit for bit.  The exchange step per pass is one halo shift (rank g sends its
  last H slabs to g+1): f and the pre-smoothed u before the up pass, the
  corrected u after it (the next level up reads it as u_coarse);
* the first level that is not sharded is all-gathered; every rank runs the rest
  of the V-cycle there (the same deterministic kernels, so the same bits) and
  keeps its own range plus halo of the result;
* the stopping norm (``norm_at``, :447-462): each rank sums its slabs' squared
  residual norms in numpy's pairwise order (``tmg_resid_sqsum``); with R a
  power of two every rank's range is a node of np.sum's recursion, so adding
  the R partial sums in the recursion's own tree reproduces the single-device
  norm exactly -- and with it every stopping decision.

Result: iterates, residual histories and iteration counts identical to
``solve`` on one device (and to the reference).  The per-rank work is 1/R of
the sharded levels; the exchanges are latency-bound (a few KB per pass), so
sharding pays from ~2^24 slabs per rank.

The compute goes through a *slab-ops* object (``CudaSlabOps``: the C ABI on the
rank's GPU); the communication through a *comm* object (``DistComm``:
torch.distributed P2P + all_gather -- NCCL over NVLink for CUDA tensors, gloo
for CPU tensors).  Both are plain duck-typed interfaces so the host logic is
testable on CPU (tests/test_timeshard.py).
"""

from __future__ import annotations

import ctypes
import math
import time

import numpy as np

from . import _native as nat
from .hierarchy import CycleConfig, SolveStats, depth_of, max_ratio

HALO = 64


# ---------------------------------------------------------------------------
# numpy pairwise-summation structure (np.add.reduce of a contiguous vector)


def pairwise_nodes(n: int, lo: int = 0) -> set:
    """(offset, length) of every node of numpy's pairwise recursion over n
    values: blocks > 128 split at n2 = n/2 rounded down to a multiple of 8."""
    out = {(lo, n)}
    if n > 128:
        n2 = n // 2
        n2 -= n2 % 8
        out |= pairwise_nodes(n2, lo)
        out |= pairwise_nodes(n - n2, lo + n2)
    return out


def combine_pairwise(parts):
    """Add rank partial sums in the recursion's tree: (left half) + (right half)."""
    if len(parts) == 1:
        return parts[0]
    h = len(parts) // 2
    return combine_pairwise(parts[:h]) + combine_pairwise(parts[h:])


class ShardLayout:
    """Which levels are sharded and how many slabs each rank owns."""

    def __init__(self, n_slabs, world: int, halo: int = HALO, min_local: int = 4096, nu: int = 1):
        if world < 1 or world & (world - 1):
            raise ValueError(f"time sharding needs a power-of-two world size, got {world}")
        if halo < 2 or halo % 2 or halo < nu + 1:
            raise ValueError(f"halo must be even and >= nu + 1 = {nu + 1}, got {halo}")
        self.world = world
        self.halo = halo
        n_slabs = list(n_slabs)
        depth = len(n_slabs)
        g = 0
        while g < depth - 2:  # keep >= 2 levels for the gathered tail
            n = n_slabs[g]
            if n % (2 * world) or n // world < max(min_local, halo):
                break
            g += 1
        if g == 0:
            raise ValueError(f"{n_slabs[0]} slabs cannot be split over {world} ranks "
                             f"(need N/R >= {max(min_local, halo)} and N % 2R == 0)")
        self.gather_level = g
        self.n = n_slabs
        self.local = [n_slabs[l] // world for l in range(g + 1)]
        # the finest level's ranges must be nodes of np.sum's recursion
        nodes = pairwise_nodes(n_slabs[0])
        m = self.local[0]
        if world > 1 and any((r * m, m) not in nodes for r in range(world)):
            raise ValueError(f"rank ranges of {m} slabs are not pairwise-summation blocks of "
                             f"{n_slabs[0]}; the stopping norm would differ from one device")


# ---------------------------------------------------------------------------
# communication


class DistComm:
    """torch.distributed: NCCL (CUDA tensors, NVLink P2P) or gloo (CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"

    def _peer(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def shift(self, tail, halo):
        """Send ``tail`` to rank+1, receive rank-1's into ``halo`` (in place)."""
        d = self.dist
        ops = []
        if self.rank + 1 < self.world:
            ops.append(d.P2POp(d.isend, tail.contiguous(), self._peer(self.rank + 1), self.group))
        if self.rank > 0:
            ops.append(d.P2POp(d.irecv, halo, self._peer(self.rank - 1), self.group))
        if ops:
            for r in d.batch_isend_irecv(ops):
                r.wait()

    def all_gather_rows(self, local):
        import torch
        bufs = [torch.empty_like(local) for _ in range(self.world)]
        self.dist.all_gather(bufs, local.contiguous(), group=self.group)
        return torch.cat(bufs)

    def all_gather_value(self, x):
        """Every rank's scalar (a 1-element float64 tensor on this rank's
        device, or a float), as a list of 1-element tensors -- no host sync
        for device tensors (NCCL all_gather on the stream)."""
        import torch
        t = x if torch.is_tensor(x) else torch.tensor([float(x)], dtype=torch.float64)
        t = t.reshape(1).to(device=self.device, dtype=torch.float64)
        bufs = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(bufs, t, group=self.group)
        return bufs


# ---------------------------------------------------------------------------
# compute: the C ABI on this rank's GPU


class CudaSlabOps:
    """Fused level passes of the sm_100a kernels on buffer views (torch CUDA)."""

    def __init__(self, hier, omegas, config: CycleConfig, depth: int):
        from .solver import _torch
        self.torch = _torch()
        self.hier = hier
        self.omegas = omegas
        self.config = config
        self.depth = depth
        self.lib = nat.load()

    def _desc(self, l, n):
        lev = self.hier.levels[l]
        return nat.level_desc(lev.ops, n, self.omegas[l], lev.r1, lev.r2)

    def _s(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream().cuda_stream)

    @staticmethod
    def _p(t):
        return None if t is None else ctypes.c_void_p(t.data_ptr())

    def zeros(self, n, nt):
        return self.torch.zeros((n, nt), dtype=self.torch.float64, device="cuda")

    def upload(self, x):
        return self.torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to("cuda")

    def download(self, t):
        return t.cpu().numpy()

    def active_flag(self):
        """The device stopping mask the passes honour (int32, 1 = keep going)."""
        return self.torch.ones(1, dtype=self.torch.int32, device="cuda")

    def down(self, l, f, u_in, u_out, fc, nu, active=None):
        d = self._desc(l, f.shape[0])
        nat.check(self.lib.tmg_down(nat.F64, ctypes.byref(d), self._p(f), self._p(u_in), self._p(u_out),
                                    self._p(fc), 1, int(nu), self._p(active), self._s()), "tmg_down")

    def up(self, l, f, u_in, uc, u_out, nu, active=None):
        d = self._desc(l, f.shape[0])
        nat.check(self.lib.tmg_up(nat.F64, ctypes.byref(d), self._p(f), self._p(u_in), self._p(uc),
                                  self._p(u_out), None, 1, int(nu), self._p(active), self._s()), "tmg_up")

    def resid_sqsum(self, f, u, skip):
        """This rank's numpy-order share of the squared norm: a 1-element
        device tensor (stream-ordered, no host sync)."""
        d = self._desc(0, f.shape[0])
        out = self.torch.empty(1, dtype=self.torch.float64, device="cuda")
        nat.check(self.lib.tmg_resid_sqsum(nat.F64, ctypes.byref(d), self._p(f), self._p(u), int(skip),
                                           self._p(out), 1, self._s()), "tmg_resid_sqsum")
        return out

    def tail_cycle(self, level, f_full):
        """V-cycle from ``level`` down with a zero initial guess (every rank
        runs it on the gathered right-hand side).  The plan is this object's
        own: plans keep per-level scratch, so they are never shared between
        concurrent solvers."""
        from .solver import DevicePlan
        if getattr(self, "_tail", None) is None or self._tail[0] != level:
            self._tail = (level, DevicePlan(self.hier, level, self.depth - level,
                                            self.omegas[level:self.depth], self.config, 1))
        u = self.torch.zeros_like(f_full)
        self._tail[1].cycles(f_full, u, 1)
        return u


# ---------------------------------------------------------------------------
# the sharded solver


class TimeShardedSolver:
    """``solve`` (multigrid.py:509-531) for one problem sharded along time.

    Every rank calls ``solve`` with the same full right-hand side (host array)
    and gets the full solution back; ranks hold only their range plus halo of
    each level on the device.  V-cycles only (the reference's cycle)."""

    def __init__(self, hier, config: CycleConfig = None, comm=None, ops=None, halo: int = HALO,
                 min_local: int = 4096):
        config = config or CycleConfig()
        if config.cycle != "V":
            raise ValueError("time sharding runs V-cycles (the reference's cycle)")
        self.hier = hier
        self.config = config
        self.depth = depth_of(hier, config)
        if self.depth < 2:
            raise ValueError("time sharding needs a hierarchy with at least 2 levels")
        self.comm = comm if comm is not None else DistComm()
        from .hierarchy import level_omegas
        self.omegas = level_omegas(hier, config, self.depth)
        self.ops = ops if ops is not None else CudaSlabOps(hier, self.omegas, config, self.depth)
        self.layout = ShardLayout([lev.n_steps for lev in hier.levels[:self.depth]], self.comm.world,
                                  halo, min_local, max(config.nu1, config.nu2))
        self.H = halo
        self.nt = hier.levels[0].ops.n_t
        G = self.layout.gather_level
        o = self.ops
        # level buffers [H halo | own range]: f, iterate/correction u, pre-smoothed p
        self.F = [o.zeros(halo + self.layout.local[l], self.nt) for l in range(G + 1)]
        self.U = [o.zeros(halo + self.layout.local[l], self.nt) for l in range(G + 1)]
        self.P = [o.zeros(halo + self.layout.local[l], self.nt) for l in range(G)]

    # views of a level buffer for the kernels: rank 0 has no left neighbour, so
    # its passes start at its own slab 0 (the true problem start)
    def _own(self, buf):
        return buf[self.H:] if self.comm.rank == 0 else buf

    def _coarse_out(self, buf):
        # fine buffer slab H maps to coarse buffer slab H: rank 0's buffer starts
        # at H, the others' restriction of the halo lands in the coarse halo
        return buf[self.H:] if self.comm.rank == 0 else buf[self.H // 2:]

    def _shift(self, buf):
        self.comm.shift(buf[-self.H:], buf[:self.H])

    def _cycle(self, l, active=None):
        c, o, H = self.config, self.ops, self.H
        G = self.layout.gather_level
        zero = l > 0
        o.down(l, self._own(self.F[l]), None if zero else self._own(self.U[l]), self._own(self.P[l]),
               self._coarse_out(self.F[l + 1]), c.nu1, active=active)
        self._shift(self.P[l])
        if l + 1 < G:
            self._shift(self.F[l + 1])
            self._cycle(l + 1, active)
        else:
            m, g = self.layout.local[G], self.comm.rank
            f_full = self.comm.all_gather_rows(self.F[G][H:])
            u_full = o.tail_cycle(G, f_full)
            self.U[G][H:] = u_full[g * m:(g + 1) * m]
            if g > 0:
                self.U[G][:H] = u_full[g * m - H:g * m]
        o.up(l, self._own(self.F[l]), self._own(self.P[l]), self._coarse_out(self.U[l + 1]),
             self._own(self.U[l]), c.nu2, active=active)
        self._shift(self.U[l])

    def _norm(self):
        """||f - L u|| of the whole problem as a 1-element tensor on the
        comm's device: the ranks' numpy-order partial sums, combined in the
        recursion's own tree (bitwise the single-device np.sum), IEEE sqrt --
        all on the device, no host sync."""
        import torch
        skip = 0 if self.comm.rank == 0 else self.H
        s = self.ops.resid_sqsum(self._own(self.F[0]), self._own(self.U[0]), skip)
        return torch.sqrt(combine_pairwise(self.comm.all_gather_value(s)))

    def solve(self, f, u_init=None, check_every: int = 4):
        """(u, SolveStats) with the stopping rule of _iterate (multigrid.py:427-500).

        The stopping test runs on the device: every cycle updates a device
        flag active = (r_k > tol) & (k < max_iters) that the level passes
        honour (a finished solve's remaining queued cycles are no-ops), and the
        host looks at it once per ``check_every`` cycles -- no host round trip
        per cycle.  Iterates, norms and counts equal the per-cycle test's."""
        import torch
        c, H = self.config, self.H
        f = np.ascontiguousarray(f, dtype=np.float64)
        N = self.layout.n[0]
        if f.shape != (N, self.nt):
            raise ValueError(f"f has shape {f.shape}, expected {(N, self.nt)}")
        if u_init is None:
            from .solver import random_initial_guess
            u_init = random_initial_guess(self.hier, c.seed)
        u_init = np.ascontiguousarray(u_init, dtype=np.float64)
        g, m = self.comm.rank, self.layout.local[0]
        lo = g * m - H if g > 0 else 0
        pad = H if g == 0 else 0
        self.F[0][pad:] = self.ops.upload(f[lo:(g + 1) * m])
        self.U[0][pad:] = self.ops.upload(u_init[lo:(g + 1) * m])
        floor = 1e-12 * float(np.linalg.norm(f))
        t0 = time.perf_counter()
        r0 = self._norm()
        dev = r0.device
        tol = torch.maximum(r0 * c.eps, torch.tensor([floor], dtype=torch.float64, device=dev))
        hist = [r0]
        iters_t = torch.zeros(1, dtype=torch.int32, device=dev)
        active = r0 > tol
        act = self.ops.active_flag() if hasattr(self.ops, "active_flag") else None
        queued = 0
        while queued < c.max_iters:
            for _ in range(max(1, int(check_every))):
                if queued >= c.max_iters:
                    break
                if act is not None:
                    act.copy_(active.to(act.dtype).to(act.device))
                self._cycle(0, act if act is not None else active)
                rk = self._norm()
                hist.append(rk)
                iters_t = iters_t + active.to(torch.int32)
                active = active & (rk > tol) & (iters_t < c.max_iters)
                queued += 1
            if not bool(active.item()):
                break
        iters = int(iters_t.item())
        norms = [float(v) for v in torch.cat(hist[:iters + 1]).cpu()]
        u = self.comm.all_gather_rows(self.U[0][H:])
        elapsed = time.perf_counter() - t0
        stats = SolveStats(iterations=iters, residual_norms=norms, factor=max_ratio(norms),
                           times={"smoothing": elapsed, "transfer": 0.0, "coarse": 0.0, "residual": 0.0},
                           converged=norms[-1] <= max(c.eps * norms[0], floor), seed=c.seed,
                           workers=self.comm.world)
        return self.ops.download(u), stats


def solve_time_sharded(hier, f, u_init=None, config: CycleConfig = None, group=None, **kw):
    """One problem, sharded along time over the ranks of ``group`` (torch.distributed
    initialised with NCCL, one process per GPU).  Same results as ``solve``."""
    return TimeShardedSolver(hier, config, DistComm(group), **kw).solve(f, u_init)
