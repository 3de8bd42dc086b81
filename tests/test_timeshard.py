"""Time-axis sharding of one problem (paper_1409_5254_b200.timeshard).

CPU (gloo, world sizes 2 and 4): the sharded host logic -- halo shifts, the
gathered tail, the rank-order norm combination -- driven by a test-only
slab-ops object built on the oracle, compared bit for bit with the oracle's
single-process ``_iterate``.  GPU: the same driver on the sm_100a kernels with
R ranks emulated by threads on one device (host-orchestrated; no kernel waits
on another), compared bit for bit with the single-device ``solve``.
"""

import os
import socket
import threading

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import paper_1409_5254_b200 as tmg
from paper_1409_5254_b200 import problems, timeshard as ts


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleSlabOps:
    """Test double of CudaSlabOps on CPU torch tensors, computed by the oracle
    (the checker) -- exercises only the sharding logic around the kernels."""

    def __init__(self, hier, omegas, nu1, nu2, depth):
        from oracle import oracle as O
        self.O, self.hier, self.om, self.nu, self.depth = O, hier, omegas, (nu1, nu2), depth

    def zeros(self, n, nt):
        return torch.zeros((n, nt), dtype=torch.float64)

    def upload(self, x):
        return torch.from_numpy(np.array(x, dtype=np.float64))

    def download(self, t):
        return t.numpy()

    def down(self, l, f, u_in, u_out, fc, nu, active=None):
        if active is not None and not bool(active):
            return  # the solve has stopped: queued cycles are no-ops
        lev = self.hier.levels[l]
        u = np.zeros(tuple(f.shape)) if u_in is None else u_in.numpy()
        uo, fco = self.O.down_pass(lev.ops, lev.r1, lev.r2, self.om[l], u, f.numpy(), nu)
        u_out[:] = torch.from_numpy(uo)
        fc[:] = torch.from_numpy(fco)

    def up(self, l, f, u_in, uc, u_out, nu, active=None):
        if active is not None and not bool(active):
            return
        lev = self.hier.levels[l]
        x = self.O.prolong_add(lev.ops, lev.r1, lev.r2, uc.numpy()[: f.shape[0] // 2], u_in.numpy())
        u_out[:] = torch.from_numpy(self.O.block_jacobi(lev.ops, x, f.numpy(), self.om[l], nu))

    def resid_sqsum(self, f, u, skip):
        r = self.O.residual(self.hier.levels[0].ops, f.numpy(), u.numpy())
        sq = r[:, 0] * r[:, 0]
        for j in range(1, r.shape[1]):
            sq = sq + r[:, j] * r[:, j]
        return float(np.sum(sq[skip:]))

    def tail_cycle(self, level, f_full):
        u = self.O.cycle(self.hier, self.om, np.zeros(tuple(f_full.shape)), f_full.numpy(), *self.nu,
                         depth=self.depth - level, level=level)
        return torch.from_numpy(u)


def _case(p_t, n, nu, seed=3):
    T = 1.0
    a, phi, u0 = problems.forcing_params(seed)
    basis = tmg.BasisSpec(p_t)
    rhs = tmg.rhs_moments(problems.make_forcing(a, phi, T), basis, T / n, n, u0=u0)
    hier = tmg.TimeHierarchy.build(basis, T / n, n, coarsest=2)
    cfg = tmg.CycleConfig(nu1=nu, nu2=nu, eps=1e-8)
    return hier, rhs, cfg


def _gloo_worker(rank, world, port, p_t, n, nu, min_local, out, max_iters=250):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    hier, rhs, cfg = _case(p_t, n, nu)
    cfg.max_iters = max_iters
    depth = len(hier.levels)
    om = [tmg.optimal_omega(tmg.alpha(hier.basis, l.tau)) for l in hier.levels]
    ops = OracleSlabOps(hier, om, nu, nu, depth)
    s = ts.TimeShardedSolver(hier, cfg, ts.DistComm(), ops, halo=64, min_local=min_local)
    u, st = s.solve(rhs, np.zeros_like(rhs), check_every=3)
    out[rank] = (u.tobytes(), st.residual_norms, st.iterations, s.layout.gather_level)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,p_t,n,nu,min_local", [(2, 1, 1 << 13, 1, 256), (4, 2, 1 << 13, 2, 128)])
def test_gloo_time_sharded_solve_bitwise(oracle_mod, world, p_t, n, nu, min_local):
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_gloo_worker, args=(world, port, p_t, n, nu, min_local, out), nprocs=world, join=True)
        res = dict(out)
    hier, rhs, cfg = _case(p_t, n, nu)
    om = [tmg.optimal_omega(tmg.alpha(hier.basis, l.tau)) for l in hier.levels]
    ur, norms, iters = oracle_mod.iterate(hier, om, rhs, np.zeros_like(rhs), nu, nu, 1e-8, 250)
    assert res[0][3] >= 2  # at least two sharded levels
    for r in range(world):
        ub, nr, it, _ = res[r]
        assert it == iters
        assert nr == norms
        assert ub == ur.tobytes()


def test_gloo_time_sharded_max_iters_mid_batch(oracle_mod):
    """max_iters reached inside a batch of queued cycles: the device flag
    turns the rest into no-ops; result = the oracle's 3-cycle iterate."""
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_gloo_worker, args=(2, port, 1, 1 << 13, 1, 256, out, 3), nprocs=2, join=True)
        res = dict(out)
    hier, rhs, cfg = _case(1, 1 << 13, 1)
    om = [tmg.optimal_omega(tmg.alpha(hier.basis, l.tau)) for l in hier.levels]
    ur, norms, iters = oracle_mod.iterate(hier, om, rhs, np.zeros_like(rhs), 1, 1, 1e-8, 3)
    assert iters == 3
    for r in range(2):
        ub, nr, it, _ = res[r]
        assert it == 3 and nr == norms and ub == ur.tobytes()


def test_pairwise_structure():
    rng = np.random.default_rng(0)
    for n, R in ((1 << 13, 2), (1 << 13, 4), (1 << 16, 8), (3 << 12, 2)):
        x = rng.random(n)
        m = n // R
        nodes = ts.pairwise_nodes(n)
        if all((r * m, m) in nodes for r in range(R)):
            parts = [float(np.sum(x[r * m:(r + 1) * m])) for r in range(R)]
            assert ts.combine_pairwise(parts) == float(np.sum(x))
    # 1000 slabs over 2 ranks: numpy splits at 496, not 500
    assert (0, 500) not in ts.pairwise_nodes(1000) and (0, 496) in ts.pairwise_nodes(1000)


def test_layout_validation():
    lay = ts.ShardLayout([1 << 14 >> k for k in range(13)], 4, 64, 256)
    assert lay.gather_level == 5 and lay.local[:5] == [4096, 2048, 1024, 512, 256]
    with pytest.raises(ValueError):
        ts.ShardLayout([1 << 14 >> k for k in range(13)], 3)       # not a power of two
    with pytest.raises(ValueError):
        ts.ShardLayout([1 << 14 >> k for k in range(13)], 2, halo=63)
    with pytest.raises(ValueError):
        ts.ShardLayout([1 << 10 >> k for k in range(9)], 4, 64, 4096)  # too small to split
    with pytest.raises(ValueError):
        ts.ShardLayout([96, 48, 24], 2, 2, 8)  # ranges not pairwise blocks


# --------------------------------------------------------------------------- GPU


class ThreadComm:
    """R ranks as threads on one GPU (host-orchestrated exchanges)."""

    def __init__(self, rank, world, shared):
        self.rank, self.world, self.sh = rank, world, shared

    def shift(self, tail, halo):
        sh = self.sh
        if self.rank + 1 < self.world:
            sh["box"][self.rank + 1].put(tail.clone())
        if self.rank > 0:
            halo.copy_(sh["box"][self.rank].get())

    def _exchange(self, x):
        sh = self.sh
        sh["slots"][self.rank] = x
        sh["bar"].wait()
        vals = list(sh["slots"])
        sh["bar"].wait()
        return vals

    def all_gather_rows(self, local):
        return torch.cat(self._exchange(local.clone()))

    def all_gather_value(self, x):
        return [v.reshape(1) for v in self._exchange(x)]


@pytest.mark.gpu
@pytest.mark.parametrize("world,p_t,n,nu", [(2, 1, 1 << 16, 1), (4, 3, 1 << 16, 2), (8, 1, 1 << 18, 1)])
def test_gpu_time_sharded_solve_bitwise(world, p_t, n, nu):
    import queue
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    hier, rhs, cfg = _case(p_t, n, nu)
    u_ref, st_ref = tmg.solve(hier, rhs, np.zeros_like(rhs), cfg)
    sh = {"box": [queue.Queue() for _ in range(world)], "slots": [None] * world,
          "bar": threading.Barrier(world)}
    res, errs = {}, []

    def run(r):
        try:
            torch.cuda.set_device(0)
            s = ts.TimeShardedSolver(hier, cfg, ThreadComm(r, world, sh), halo=64, min_local=2048)
            res[r] = s.solve(rhs, np.zeros_like(rhs)) + (s.layout.gather_level,)
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)
            sh["bar"].abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    assert not errs, errs
    for r in range(world):
        u, st, g = res[r]
        assert g >= 2
        assert st.iterations == st_ref.iterations
        assert st.residual_norms == st_ref.residual_norms
        assert u.tobytes() == u_ref.tobytes()
