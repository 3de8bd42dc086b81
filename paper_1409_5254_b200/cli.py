"""Command line for the GPU time-multigrid solver: ``solve`` and ``bench``.

Usage contract shared with the reference's ``timemg`` command
(pkg/src/timemg/cli.py): the ``solve`` flags and their defaults, the layering
"built-in defaults < JSON config file (--config) < explicit flags" with
unknown config keys rejected, the output files (solve_solution.{csv,json},
solve_stats.json, solve_residuals.csv) and the exit codes 0 (ok), 2 (usage
error) and 3 (no convergence within max_iters).  The analysis subcommands
(analyze, verify) are out of scope.

``bench`` is the GPU counterpart of the reference's scaling harness
(pkg/src/timemg/bench.py:77-137): every point solves the reference's bench
problem (f = 0, the seeded random initial guess, default coarsest level),
repeats it ``--reps`` times and reports the median.  Its "workers" are GPUs:
one rank of the time-sharded solver per GPU (timeshard.py) when run under
torchrun, the fused single-GPU plan for one worker.  Rows carry the reference's
fields (mode, workers, steps, p_t, median_time, scaled, iterations, samples)
plus time-DoF/s.
"""

from __future__ import annotations

import argparse
import csv
import dataclasses
import json
import os
import statistics
import sys
import time

import numpy as np

from .hierarchy import CYCLES

EXIT_OK, EXIT_USAGE, EXIT_NOT_CONVERGED = 0, 2, 3


class UsageError(Exception):
    """Bad flags or configuration (exit code 2)."""


@dataclasses.dataclass(frozen=True)
class Opt:
    """One option of a subcommand: flag spelling, config key, parser, default."""
    flag: str
    key: str
    kind: object
    default: object
    help: str = ""
    choices: tuple = ()


def _omega_value(text):
    if text == "optimal":
        return "optimal"
    try:
        return float(text)
    except (TypeError, ValueError):
        raise argparse.ArgumentTypeError(f"--omega takes 'optimal' or a number, not {text!r}")


def _int_list(text):
    if isinstance(text, (list, tuple)):
        return [int(v) for v in text]
    return [int(tok) for tok in str(text).replace(" ", "").split(",") if tok]


SOLVE_OPTS = (
    Opt("--pt", "pt", int, 0, "DG degree p_t (n_t = p_t + 1 DoFs per slab)"),
    Opt("--steps", "steps", int, 64, "number of time slabs N"),
    Opt("--T", "T", float, 1.0, "final time (tau = T / steps)"),
    Opt("--tau", "tau", float, None, "slab length (overrides --T)"),
    Opt("--u0", "u0", float, 1.0, "initial value u(0)"),
    Opt("--f", "f", str, "zero", "right-hand side preset", ("zero", "const", "poly", "sin")),
    Opt("--f-param", "f_param", float, 1.0, "preset parameter"),
    Opt("--nu1", "nu1", int, 2, "pre-smoothing sweeps"),
    Opt("--nu2", "nu2", int, 2, "post-smoothing sweeps"),
    Opt("--omega", "omega", _omega_value, "optimal", "damping: 'optimal' or a number"),
    Opt("--levels", "levels", str, "max", "hierarchy depth: 'max' or a count"),
    Opt("--eps", "eps", float, 1e-8, "relative residual reduction"),
    Opt("--seed", "seed", int, 42, "seed of the random initial guess"),
    Opt("--workers", "workers", int, 1, "accepted for compatibility (the GPU ignores it)"),
    Opt("--max-iters", "max_iters", int, 250, "cycle limit"),
    Opt("--cycle", "cycle", str, "V", "cycle type (GPU addition)", CYCLES),
)

BENCH_OPTS = (
    Opt("--mode", "mode", str, "strong", "strong: fixed problem; weak: fixed steps per worker",
        ("strong", "weak")),
    Opt("--workers", "workers", _int_list, [1], "GPU counts (powers of two, nondecreasing)"),
    Opt("--steps-per-worker", "steps_per_worker", int, 1 << 15, "weak mode: slabs per GPU"),
    Opt("--total-steps", "total_steps", int, 1 << 17, "strong mode: slabs of the problem"),
    Opt("--pt", "pt", _int_list, [0], "comma-separated DG degrees"),
    Opt("--tau", "tau", float, 1e-6, "slab length"),
    Opt("--eps", "eps", float, 1e-8, "relative residual reduction"),
    Opt("--reps", "reps", int, 3, "repetitions per point (median; >= 3)"),
    Opt("--seed", "seed", int, 42, "seed of the random initial guess"),
    Opt("--nu1", "nu1", int, 2, "pre-smoothing sweeps"),
    Opt("--nu2", "nu2", int, 2, "post-smoothing sweeps"),
)

COMMON_OPTS = (
    Opt("--out", "out", str, ".", "output directory"),
    Opt("--format", "format", str, "csv", "table format", ("csv", "json")),
)


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # never sys.exit from inside main()
        raise UsageError(message)


def build_parser() -> argparse.ArgumentParser:
    top = _Parser(prog="timemg-b200", description="GPU time-multigrid solver (B200)")
    subs = top.add_subparsers(dest="command")
    for name, opts, text in (("solve", SOLVE_OPTS, "solve u' + u = f on the GPU"),
                             ("bench", BENCH_OPTS, "GPU scaling study")):
        sp = subs.add_parser(name, help=text, argument_default=argparse.SUPPRESS)
        for o in opts + COMMON_OPTS:
            kw = {"dest": o.key, "type": o.kind, "help": o.help}
            if o.choices:
                kw["choices"] = o.choices
            sp.add_argument(o.flag, **kw)
        sp.add_argument("--config", dest="config", help="JSON file of option values")
        if name == "solve":
            sp.add_argument("--compare-sequential", dest="compare_sequential",
                            action="store_true",
                            help="also report the deviation from exact forward substitution")
            sp.add_argument("--time-shard", dest="time_shard", action="store_true",
                            help="shard the time axis over the torchrun ranks")
    return top


def settings(command: str, flags: dict) -> dict:
    """defaults < config file < explicit flags; unknown config keys are errors."""
    opts = {"solve": SOLVE_OPTS, "bench": BENCH_OPTS}[command] + COMMON_OPTS
    values = {o.key: o.default for o in opts}
    if command == "solve":
        values.update(compare_sequential=False, time_shard=False)
    path = flags.get("config")
    if path:
        with open(path) as fh:
            layer = json.load(fh)
        if not isinstance(layer, dict):
            raise UsageError(f"{path}: expected a JSON object")
        stray = sorted(set(layer) - set(values))
        if stray:
            raise UsageError(f"unknown config keys: {stray}")
        by_key = {o.key: o for o in opts}
        for k, v in layer.items():
            if k in by_key and isinstance(v, str) and by_key[k].kind not in (str,):
                v = by_key[k].kind(v)
            values[k] = v
    values.update({k: v for k, v in flags.items() if k not in ("config", "command")})
    return values


# ---------------------------------------------------------------------------
# output


def write_table(path: str, rows: list, fmt: str) -> None:
    if fmt == "json":
        with open(path, "w") as fh:
            json.dump(rows, fh, indent=2)
        return
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(list(rows[0]))
        for r in rows:
            w.writerow([r[k] for k in rows[0]])


def forcing(name: str, p: float):
    presets = {
        "zero": lambda t: 0.0 * t,
        "const": lambda t: np.full_like(t, p),
        "poly": lambda t: np.power(t, p),
        "sin": lambda t: np.sin(p * t),
    }
    if name not in presets:
        raise UsageError(f"unknown forcing {name!r}")
    return presets[name]


# ---------------------------------------------------------------------------
# solve


def run_solve(s: dict) -> int:
    import paper_1409_5254_b200 as tmg

    basis = tmg.BasisSpec(int(s["pt"]))
    n = int(s["steps"])
    tau = float(s["tau"]) if s["tau"] is not None else float(s["T"]) / n
    depth = s["levels"] if s["levels"] == "max" else int(s["levels"])
    hier = tmg.TimeHierarchy.build(basis, tau, n, n_levels=depth)
    cfg = tmg.CycleConfig(nu1=int(s["nu1"]), nu2=int(s["nu2"]), damping=s["omega"],
                          levels=depth, eps=float(s["eps"]), max_iters=int(s["max_iters"]),
                          seed=int(s["seed"]), workers=int(s["workers"]), cycle=s["cycle"])
    rhs = tmg.rhs_moments(forcing(s["f"], float(s["f_param"])), basis, tau, n, u0=float(s["u0"]))
    if s.get("time_shard"):
        from .timeshard import solve_time_sharded
        u, stats = solve_time_sharded(hier, rhs, None, cfg)
    else:
        u, stats = tmg.solve(hier, rhs, None, cfg)
    u = np.asarray(u)

    os.makedirs(s["out"], exist_ok=True)
    ends = u @ hier.finest.ops.eval_end
    table = []
    for k in range(n):
        row = {"step": k, "t_end": (k + 1) * tau, "u_end": float(ends[k])}
        row.update({f"c{i}": float(u[k, i]) for i in range(basis.n_t)})
        table.append(row)
    sol = os.path.join(s["out"], f"solve_solution.{s['format']}")
    write_table(sol, table, s["format"])
    st_path = os.path.join(s["out"], "solve_stats.json")
    with open(st_path, "w") as fh:
        json.dump(stats.to_dict(), fh, indent=2)
    res_path = os.path.join(s["out"], "solve_residuals.csv")
    write_table(res_path, [{"iteration": i, "residual_norm": v}
                           for i, v in enumerate(stats.residual_norms)], "csv")
    print(f"measured convergence factor: {stats.factor:.6e}")
    print(f"wrote {sol}, {st_path} and {res_path}")
    if s["compare_sequential"]:
        exact = tmg.forward_solve(tmg.GlobalSystem(hier.finest.ops, n), rhs)
        print(f"max deviation from forward substitution: {float(np.max(np.abs(u - exact))):.6e}")
    if not stats.converged:
        print(f"did not converge within {cfg.max_iters} iterations", file=sys.stderr)
        return EXIT_NOT_CONVERGED
    return EXIT_OK


# ---------------------------------------------------------------------------
# bench


def _world():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("RANK", 0))


def bench_point(p_t: int, n: int, workers: int, s: dict):
    """(median seconds, iterations, samples) of the reference bench problem
    (bench.py:77-90) on ``workers`` GPUs."""
    import torch

    import paper_1409_5254_b200 as tmg
    basis = tmg.BasisSpec(p_t)
    hier = tmg.TimeHierarchy.build(basis, float(s["tau"]), n)
    cfg = tmg.CycleConfig(nu1=int(s["nu1"]), nu2=int(s["nu2"]), eps=float(s["eps"]),
                          seed=int(s["seed"]))
    u0 = tmg.random_initial_guess(hier, cfg.seed)
    f = np.zeros_like(u0)
    samples, iters = [], 0
    if workers == 1:
        fd = torch.from_numpy(f).cuda()
        ud = torch.from_numpy(u0).cuda()
        for _ in range(int(s["reps"])):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _, st = tmg.solve(hier, fd, ud, cfg)
            e1.record()
            torch.cuda.synchronize()
            samples.append(e0.elapsed_time(e1) * 1e-3)
            iters = st.iterations
    else:
        import torch.distributed as dist
        from .timeshard import solve_time_sharded
        group = dist.new_group(list(range(workers)))
        if dist.get_rank() < workers:
            for _ in range(int(s["reps"])):
                dist.barrier(group=group)
                t0 = time.perf_counter()
                _, st = solve_time_sharded(hier, f, u0, cfg, group=group)
                torch.cuda.synchronize()
                dt = torch.tensor([time.perf_counter() - t0], device="cuda")
                dist.all_reduce(dt, op=dist.ReduceOp.MAX, group=group)
                samples.append(float(dt))
                iters = st.iterations
    return (statistics.median(samples) if samples else float("nan")), iters, samples


def run_bench(s: dict) -> int:
    workers = _int_list(s["workers"])
    if not workers or any(w < 1 or w & (w - 1) for w in workers) or workers != sorted(workers):
        raise UsageError(f"workers must be nondecreasing powers of two, got {workers}")
    if int(s["reps"]) < 3:
        raise UsageError(f"need >= 3 repetitions for a median, got {s['reps']}")
    world, rank = _world()
    if max(workers) > world:
        raise UsageError(f"{max(workers)} workers need as many torchrun ranks (have {world})")
    if world > 1:
        import torch
        import torch.distributed as dist
        if not dist.is_initialized():
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
            dist.init_process_group("nccl")
    if s["mode"] == "strong" and int(s["total_steps"]) % max(workers):
        raise UsageError(f"total steps {s['total_steps']} not divisible by {max(workers)} workers")
    rows = []
    for p_t in _int_list(s["pt"]):
        base = None
        for w in workers:
            n = int(s["total_steps"]) if s["mode"] == "strong" else w * int(s["steps_per_worker"])
            med, iters, samples = bench_point(p_t, n, w, s)
            base = med if base is None else base
            rows.append({"mode": s["mode"], "workers": w, "steps": n, "p_t": p_t,
                         "median_time": med,
                         "scaled": base / med if s["mode"] == "strong" else med / base,
                         "iterations": iters, "samples": samples,
                         "time_dof_per_s": n * (p_t + 1) * iters / med if med > 0 else 0.0})
    if rank == 0:
        os.makedirs(s["out"], exist_ok=True)
        path = os.path.join(s["out"], f"bench_{s['mode']}.{s['format']}")
        write_table(path, rows, s["format"])
        print(f"wrote {len(rows)} rows to {path}")
    return EXIT_OK


# ---------------------------------------------------------------------------


def main(argv=None) -> int:
    parser = build_parser()
    try:
        ns = parser.parse_args(argv)
        flags = vars(ns)
        command = flags.get("command")
        if command is None:
            raise UsageError("a subcommand is required: solve or bench")
        s = settings(command, flags)
        return run_solve(s) if command == "solve" else run_bench(s)
    except UsageError as e:
        print(f"usage error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except SystemExit as e:  # --help
        return e.code if isinstance(e.code, int) else EXIT_USAGE
    except (ValueError, OSError, json.JSONDecodeError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
