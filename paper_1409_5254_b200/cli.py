"""GPU-backed ``timemg solve`` (the reference's CLI caller of the hot path,
pkg/src/timemg/cli.py:232-290).

Same subcommand, flags, defaults (``_SOLVE_DEFAULTS``, cli.py:235-238),
config-file layering (cli.py:46-59), output files and exit codes (0 ok,
2 usage error, 3 non-convergence; cli.py:1-7) as the reference; the solve runs
in the sm_100a kernels.  With ``--time-shard`` under torchrun (one process per
GPU, NCCL) the problem is sharded along time (``timeshard.py``); rank 0 writes
the files.

    python -m paper_1409_5254_b200.cli solve --pt 1 --steps 1048576 --nu1 1 --nu2 1
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import sys

import numpy as np

_FORMATS = ("csv", "json")
_SOLVE_DEFAULTS = dict(pt=0, steps=64, T=1.0, tau=None, u0=1.0, f="zero", f_param=1.0,
                       nu1=2, nu2=2, omega="optimal", levels="max", eps=1e-8,
                       seed=42, workers=1, max_iters=250, compare_sequential=False,
                       out=".", format="csv", time_shard=False)


def _write_rows(path: str, rows: list, fmt: str) -> None:
    if fmt == "json":
        with open(path, "w") as fh:
            json.dump(rows, fh, indent=2)
        return
    with open(path, "w", newline="") as fh:
        writer = csv.DictWriter(fh, fieldnames=list(rows[0].keys()))
        writer.writeheader()
        writer.writerows(rows)


def _merge_config(args, parser, defaults: dict):
    """defaults < JSON config file < explicit flags; unknown file keys are an error."""
    merged = dict(defaults)
    path = getattr(args, "config", None)
    if path:
        with open(path) as fh:
            file_values = json.load(fh)
        unknown = set(file_values) - set(defaults)
        if unknown:
            parser.error(f"unknown config keys: {sorted(unknown)}")
        merged.update(file_values)
    merged.update(vars(args))
    return argparse.Namespace(**merged)


def _parse_omega(value: str):
    if value == "optimal":
        return value
    try:
        return float(value)
    except ValueError:
        raise argparse.ArgumentTypeError(f"omega must be 'optimal' or a number, got {value!r}")


def _preset_f(name: str, param: float):
    if name == "zero":
        return lambda t: np.zeros_like(t)
    if name == "const":
        return lambda t: np.full_like(t, param)
    if name == "poly":
        return lambda t: t ** param
    if name == "sin":
        return lambda t: np.sin(param * t)
    raise ValueError(f"unknown f preset {name!r}")


def cmd_solve(args) -> int:
    import paper_1409_5254_b200 as tmg
    basis = tmg.BasisSpec(args.pt)
    tau = args.tau if args.tau is not None else args.T / args.steps
    levels = args.levels if args.levels == "max" else int(args.levels)
    hier = tmg.TimeHierarchy.build(basis, tau, args.steps, n_levels=levels)
    config = tmg.CycleConfig(nu1=args.nu1, nu2=args.nu2, damping=args.omega, levels=levels,
                             eps=args.eps, max_iters=args.max_iters, seed=args.seed,
                             workers=args.workers)
    rhs = tmg.rhs_moments(_preset_f(args.f, args.f_param), basis, tau, args.steps, u0=args.u0)
    rank = 0
    if args.time_shard:
        import torch
        import torch.distributed as dist
        from . import timeshard
        if not dist.is_initialized():
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
            dist.init_process_group("nccl")
        rank = dist.get_rank()
        u, stats = timeshard.solve_time_sharded(hier, rhs, None, config)
    else:
        u, stats = tmg.solve(hier, rhs, None, config)
    if rank != 0:
        return 0 if stats.converged else 3

    os.makedirs(args.out, exist_ok=True)
    end_vals = u @ hier.finest.ops.eval_end
    rows = [{"step": n, "t_end": (n + 1) * tau, "u_end": float(end_vals[n]),
             **{f"c{i}": float(u[n, i]) for i in range(basis.n_t)}}
            for n in range(args.steps)]
    sol_path = os.path.join(args.out, f"solve_solution.{args.format}")
    _write_rows(sol_path, rows, args.format)
    stats_path = os.path.join(args.out, "solve_stats.json")
    with open(stats_path, "w") as fh:
        json.dump(stats.to_dict(), fh, indent=2)
    res_path = os.path.join(args.out, "solve_residuals.csv")
    with open(res_path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(["iteration", "residual_norm"])
        writer.writerows(enumerate(stats.residual_norms))
    print(f"measured convergence factor: {stats.factor:.6e}")
    print(f"wrote {sol_path}, {stats_path} and {res_path}")

    if args.compare_sequential:
        ref = tmg.forward_solve(tmg.GlobalSystem(hier.finest.ops, args.steps), rhs, method="serial")
        dev = float(np.max(np.abs(u - ref)))
        print(f"max deviation from forward substitution: {dev:.6e}")

    if not stats.converged:
        print(f"did not converge within {config.max_iters} iterations", file=sys.stderr)
        return 3
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="timemg-b200",
                                     description="time-multigrid solver on B200 (sm_100a)")
    subs = parser.add_subparsers(dest="command", required=True)
    p = subs.add_parser("solve", help="solve u' + u = f with the time-multigrid solver",
                        argument_default=argparse.SUPPRESS)
    p.add_argument("--pt", type=int)
    p.add_argument("--steps", type=int)
    p.add_argument("--T", type=float)
    p.add_argument("--tau", type=float, help="step size (overrides --T)")
    p.add_argument("--u0", type=float)
    p.add_argument("--f", choices=("zero", "const", "poly", "sin"))
    p.add_argument("--f-param", type=float)
    p.add_argument("--nu1", type=int)
    p.add_argument("--nu2", type=int)
    p.add_argument("--omega", type=_parse_omega)
    p.add_argument("--levels")
    p.add_argument("--eps", type=float)
    p.add_argument("--seed", type=int)
    p.add_argument("--workers", type=int)
    p.add_argument("--max-iters", type=int)
    p.add_argument("--compare-sequential", action="store_true")
    p.add_argument("--time-shard", action="store_true",
                   help="shard the time axis over the torchrun ranks (one GPU each)")
    p.add_argument("--config", help="JSON file with defaults for this subcommand")
    p.add_argument("--out", help="output directory")
    p.add_argument("--format", choices=_FORMATS, help="output file format")
    p.set_defaults(func=cmd_solve, defaults=_SOLVE_DEFAULTS)
    return parser


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return exc.code if isinstance(exc.code, int) else 2
    try:
        if args.defaults is not None:
            args = _merge_config(args, parser, args.defaults)
        return args.func(args)
    except SystemExit as exc:  # parser.error inside merge
        return exc.code if isinstance(exc.code, int) else 2
    except (ValueError, OSError, json.JSONDecodeError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
