#!/usr/bin/env python
"""Benchmark of the B200 time-multigrid slab sweep (BASELINE.json metric:
"V-cycle time-DoF/s (fp64) and % of HBM roofline; wall time to 1e-8").

Default workload (BASELINE config 3, the largest single-GPU configuration):
B = 64 independent seeded problems, p_t = 1, N = 2^22 slabs each, T = 1, fp64,
V(1,1)-cycles coarsening to 2 slabs, zero initial guess, iterated to a 1e-8
relative residual with every problem stopping on its own (the reference
stopping rule, multigrid.py:481-496).  One step = one batched solve with the
inputs resident in HBM (4 GiB per array > 126 MB L2: no L2 flush needed).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload config3]
    python bench.py --impl reference      # the CPU reference arm (oracle port)

Under torchrun each rank solves its own 64 problems (problem ids rank*64+b):
weak scaling with no data-path collective; time = max over ranks.
Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "V-cycle time-DoF/s (fp64)"
UNIT = "time-DoF/s"
PROFILE_SUMMARY = os.path.join(REPO, "profiles", "ncu_summary.json")

WORKLOADS = {
    "config3": dict(batch=64, n=1 << 22, p_t=1, T=1.0, nu=1),
    "config2": dict(batch=1, n=1 << 20, p_t=1, T=1.0, nu=1),
    "config2_p3": dict(batch=1, n=1 << 20, p_t=3, T=1.0, nu=1),
    "config1": dict(batch=1, n=1 << 10, p_t=1, T=1.0, nu=1),
    # BASELINE config 5: ONE fused pass (nu1 = 2 sweeps + residual +
    # restriction) over N = 2^26 slabs, p_t = 3, u and f iid N(0, 1)
    "config5": dict(batch=1, n=1 << 26, p_t=3, T=1.0, nu=2),
}
C5_METRIC = "fused down pass time-DoF/s (fp64) and % of HBM roofline"
C5_BYTES = 3.5  # algorithmic bytes per fine slab, units of n_t * s


# ---------------------------------------------------------------------------
# helpers

def dist_env():
    from paper_1409_5254_b200 import dist as tdist
    return tdist.env()


def peak_hbm():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = f"/tmp/tmg_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.fh,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 3:
                    continue
                try:
                    s, m = float(parts[0]), float(parts[1])
                    bits = int(parts[2], 16)
                except ValueError:
                    continue
                mx = max(mx, m)
                if bits & 0x1:  # idle samples are not "under load"
                    continue
                sm.append(s)
                for bit, name in REASON_BITS.items():
                    if bits & bit:
                        reasons.add(name)
        except FileNotFoundError:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_hier(w):
    import paper_1409_5254_b200 as tmg
    return tmg.TimeHierarchy.build(tmg.BasisSpec(w["p_t"]), w["T"] / w["n"], w["n"], coarsest=2)


# ---------------------------------------------------------------------------
# CPU: oracle port of the reference (the reference arm and cpu_baseline)

def cpu_solve_sample(w, F_host_list, budget_s=12.0, threads=None):
    """Full reference-order solves of whole problems on the host until the
    time budget is used (at least one problem).  Returns (value, sample, cores)."""
    from oracle import oracle as O
    import paper_1409_5254_b200 as tmg
    if threads:
        O.set_threads(threads)
    cores = O.num_threads()
    hier = make_hier(w)
    om = [tmg.optimal_omega(tmg.alpha(hier.basis, l.tau)) for l in hier.levels]
    dofs = 0
    secs = 0.0
    done = 0
    for rhs in F_host_list:
        t0 = time.perf_counter()
        _, _, it = O.iterate(hier, om, rhs, np.zeros_like(rhs), w["nu"], w["nu"], 1e-8, 250)
        secs += time.perf_counter() - t0
        dofs += w["n"] * (w["p_t"] + 1) * it
        done += 1
        if secs >= budget_s:
            break
    sample = (f"{done} of {w['batch']} problems solved to 1e-8 (N={w['n']}, p_t={w['p_t']}, "
              f"V({w['nu']},{w['nu']})) by the C restatement of the reference, {cores} OpenMP threads")
    return dofs / secs, sample, cores, secs


def run_reference_arm(args, w):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    if args.workload == "config5":
        return run_reference_c5(args, w, ws)
    import torch
    from paper_1409_5254_b200 import problems
    # same seeded inputs as the GPU arm (assembled on the host here)
    hosts = []
    vals = []
    total_steps = args.warmup + args.steps
    for s in range(total_steps):
        b = s % w["batch"]
        rhs, _, _ = problems.seeded_rhs(w["p_t"], w["n"], w["T"], 42, b if w["batch"] > 1 else None)
        hosts.append(rhs)
    from oracle import oracle as O
    import paper_1409_5254_b200 as tmg
    cores = os.cpu_count() or 1
    O.set_threads(cores)
    hier = make_hier(w)
    om = [tmg.optimal_omega(tmg.alpha(hier.basis, l.tau)) for l in hier.levels]
    times, dofs = [], []
    for s, rhs in enumerate(hosts):
        t0 = time.perf_counter()
        _, _, it = O.iterate(hier, om, rhs, np.zeros_like(rhs), w["nu"], w["nu"], 1e-8, 250)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            dofs.append(w["n"] * (w["p_t"] + 1) * it)
    value = sum(dofs) / sum(times)
    sample = (f"each step: one of the {w['batch']} problems (N={w['n']}, p_t={w['p_t']}) solved to "
              f"1e-8 by the C restatement of the reference (oracle/), {cores} threads")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, w),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_reference_c5(args, w, ws):
    """Reference arm of config 5: the oracle's fused pass over a bounded
    sample (2^22 of the 2^26 slabs) per step, all host threads."""
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    O.set_threads(cores)
    m = 1 << 22
    nt = w["p_t"] + 1
    rng = np.random.default_rng(0)
    u = rng.standard_normal((m, nt))
    f = rng.standard_normal((m, nt))
    ops, r1, r2, om = c5_level(w)
    times = []
    for s_ in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        O.down_pass(ops, r1, r2, om, u, f, nu=w["nu"])
        if s_ >= args.warmup:
            times.append(time.perf_counter() - t0)
    value = m * nt * len(times) / sum(times)
    sample = (f"each step: the fused pass over {m} of the {w['n']} slabs by the C restatement of "
              f"the reference (oracle/), {cores} threads")
    line = {"impl": "reference", "metric": C5_METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config5 (bounded CPU sample)", "n_slabs": w["n"], "p_t": w["p_t"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(args, w):
    return {"workload": (f"{args.workload}: B={w['batch']} x N=2^{int(np.log2(w['n']))} slabs, "
                         f"p_t={w['p_t']}, T={w['T']:g}, V({w['nu']},{w['nu']})-cycles to 1e-8, "
                         "coarsest=2, zero initial guess, optimal omega"),
            "batch_per_gpu": w["batch"], "n_slabs": w["n"], "p_t": w["p_t"], "nu": w["nu"],
            "problems": "seeded (SURVEY 8d): default_rng([42, b]) a, phi, u0",
            "l2": "inputs larger than L2 (no flush)" if w["batch"] * w["n"] * (w["p_t"] + 1) * 8 > 2 ** 27
            else "working set L2-resident; L2 flushed between steps"}


# ---------------------------------------------------------------------------
# GPU arm

def live_kernel_times(plan, F, U, floors, eps, max_iters):
    """Per-kernel device times of one solve of the plan's OWN launches: the C
    ABI's trace mode launches the same kernels directly (no graph) with a CUDA
    event on the launch stream after each one (tmg_trace_enable/read).
    Returns {description: (launches, total_s)}."""
    from paper_1409_5254_b200 import _native as nat
    L = nat.load()
    U.zero_()
    L.tmg_trace_enable(1)
    try:
        plan.solve(F, U, floors, eps, max_iters)
        buf = ctypes.create_string_buffer(1 << 20)
        L.tmg_trace_read(buf, len(buf))
    finally:
        L.tmg_trace_enable(0)
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.split("\t")
        out[name] = (int(cnt), float(ms) * 1e-3)
    return out


# algorithmic bytes per fine slab (units of n_t * 8 B) of the stream kernel kinds
# the plan launches: K_UP2DOWN (7) = finest up pass of cycle k
# fused with the finest down pass of cycle k+1: reads u, f, u_c/2, writes u,
# f_c/2; K_UP2 (5) at a coarse level (zero original iterate): reads f, u_c/2,
# writes u; K_DOWN (1) at a coarse level (zero guess): reads f, writes f_c/2
# "v" = stream_kernel_v: K_UP2DOWN with the level-1 up pass fused in (vertical
# fusion): reads u, f, f_1/2, u_2/4, writes u, f_c/2 -> 4.25
KIND_BYTES = {"v": 4.25, 7: 4.0, 5: 2.5, 1: 1.5, 4: 2.5}


def kernel_roofline(times, n, nt, B, kind):
    """(average launch seconds, algorithmic bytes per launch, description) of
    the stream kernel of a kind at the level with n slabs per problem (kind
    "v": the vertically fused finest pass)."""
    for name, (cnt, tot) in times.items():
        hit = name.startswith("stream_kernel_v (") if kind == "v" else \
            (f"kind={kind}>" in name and f" n={n} " in name)
        if hit:
            return tot / cnt, KIND_BYTES[kind] * nt * 8 * n * B, name
    return None, None, None


GOLDEN = os.path.join(REPO, "tests", "golden", "golden.json")
# golden solves of each workload: (batch slot, golden case name, batch index)
PIN_CASES = {"config3": [(0, "config3_b0", 0), (1, "config3_b1", 1)],
             "config2": [(0, "config2_p1", None)], "config2_p3": [(0, "config2_p3", None)]}


def _sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def parity_pins(workload, ids):
    """[(slot, golden case, host rhs)] for the batch slots holding golden
    problems (only where this rank's problem ids include them)."""
    from paper_1409_5254_b200 import problems
    try:
        with open(GOLDEN) as fh:
            cases = {c["name"]: c for c in json.load(fh)["big_solves"]}
    except OSError:
        return []
    out = []
    for slot, name, bidx in PIN_CASES.get(workload, []):
        if bidx is not None and (slot >= len(ids) or ids[slot] != bidx):
            continue
        c = cases[name]
        rhs, _, _ = problems.seeded_rhs(c["p_t"], c["n"], c["T"], 42, c["batch_index"])
        out.append((slot, c, rhs))
    return out


def check_pins(pins, U, stats):
    """{case: {sha_rhs, sha_u, norms, iterations}} -- each True iff identical to
    the reference's own solve of that problem (tests/golden/make_golden.py)."""
    res = {}
    for slot, c, rhs in pins:
        st = stats[slot]
        res[c["name"]] = {"sha_rhs": _sha(rhs) == c["sha_rhs"],
                          "sha_u": _sha(U[slot].cpu().numpy()) == c["sha_u"],
                          "norms": st.residual_norms == c["residual_norms"],
                          "iterations": st.iterations == c["iterations"]}
    res["all"] = bool(pins) and all(all(v.values()) for k, v in res.items())
    return res


def c5_level(w):
    """(LevelDesc-ready operators) of config 5: tau = T / N = 2^-26, optimal omega."""
    import paper_1409_5254_b200 as tmg
    tau = w["T"] / w["n"]
    basis = tmg.BasisSpec(w["p_t"])
    ops = tmg.assemble_local(basis, tau)
    r1, r2 = tmg.build_transfers(basis, tau)
    return ops, r1, r2, tmg.optimal_omega(tmg.alpha(basis, tau))


def run_config5(args, w):
    """BASELINE config 5 through the C ABI's tmg_down: fp64 (the parity path)
    with the reference's config-5 inputs on the first 2^16 slabs (their
    outputs must hash to the reference's, tests/golden), seeded N(0,1)
    elsewhere; fp32 beside it (normwise vs fp64)."""
    import torch
    import torch.distributed as dist
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl")
    from paper_1409_5254_b200 import _native as nat, problems
    from paper_1409_5254_b200 import dist as tdist
    L = nat.load()
    n, nt, nu = w["n"], w["p_t"] + 1, w["nu"]
    ops, r1, r2, om = c5_level(w)
    d = nat.level_desc(ops, n, om, r1, r2)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5000 + rank)
    u = torch.randn((n, nt), generator=gen, device="cuda", dtype=torch.float64)
    f = torch.randn((n, nt), generator=gen, device="cuda", dtype=torch.float64)
    npre = 1 << 16
    up, fp = problems.kernel_inputs(npre, nt, 0)
    u[:npre].copy_(torch.from_numpy(up))
    f[:npre].copy_(torch.from_numpy(fp))
    uo = torch.empty_like(u)
    fc = torch.empty((n // 2, nt), dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    sp = ctypes.c_void_p(stream.cuda_stream)

    def step(dt, uu, ff, o, c):
        nat.check(L.tmg_down(dt, ctypes.byref(d), P(ff), P(uu), P(o), P(c), 1, nu, None, sp), "tmg_down")

    def timed(dt, uu, ff, o, c, k):
        for _ in range(args.warmup):
            step(dt, uu, ff, o, c)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            step(dt, uu, ff, o, c)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e-3

    with ClockSampler(local) as clk:
        elapsed = timed(0, u, f, uo, fc, args.steps)
    el_max, dof = tdist.reduce_time_and_work(elapsed, float(n * nt * args.steps), device="cuda")
    launch_s = elapsed / args.steps
    peak, peak_kind = peak_hbm()
    bytes_f64 = C5_BYTES * nt * 8 * n
    parity = {"prefix_sha_u": _sha(uo[:npre].cpu().numpy()) == golden_c5()["sha_u"],
              "prefix_sha_fc": _sha(fc[:npre // 2].cpu().numpy()) == golden_c5()["sha_fc"]}
    # fp32 variant of the same pass (throughput variant; normwise bar 1e-5)
    u32, f32 = u.float(), f.float()
    uo32, fc32 = torch.empty_like(u32), torch.empty_like(fc, dtype=torch.float32)
    el32 = timed(1, u32, f32, uo32, fc32, args.steps)
    err_u = float(torch.linalg.norm(uo32.double() - uo) / torch.linalg.norm(uo))
    err_fc = float(torch.linalg.norm(fc32.double() - fc) / torch.linalg.norm(fc))
    parity["fp32_normwise_u"] = err_u
    parity["fp32_normwise_fc"] = err_fc
    parity["all"] = parity["prefix_sha_u"] and parity["prefix_sha_fc"] and max(err_u, err_fc) <= 1e-5
    del u32, f32, uo32, fc32

    # e2e: host buffers (pinned) in and out every step through the C ABI call
    uh, fh = u.cpu().pin_memory(), f.cpu().pin_memory()
    uoh, fch = torch.empty_like(uh).pin_memory(), torch.empty_like(fc, device="cpu").pin_memory()

    def e2e():
        u.copy_(uh, non_blocking=True)
        f.copy_(fh, non_blocking=True)
        step(0, u, f, uo, fc)
        uoh.copy_(uo, non_blocking=True)
        fch.copy_(fc, non_blocking=True)
    e2e()
    torch.cuda.synchronize()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    for _ in range(args.steps):
        e2e()
    g1.record(stream)
    torch.cuda.synchronize()
    e2e_s, e2e_dof = tdist.reduce_time_and_work(g0.elapsed_time(g1) * 1e-3,
                                                float(n * nt * args.steps), device="cuda")
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = c5_cpu_sample(w, uh.numpy(), fh.numpy(), 1 << 22)
    if rank == 0:
        traffic = None
        try:
            with open(PROFILE_SUMMARY) as fh_:
                traffic = json.load(fh_).get("config5", {}).get("dram_bytes_per_launch")
        except Exception:
            pass
        line = {
            "metric": C5_METRIC, "value": dof / el_max, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "config5: one fused pass (nu1=2 sweeps + residual + restriction) "
                                   "over N=2^26 slabs, p_t=3, T=1 (tau=2^-26), optimal omega",
                       "n_slabs": n, "p_t": w["p_t"], "nu": nu,
                       "inputs": "u, f ~ N(0,1): first 2^16 slabs = the reference's config-5 "
                                 "inputs (default_rng(0)), the rest torch.randn (seed 5000+rank)",
                       "l2": "inputs larger than L2 (no flush)"},
            "roofline": {"bound": "hbm", "achieved": bytes_f64 / launch_s / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": bytes_f64 / launch_s / 1e9 / peak,
                         "traffic": traffic, "kernel": "stream_kernel<double,4,2,...,K_DOWN> (tmg_down)",
                         "bytes_per_launch": bytes_f64, "launch_s": launch_s,
                         "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                         "fp32": {"launch_s": el32 / args.steps,
                                  "achieved": bytes_f64 / 2 / (el32 / args.steps) / 1e9,
                                  "frac": bytes_f64 / 2 / (el32 / args.steps) / 1e9 / peak}},
            "e2e": {"value": e2e_dof / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 2 * n * nt * 8,
                    "d2h_bytes_per_step": n * nt * 8 + (n // 2) * nt * 8,
                    "path": "pinned host u, f -> H2D -> tmg_down (C ABI) -> D2H u, f_coarse, one stream"},
            "gpu_launches": args.steps,
            "parity": parity,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def config5_side_line(rank, steps=10, warmup=3):
    """BASELINE config 5 (the north-star gate: one fused pass of nu1 = 2 sweeps
    + residual + restriction over N = 2^26 slabs, p_t = 3) measured beside the
    headline, so that the default run carries it: fp64 GB/s against the HBM
    peak with the reference's golden prefix hashes, fp32 beside it.  Its own
    full line (e2e, CPU baseline): --workload config5."""
    import torch
    from paper_1409_5254_b200 import _native as nat, problems
    w = WORKLOADS["config5"]
    L = nat.load()
    n, nt, nu = w["n"], w["p_t"] + 1, w["nu"]
    ops, r1, r2, om = c5_level(w)
    d = nat.level_desc(ops, n, om, r1, r2)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5000 + rank)
    u = torch.randn((n, nt), generator=gen, device="cuda", dtype=torch.float64)
    f = torch.randn((n, nt), generator=gen, device="cuda", dtype=torch.float64)
    npre = 1 << 16
    up, fp = problems.kernel_inputs(npre, nt, 0)
    u[:npre].copy_(torch.from_numpy(up))
    f[:npre].copy_(torch.from_numpy(fp))
    uo = torch.empty_like(u)
    fc = torch.empty((n // 2, nt), dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    sp = ctypes.c_void_p(stream.cuda_stream)

    def timed(dt, uu, ff, o, c):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for k in range(warmup + steps):
            if k == warmup:
                e0.record(stream)
            nat.check(L.tmg_down(dt, ctypes.byref(d), P(ff), P(uu), P(o), P(c), 1, nu, None, sp), "tmg_down")
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e-3 / steps

    t64 = timed(0, u, f, uo, fc)
    peak, _ = peak_hbm()
    nbytes = C5_BYTES * nt * 8 * n
    out = {"workload": "config5: tmg_down (nu1=2 sweeps + residual + restriction), N=2^26, p_t=3, inputs > L2",
           "steps": steps, "warmup": warmup, "dtype": "f64", "launch_s": t64, "bytes_per_launch": nbytes,
           "achieved": nbytes / t64 / 1e9, "peak": peak, "unit": "GB/s", "frac": nbytes / t64 / 1e9 / peak,
           "parity": {"prefix_sha_u": _sha(uo[:npre].cpu().numpy()) == golden_c5()["sha_u"],
                      "prefix_sha_fc": _sha(fc[:npre // 2].cpu().numpy()) == golden_c5()["sha_fc"]}}
    u32, f32 = u.float(), f.float()
    uo32, fc32 = torch.empty_like(u32), torch.empty_like(fc, dtype=torch.float32)
    t32 = timed(1, u32, f32, uo32, fc32)
    out["fp32"] = {"launch_s": t32, "achieved": nbytes / 2 / t32 / 1e9, "frac": nbytes / 2 / t32 / 1e9 / peak,
                   "normwise_u": float(torch.linalg.norm(uo32.double() - uo) / torch.linalg.norm(uo)),
                   "normwise_fc": float(torch.linalg.norm(fc32.double() - fc) / torch.linalg.norm(fc))}
    out["parity"]["all"] = bool(out["parity"]["prefix_sha_u"] and out["parity"]["prefix_sha_fc"]
                                and max(out["fp32"]["normwise_u"], out["fp32"]["normwise_fc"]) <= 1e-5)
    return out


def golden_c5():
    with open(GOLDEN) as fh:
        return json.load(fh)["config5"]


def c5_cpu_sample(w, u, f, m, threads=None):
    """The oracle's fused pass (C restatement of the reference order) over the
    first m slabs, all host threads: {value (time-DoF/s), ...}."""
    from oracle import oracle as O
    if threads:
        O.set_threads(threads)
    cores = O.num_threads()
    ops, r1, r2, om = c5_level(w)
    uu, ff = np.ascontiguousarray(u[:m]), np.ascontiguousarray(f[:m])
    O.down_pass(ops, r1, r2, om, uu[:1024], ff[:1024], nu=w["nu"])
    t0 = time.perf_counter()
    reps = 0
    while True:
        O.down_pass(ops, r1, r2, om, uu, ff, nu=w["nu"])
        reps += 1
        if time.perf_counter() - t0 > 5.0 or reps >= 20:
            break
    secs = (time.perf_counter() - t0) / reps
    nt = w["p_t"] + 1
    return {"value": m * nt / secs, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"the fused pass over the first {m} of {w['n']} slabs by the C restatement of "
                      f"the reference (oracle/), {cores} OpenMP threads, {reps} repetitions",
            "gbs": C5_BYTES * nt * 8 * m / secs / 1e9, "seconds": secs}


def run_gpu_arm(args, w):
    if args.workload == "config5":
        return run_config5(args, w)
    import torch
    import torch.distributed as dist
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    import paper_1409_5254_b200 as tmg
    from paper_1409_5254_b200 import problems, solver

    B, n, p_t = w["batch"], w["n"], w["p_t"]
    nt = p_t + 1
    from paper_1409_5254_b200 import dist as tdist
    ids = tdist.problem_ids(rank, ws, B) if B > 1 else [None]
    F = problems.seeded_rhs_batch_device(p_t, n, w["T"], 42, ids if B > 1 else (None,))
    # parity pins: the golden problems of this workload (the reference's own
    # solves, tests/golden) are assembled on the host exactly as the reference
    # does and placed in the batch; their solutions are checked after the
    # timed region
    pins = parity_pins(args.workload, ids)
    for slot, case, rhs in pins:
        F[slot].copy_(torch.from_numpy(rhs))
    floors = [1e-12 * float(v) for v in torch.linalg.norm(F.reshape(B, -1), dim=1).cpu()]
    hier = make_hier(w)
    cfg = tmg.CycleConfig(nu1=w["nu"], nu2=w["nu"], eps=1e-8)
    U = torch.zeros_like(F)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if B * n * nt * 8 <= 2 ** 27 else None

    def step():
        U.zero_()
        if flush is not None:
            flush.zero_()
        return tmg.solve_batched(hier, F, U, cfg, floors=floors, inplace=True)

    for _ in range(args.warmup):
        _, stats = step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            _, stats = step()
            iters.append([s.iterations for s in stats])
        e1.record()
        torch.cuda.synchronize()
    elapsed = e0.elapsed_time(e1) * 1e-3
    if ws > 1:
        dist.barrier()
    dof = float(sum(n * nt * k for row in iters for k in row))
    elapsed, dof = tdist.reduce_time_and_work(elapsed, dof, device="cuda")
    value = dof / elapsed
    plan = solver.get_plan(hier, 0, len(hier.levels), solver.omegas_for(hier, cfg, len(hier.levels)),
                           cfg, B)
    info = plan.info()
    max_it = max(max(r) for r in iters)
    launches_per_step = 3 + info["kernels_per_cycle"] * max_it

    # e2e: through the public API with HOST buffers (pinned): every step copies
    # its batch in (H2D) and its solution out (D2H).  Headline: the streamed
    # API (solve_batched_stream -> tmg_plan_solve_host_stream), which overlaps
    # step k's solve with step k+1's copy-in and step k-1's copy-out; beside
    # it the one-call-per-step form (tmg_plan_solve_host: the batch's copies
    # overlap its own sub-batch solves only)
    F_host = F.cpu().pin_memory()
    U_host = torch.empty_like(F_host).pin_memory()
    U_ring = [U_host] + [torch.empty_like(F_host).pin_memory() for _ in range(2)]

    def e2e_step():
        # zero initial guess (not copied), solution written into pinned U_host
        plan_h = solver.get_plan(hier, 0, len(hier.levels),
                                 solver.omegas_for(hier, cfg, len(hier.levels)), cfg, B)
        it, norms, conv = plan_h.solve_host(F_host, None, U_host, floors, cfg.eps, cfg.max_iters)
        return [type("S", (), {"iterations": int(k)}) for k in it]

    # the golden problems' solutions of the last timed solve
    parity = check_pins(pins, U, stats)

    e2e_step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = args.steps
    dof_call = 0.0
    f0.record()
    for _ in range(e2e_steps):
        st = e2e_step()
        dof_call += sum(n * nt * s.iterations for s in st)
    f1.record()
    torch.cuda.synchronize()
    call_time = f0.elapsed_time(f1) * 1e-3
    call_time, dof_call = tdist.reduce_time_and_work(call_time, dof_call, device="cuda")

    # streamed: the K steps' batches through one call (warm-up stream first)
    floors_k = [floors] * max(args.warmup, 1)
    solver.solve_batched_stream(hier, [F_host] * len(floors_k), [U_ring[k % 3] for k in range(len(floors_k))],
                                cfg, floors=floors_k)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    g0.record()
    _, st_all = solver.solve_batched_stream(hier, [F_host] * e2e_steps,
                                            [U_ring[k % 3] for k in range(e2e_steps)], cfg,
                                            floors=[floors] * e2e_steps)
    g1.record()
    torch.cuda.synchronize()
    e2e_wall = time.perf_counter() - w0
    e2e_time = max(g0.elapsed_time(g1) * 1e-3, e2e_wall)
    dof_e2e = float(sum(n * nt * s.iterations for st in st_all for s in st))
    e2e_time, dof_e2e = tdist.reduce_time_and_work(e2e_time, dof_e2e, device="cuda")

    # roofline of the dominant kernel, timed live on the plan's own launches:
    # the finest-level fused up/next-down pass (K_UP2DOWN, ~2/3 of the solve's
    # kernel time), plus the level-1 passes beside it
    times = live_kernel_times(plan, F, U, floors, cfg.eps, cfg.max_iters)
    peak, peak_kind = peak_hbm()
    up_s, up_bytes, up_name = kernel_roofline(times, n, nt, B, "v")
    if up_s is None:  # configurations without the vertical fusion
        up_s, up_bytes, up_name = kernel_roofline(times, n, nt, B, 7)
    l1 = {}
    # the largest coarse pair kernels: down pair (levels 1, 2; 1.75 n_t 8 B per
    # level-1 slab) and up pair (levels 2, 3; 2.75 n_t 8 B per level-2 slab)
    for label, prefix, nl, per in (("down_pair_1_2", "stream_kernel_d pair n=%d+" % (n // 2), n // 2, 1.75),
                                   ("up_pair_2_3", "stream_kernel_v pair n=%d+" % (n // 4), n // 4, 2.75)):
        for name, (cnt, tot) in times.items():
            if name.startswith(prefix):
                kb = per * nt * 8 * nl * B
                l1[label] = {"kernel": name, "bytes_per_launch": kb, "launch_s": tot / cnt,
                             "achieved": kb / (tot / cnt) / 1e9, "frac": kb / (tot / cnt) / 1e9 / peak}
    traffic = None
    try:
        with open(PROFILE_SUMMARY) as fh:
            prof = json.load(fh).get(args.workload, {})
        traffic = prof.get("fused_dram_bytes_per_launch")
    except Exception:
        pass

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        hosts = [F[b].cpu().numpy() for b in range(min(B, 4))]
        v, sample, cores, secs = cpu_solve_sample(w, hosts, budget_s=args.cpu_budget)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
               "seconds": secs}

    c5 = None
    if rank == 0 and args.workload == "config3" and not args.no_config5:
        del F, U
        torch.cuda.empty_cache()
        try:
            c5 = config5_side_line(rank)
        except Exception as exc:  # the headline line must still print
            c5 = {"error": repr(exc)}

    if rank == 0:
        ms = 1e3 * elapsed / args.steps
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, w),
            "wall_s_to_1e-8": ms * 1e-3, "iterations": sorted(set(i for r in iters for i in r)),
            "roofline": {"bound": "hbm", "achieved": up_bytes / up_s / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": up_bytes / up_s / 1e9 / peak, "traffic": traffic,
                         "kernel": "finest-level fused pass: level-1 up pass of cycle k (in shared memory) + "
                                   "finest up pass of cycle k (pre-sweeps recomputed, prolong-add, nu2 sweeps) + "
                                   "finest down pass of cycle k+1 (norm leaves, nu1 sweeps, residual, "
                                   "restriction), whole batch: " + up_name,
                         "bytes_per_launch": up_bytes, "launch_s": up_s,
                         "timing": "CUDA events on the launch stream around the plan's own launches "
                                   "(tmg_trace_enable), one solve after the timed region",
                         "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                         "frac_of_nominal_8TBs": up_bytes / up_s / 1e9 / 8000.0,
                         "coarse_pairs": l1},
            "e2e": {"value": dof_e2e / e2e_time, "unit": UNIT,
                    "h2d_bytes_per_step": B * n * nt * 8, "d2h_bytes_per_step": B * n * nt * 8,
                    "steps": e2e_steps, "path": "solve_batched_stream -> C ABI tmg_plan_solve_host_stream "
                    "with pinned host buffers: every step copies its batch in (H2D f) and its solution out "
                    "(D2H u); step k's solve overlaps step k+1's copy-in and step k-1's copy-out "
                    "(copy-in, compute, copy-out streams; three full-batch plans in rotation)",
                    "per_call": {"value": dof_call / call_time, "path": "one tmg_plan_solve_host call per step "
                                 "(16 pipelined sub-batches within the step)"}},
            "gpu_launches": launches_per_step * args.steps,
            "parity": parity,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "config5": c5,
        }
        # whole-cycle HBM fraction over every problem-cycle of the run: this
        # design moves 7 n_t 8 B per finest slab per V-cycle (vertically fused
        # finest pass 4.25 + level-1 down 1.5/2 + levels >= 2 (1.5 + 2.5) / 4 /
        # (1 - 1/2)); SURVEY 8(d)'s model (separate passes, every pass stores u)
        # is 13 n_t 8 B
        cycles = sum(sum(r) for r in iters)
        line["cycle_hbm_frac"] = (7 * nt * 8 * n * cycles) / elapsed / 1e9 / peak
        line["cycle_hbm_frac_survey_model"] = (13 * nt * 8 * n * cycles) / elapsed / 1e9 / peak
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="config3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-config5", action="store_true", help="skip the config-5 side measurement")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference_arm(args, w)
    else:
        run_gpu_arm(args, w)


if __name__ == "__main__":
    main()
