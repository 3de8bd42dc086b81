"""ctypes binding of the C ABI in include/timemg_b200.h (libtimemg_b200.so).

There is no CPU fallback: if the shared library is missing or no B200 is
visible, every solver entry point raises.  ``build()`` compiles the library
in-tree for sm_100a (nvcc cross-compiles without a GPU).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
# TMG_LIB: an alternative build of the same library (A/B experiments, scripts/ab_build.sh)
LIB_PATH = os.environ.get("TMG_LIB") or os.path.join(HERE, "libtimemg_b200.so")
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(REPO, "include")
MAXNT = 8          # field capacity of tmg_level_desc (TMG_MAXNT)
KERNEL_MAXNT = 4   # n_t the kernels are instantiated for
F64, F32 = 0, 1
E_ARG, E_UNSUPPORTED, E_NOMEM = -1, -2, -3

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false",
              "-std=c++17", "-Xcompiler", "-fPIC", "-diag-suppress", "1886,128"]


class LevelDesc(ctypes.Structure):
    _fields_ = [
        ("n_t", ctypes.c_int32),
        ("has_transfer", ctypes.c_int32),
        ("n_slabs", ctypes.c_int64),
        ("omega", ctypes.c_double),
        ("minus_step", ctypes.c_double * (MAXNT * MAXNT)),
        ("coupling", ctypes.c_double * (MAXNT * MAXNT)),
        ("lu", ctypes.c_double * (MAXNT * MAXNT)),
        ("r1", ctypes.c_double * (MAXNT * MAXNT)),
        ("r2", ctypes.c_double * (MAXNT * MAXNT)),
        ("perm", ctypes.c_int32 * MAXNT),
    ]


class PlanOpts(ctypes.Structure):
    _fields_ = [
        ("dtype", ctypes.c_int32),
        ("nu1", ctypes.c_int32),
        ("nu2", ctypes.c_int32),
        ("gamma", ctypes.c_int32),
        ("coarse", ctypes.c_int32),
        ("dot_variant", ctypes.c_int32),
        ("use_graph", ctypes.c_int32),
        ("tail_max_slabs", ctypes.c_int32),
    ]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cuh")))


# translation units: the C ABI / driver, and one kernel-instantiation unit per
# (dtype, n_t) -- compiled in parallel, then linked into one shared library
# (dtype, n_t, part): tmg_inst.cu's instantiations split in four parts
# (dtype, n_t, part): tmg_inst.cu's instantiations split in four parts, plus
# the tail engine and coarse solves (tmg_inst_tail.cu)
_TYPES = (("double", "f64"), ("float", "f32"))
UNITS = [("tmg_api", "tmg_api.cu", []), ("tmg_rhs", "tmg_rhs.cu", [])] + [
    (f"tmg_inst_{tn}_{nt}_p{part}", "tmg_inst.cu", [f"-DTMG_T={t}", f"-DTMG_NT={nt}", f"-DTMG_PART={part}"])
    for t, tn in _TYPES for nt in (1, 2, 3, 4) for part in (0, 1, 2, 3)] + [
    (f"tmg_inst_{tn}_{nt}_tail", "tmg_inst_tail.cu", [f"-DTMG_T={t}", f"-DTMG_NT={nt}"])
    for t, tn in _TYPES for nt in (1, 2, 3, 4)]
# heaviest first, so the parallel build's tail is short
UNITS.sort(key=lambda u: (0 if "f64" in u[0] else 1 if "inst" in u[0] else 2,
                          -int(u[0].split("_")[3]) if "inst" in u[0] else 0, u[0]))


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libtimemg_b200.so in-tree for sm_100a (skipped when up to date)."""
    from concurrent.futures import ThreadPoolExecutor

    stamp = LIB_PATH + ".flags"
    flags_key = " ".join(NVCC_FLAGS)
    same_flags = os.path.exists(stamp) and open(stamp).read() == flags_key
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    # objects stay outside the tree (they need not travel with the snapshot)
    objdir = os.environ.get("TMG_OBJDIR", "/tmp/tmg_b200_obj")
    os.makedirs(objdir, exist_ok=True)

    def unit_newest(src):
        """newest mtime of a unit's source and the headers it includes (recursively)."""
        seen, todo = set(), [os.path.join(CSRC, src)]
        while todo:
            p = todo.pop()
            if p in seen or not os.path.exists(p):
                continue
            seen.add(p)
            for line in open(p, errors="replace"):
                line = line.strip()
                if line.startswith("#include \""):
                    name = line.split('"')[1]
                    todo += [os.path.join(CSRC, name), os.path.join(INCLUDE, name)]
        return max(os.path.getmtime(p) for p in seen)

    def stale(unit):
        obj = os.path.join(objdir, unit[0] + ".o")
        return force or not same_flags or not os.path.exists(obj) or \
            os.path.getmtime(obj) < unit_newest(unit[1])

    todo_units = [u for u in UNITS if stale(u)]
    if not todo_units and os.path.exists(LIB_PATH) and \
            os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(os.path.join(objdir, u[0] + ".o"))
                                              for u in UNITS):
        return LIB_PATH

    def compile_unit(unit):
        name, src, defs = unit
        obj = os.path.join(objdir, name + ".o")
        if unit not in todo_units:
            return obj
        extra = os.environ.get("TMG_NVCC_EXTRA", "").split()  # experiments: e.g. -DTMG_P2_WARPS=8
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-c", *defs, "-I", INCLUDE, "-I", CSRC, "-o", obj,
               os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"nvcc failed for {name}:\n{r.stderr[-4000:]}")
        return obj

    jobs = max(1, min(len(UNITS), os.cpu_count() or 1))
    with ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(compile_unit, UNITS))
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB_PATH + ".tmp",
           *objs]
    subprocess.run(cmd, check=True)
    os.replace(LIB_PATH + ".tmp", LIB_PATH)
    with open(stamp, "w") as fh:
        fh.write(flags_key)
    return LIB_PATH


_lib = None

EXPORTS = ("tmg_last_error", "tmg_version", "tmg_device_check", "tmg_sweep", "tmg_residual",
           "tmg_down", "tmg_up", "tmg_coarse_solve", "tmg_resid_norm", "tmg_resid_sqsum", "tmg_trace_enable", "tmg_trace_read", "tmg_plan_create",
           "tmg_plan_create_multi",
           "tmg_plan_destroy", "tmg_plan_cycles", "tmg_plan_solve", "tmg_plan_solve_host",
           "tmg_plan_stats", "tmg_plan_info", "tmg_rhs_samples", "tmg_rhs_sines", "tmg_rhs_last_error",
           "tmg_plan_solve_host_stream")


def load():
    """Load the shared library (no GPU needed to load it)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run paper_1409_5254_b200._native.build() "
                           "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, ci, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_double)
    lp = ctypes.POINTER(LevelDesc)
    i32p = ctypes.POINTER(ctypes.c_int32)
    L.tmg_last_error.restype = ctypes.c_char_p
    L.tmg_version.restype = ci
    L.tmg_device_check.argtypes = [ci]
    L.tmg_sweep.argtypes = [ci, lp, vp, vp, vp, i64, ci, vp, vp]
    L.tmg_residual.argtypes = [ci, lp, vp, vp, vp, i64, vp]
    L.tmg_down.argtypes = [ci, lp, vp, vp, vp, vp, i64, ci, vp, vp]
    L.tmg_up.argtypes = [ci, lp, vp, vp, vp, vp, vp, i64, ci, vp, vp]
    L.tmg_coarse_solve.argtypes = [ci, lp, vp, vp, i64, ci, ci, vp]
    L.tmg_resid_norm.argtypes = [ci, lp, vp, vp, vp, i64, vp]
    L.tmg_resid_sqsum.argtypes = [ci, lp, vp, vp, i64, vp, i64, vp]
    L.tmg_trace_enable.argtypes = [ci]
    L.tmg_trace_read.argtypes = [ctypes.c_char_p, i64]
    L.tmg_trace_read.restype = i64
    L.tmg_plan_create.argtypes = [ctypes.POINTER(vp), lp, ci, i64, ctypes.POINTER(PlanOpts)]
    L.tmg_plan_create_multi.argtypes = [ctypes.POINTER(vp), lp, ci, i64, ctypes.POINTER(PlanOpts)]
    L.tmg_plan_destroy.argtypes = [vp]
    L.tmg_plan_cycles.argtypes = [vp, vp, vp, ci, vp]
    L.tmg_plan_solve.argtypes = [vp, vp, vp, dp, ctypes.c_double, ci, vp]
    L.tmg_plan_solve_host.argtypes = [vp, vp, vp, vp, dp, ctypes.c_double, ci]
    L.tmg_plan_stats.argtypes = [vp, i32p, dp, i32p]
    L.tmg_plan_solve_host_stream.argtypes = [vp, ci, ctypes.POINTER(vp), ctypes.POINTER(vp), dp,
                                             ctypes.c_double, ci, i32p, dp, i32p]
    L.tmg_plan_info.argtypes = [vp, i32p, i32p, i32p]
    L.tmg_rhs_last_error.restype = ctypes.c_char_p
    L.tmg_rhs_samples.argtypes = [vp, vp, dp, dp, dp, ci, ci, vp, i64, i64, vp]
    L.tmg_rhs_sines.argtypes = [vp, vp, vp, dp, ci, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                dp, dp, dp, ci, ci, vp, i64, i64, vp]
    for name in EXPORTS:
        getattr(L, name).restype = getattr(L, name).restype or ci
    _lib = L
    return L


def check(rc: int, what: str = "timemg_b200"):
    if rc == 0:
        return
    msg = load().tmg_last_error().decode(errors="replace")
    if rc == E_ARG:
        raise ValueError(f"{what}: {msg}")
    if rc == E_UNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: CUDA error {rc}: {msg}")


def level_desc(ops, n_slabs: int, omega: float = 1.0, r1=None, r2=None) -> LevelDesc:
    import numpy as np

    d = LevelDesc()
    nt = int(ops.n_t)
    if not 1 <= nt <= KERNEL_MAXNT:
        # the kernels are instantiated for n_t = 1..4 (p_t <= 3); refuse before
        # any copy into the fixed-size fields
        raise NotImplementedError(f"n_t = {nt} (p_t = {nt - 1}): the GPU kernels support "
                                  f"n_t in 1..{KERNEL_MAXNT}")
    d.n_t = nt
    d.n_slabs = int(n_slabs)
    d.omega = float(omega)
    d.has_transfer = int(r1 is not None)

    def put(field, m):
        vals = np.ascontiguousarray(m, dtype=np.float64).ravel()
        if vals.size != nt * nt or vals.size > len(field):
            raise ValueError(f"level matrix of {vals.size} entries, expected {nt}x{nt}")
        ctypes.memmove(ctypes.addressof(field), vals.ctypes.data, vals.nbytes)

    put(d.minus_step, ops.minus_step_matrix)
    put(d.coupling, ops.coupling)
    put(d.lu, ops.lu.lu)
    if r1 is not None:
        put(d.r1, r1)
        put(d.r2, r2)
    for i, p in enumerate(ops.lu.perm):
        d.perm[i] = int(p)
    return d
