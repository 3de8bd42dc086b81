"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/timemg_b200.h declares; struct layouts agree with the header."""

import ctypes
import os
import re

import pytest

from paper_1409_5254_b200 import _native as nat

HEADER = os.path.join(nat.INCLUDE, "timemg_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tmg_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(nat.LIB_PATH):
        nat.build()
    return nat.load()


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(nat.EXPORTS)


def test_version_and_errors_without_gpu(lib):
    assert lib.tmg_version() == 100
    # argument validation happens before any CUDA call
    d = nat.LevelDesc()
    d.n_t = 9
    d.n_slabs = 4
    rc = lib.tmg_sweep(0, ctypes.byref(d), None, None, None, 1, -1, None, None)
    assert rc == nat.E_ARG
    assert b"sweep count" in lib.tmg_last_error()
    rc = lib.tmg_residual(0, ctypes.byref(d), None, None, None, 1, None)
    assert rc == nat.E_UNSUPPORTED
    with pytest.raises(NotImplementedError):
        nat.check(rc)


def test_struct_layout_matches_header():
    # tmg_level_desc: 2 x int32, int64, double, 5 x 64 doubles, 8 x int32
    assert ctypes.sizeof(nat.LevelDesc) == 4 + 4 + 8 + 8 + 5 * 64 * 8 + 8 * 4
    assert nat.LevelDesc.n_slabs.offset == 8
    assert nat.LevelDesc.minus_step.offset == 24
    assert ctypes.sizeof(nat.PlanOpts) == 8 * 4


def test_level_desc_packing():
    import numpy as np
    from paper_1409_5254_b200 import assemble_local, BasisSpec, build_transfers
    ops = assemble_local(BasisSpec(2), 0.01)
    r1, r2 = build_transfers(BasisSpec(2), 0.01)
    d = nat.level_desc(ops, 64, 0.7, r1, r2)
    assert d.n_t == 3 and d.n_slabs == 64 and d.has_transfer == 1
    assert list(d.minus_step[:9]) == list(np.asarray(ops.minus_step_matrix).ravel())
    assert list(d.r2[:9]) == list(r2.ravel())
    assert list(d.perm[:3]) == list(ops.lu.perm)


def test_level_desc_rejects_unsupported_degree():
    from paper_1409_5254_b200 import assemble_local, BasisSpec
    with pytest.raises(NotImplementedError):
        nat.level_desc(assemble_local(BasisSpec(4), 0.1), 8)  # n_t = 5: no kernels
    with pytest.raises(NotImplementedError):
        nat.level_desc(assemble_local(BasisSpec(8), 0.1), 8)  # n_t = 9 > TMG_MAXNT


def test_rhs_entry_points_validate_without_gpu(lib):
    import numpy as np
    dp = ctypes.POINTER(ctypes.c_double)
    z = np.zeros(16)
    p = z.ctypes.data_as(dp)
    rc = lib.tmg_rhs_samples(None, None, p, p, p, 9, 9, None, 4, 1, None)
    assert rc == nat.E_ARG and b"n_t" in lib.tmg_rhs_last_error()
    rc = lib.tmg_rhs_sines(None, None, None, p, 8, -1.0, 0.1, 0.0, p, p, p, 2, 2, None, 4, 1, None)
    assert rc == nat.E_ARG


def test_stream_split_and_phase_buckets(monkeypatch):
    """host logic of the streamed host pipeline and of SolveStats.times:
    sub-batches per batch (halves from 32 problems up, env override that must
    divide B) and the kernel-name -> phase mapping of the traced solve"""
    from paper_1409_5254_b200 import solver
    monkeypatch.delenv("TMG_STREAM_SPLIT", raising=False)
    assert solver._stream_split(64) == 2 and solver._stream_split(32) == 2
    assert solver._stream_split(16) == 1 and solver._stream_split(33) == 1 and solver._stream_split(1) == 1
    monkeypatch.setenv("TMG_STREAM_SPLIT", "4")
    assert solver._stream_split(64) == 4 and solver._stream_split(6) == 1
    assert solver._phase_bucket("tail_kernel") == "coarse"
    assert solver._phase_bucket("stream_kernel_v (level-1 up + finest up + next finest down)") == "smoothing"
    assert solver._phase_bucket("stream_kernel<nt=2,nu=1,kind=1> n=2048 flags=135") == "smoothing"
    assert solver._phase_bucket("finalize") == "residual" and solver._phase_bucket("set_active") == "residual"
    assert set(solver._times(1.5)) == {"smoothing", "transfer", "coarse", "residual"}
