"""The C-ABI library loads and exports exactly what include/sinkhorn_b200.h
declares; host-side contract logic.  No GPU compute is called here."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "sinkhorn_b200.h")


def _declared_functions() -> list[str]:
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sinkhorn_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1907_01729_b200 import _build, _lib

    if not os.path.exists(_build.lib_path()):
        _build.build()
    return _lib.load()


def test_header_declares_the_reference_ffi_pair():
    names = _declared_functions()
    # ffi.ts:80 and ffi.ts:143 -- the drop-in symbols keep the reference's names
    assert "sinkhorn_forward_v1" in names
    assert "sinkhorn_backward_v1" in names


def test_library_exports_every_declared_symbol(lib):
    from paper_1907_01729_b200 import _lib

    declared = _declared_functions()
    assert sorted(_lib.EXPORTED_SYMBOLS) == declared
    for name in declared:
        assert hasattr(lib, name), name


def test_library_exports_nothing_else(lib):
    import subprocess

    from paper_1907_01729_b200 import _build

    out = subprocess.run(["nm", "-D", "--defined-only", _build.lib_path()],
                         capture_output=True, text=True).stdout
    text = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert text == set(_declared_functions())


def test_version_and_no_error(lib):
    from paper_1907_01729_b200 import _lib

    assert _lib.version().startswith("paper_1907_01729_b200")
    assert "sm_100a" in _lib.version()


def test_status_codes_match_reference_ffi():
    """ffi.ts:21-25."""
    from paper_1907_01729_b200 import _lib

    assert (_lib.STATUS_OK, _lib.STATUS_SHAPE_MISMATCH, _lib.STATUS_INVALID_HISTOGRAM,
            _lib.STATUS_NON_FINITE_OUTPUT, _lib.STATUS_ZERO_MASS_LANE) == (0, 10, 11, 12, 13)
    src = open(HEADER).read()
    for name, val in [("OK", 0), ("SHAPE_MISMATCH", 10), ("INVALID_HISTOGRAM", 11),
                      ("NON_FINITE_OUTPUT", 12), ("ZERO_MASS_LANE", 13)]:
        assert re.search(rf"#define SINKHORN_STATUS_{name} {val}\b", src)


def _view(a):
    from paper_1907_01729_b200 import _lib

    v = _lib.View()
    v.data = a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    v.ndim = a.ndim
    v.shape[0] = a.shape[0]
    v.shape[1] = a.shape[1] if a.ndim == 2 else 0
    v.length = a.size
    return v


def test_host_abi_shape_checks_need_no_gpu(lib):
    """ffi.ts:91-106 shape mismatches return 10 before any device work;
    B = 0 is a successful no-op (ffi.ts:107-109)."""
    mu = np.array([[0.5, 0.5]])
    nu = np.array([[0.3, 0.3, 0.4]])
    c_bad = np.zeros((2, 2))
    out_c, lu, lv = np.zeros(1), np.zeros((1, 2)), np.zeros((1, 3))
    vs = [_view(a) for a in (mu, nu, c_bad, out_c, lu, lv)]
    st = lib.sinkhorn_forward_v1(*[ctypes.byref(v) for v in vs[:3]], 0.1, 10, 0.0,
                                 *[ctypes.byref(v) for v in vs[3:]])
    assert st == 10
    z = [np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((3, 3)), np.zeros(0), np.zeros((0, 3)),
         np.zeros((0, 3))]
    vz = [_view(a) for a in z]
    st = lib.sinkhorn_forward_v1(*[ctypes.byref(v) for v in vz[:3]], 0.1, 10, 0.0,
                                 *[ctypes.byref(v) for v in vz[3:]])
    assert st == 0
    # backward: upstream (3,) for B = 2 -> 10 (ffi.test.ts:263-273)
    b = [np.zeros((2, 2)), np.zeros((2, 2)), np.zeros(3), np.zeros((2, 2)), np.zeros((2, 2))]
    vb = [_view(a) for a in b]
    st = lib.sinkhorn_backward_v1(ctypes.byref(vb[0]), ctypes.byref(vb[1]), 0.5,
                                  ctypes.byref(vb[2]), ctypes.byref(vb[3]), ctypes.byref(vb[4]))
    assert st == 10


def test_capacity_check_like_viewok(lib):
    """ffi.ts:33-38: offset + size must fit in the buffer."""
    mu = np.array([[0.5, 0.5]])
    nu = np.array([[0.5, 0.5]])
    c = np.array([[0.0, 1.0], [1.0, 0.0]])
    out_c, lu, lv = np.zeros(1), np.zeros((1, 2)), np.zeros((1, 2))
    vs = [_view(a) for a in (mu, nu, c, out_c, lu, lv)]
    vs[4].length = 1    # log_u view too short
    st = lib.sinkhorn_forward_v1(*[ctypes.byref(v) for v in vs[:3]], 0.1, 10, 0.0,
                                 *[ctypes.byref(v) for v in vs[3:]])
    assert st == 10


def test_workspace_query_is_host_only(lib):
    from paper_1907_01729_b200 import _lib

    pr = _lib.Problem()
    pr.B, pr.d1, pr.d2, pr.cost_kind = 256, 784, 784, _lib.COST_SHARED
    n = lib.sinkhorn_workspace_bytes_v1(ctypes.byref(pr))
    # A2 + A2^T dominate: 2 * 832^2 floats
    assert n >= 2 * 832 * 832 * 4
    pr.cost_kind = 7
    assert lib.sinkhorn_workspace_bytes_v1(ctypes.byref(pr)) == 0
    pr.cost_kind = _lib.COST_GRID2D
    pr.grid_nx, pr.grid_ny = 28, 28
    assert lib.sinkhorn_workspace_bytes_v1(ctypes.byref(pr)) > 0
    pr.grid_nx = 27     # nx*ny != d
    assert lib.sinkhorn_workspace_bytes_v1(ctypes.byref(pr)) == 0


def test_product_path_never_imports_the_oracle():
    """The oracle is test infrastructure only (task contract): no product
    module imports it, and no CUDA source includes anything from it."""
    pkg = os.path.join(ROOT, "paper_1907_01729_b200")
    pat = re.compile(r"^\s*(from\s+oracle\b|import\s+oracle\b|from\s+\.+oracle\b)|"
                     r"#include\s+[\"<][^\">]*oracle", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                assert not pat.search(open(os.path.join(dirpath, f)).read()), f
