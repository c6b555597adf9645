"""ctypes binding of the C ABI in include/sinkhorn_b200.h.

The library is the product: there is no Python or CPU fallback.  If the
shared object is missing or does not export every declared symbol, loading
fails loudly with an ImportError that says how to build it.
"""

from __future__ import annotations

import ctypes
import os
import threading

from ._build import lib_path

STATUS_OK = 0
STATUS_SHAPE_MISMATCH = 10
STATUS_INVALID_HISTOGRAM = 11
STATUS_NON_FINITE_OUTPUT = 12
STATUS_ZERO_MASS_LANE = 13
STATUS_INVALID_CONFIG = 14
STATUS_INVALID_COST = 15
STATUS_BAD_ARGUMENT = 16
STATUS_WORKSPACE = 17
STATUS_EXACT_NEEDED = 18
STATUS_CUDA_ERROR = 20

COST_SHARED = 0
COST_PER_SAMPLE = 1
COST_GRID2D = 2
COST_POINTS = 3

FLAG_SKIP_VALIDATION = 1
FLAG_TIME_LOOP = 4
FLAG_EXACT_MAX = 8
FLAG_MUFU_ONLY = 16
FLAG_PERSISTENT = 32
FLAG_TILED_ONLY = 64
FLAG_DENSE_GRID = 128
FLAG_NO_FUSED = 256
FLAG_NO_GEMM = 512
FLAG_FORCE_GEMM = 1024
FLAG_TIME_KERNEL = 2048
FLAG_FORCE_RERUN = 4096

# every symbol include/sinkhorn_b200.h declares
EXPORTED_SYMBOLS = (
    "sinkhorn_forward_v1",
    "sinkhorn_backward_v1",
    "sinkhorn_workspace_bytes_v1",
    "sinkhorn_forward_device_v1",
    "sinkhorn_forward_warm_device_v1",
    "sinkhorn_backward_device_v1",
    "sinkhorn_workspace_bytes_f64_v1",
    "sinkhorn_forward_f64_device_v1",
    "sinkhorn_backward_f64_device_v1",
    "sinkhorn_half_sweep_workspace_bytes_v1",
    "sinkhorn_half_sweep_device_v1",
    "sinkhorn_plan_grad_device_v1",
    "sinkhorn_e0_partial_device_v1",
    "sinkhorn_set_residual_reducer_v1",
    "sinkhorn_forward_rows_device_v1",
    "sinkhorn_forward_async_device_v1",
    "sinkhorn_plan_grad_workspace_bytes_v1",
    "sinkhorn_plan_grad_ws_device_v1",
    "sinkhorn_last_error",
    "sinkhorn_version",
    "sinkhorn_launch_count_v1",
    "sinkhorn_exact_reruns_v1",
    "sinkhorn_last_loop_ms_v1",
    "sinkhorn_last_kernel_ms_v1",
    "sinkhorn_last_path_v1",
)


class View(ctypes.Structure):
    """sinkhorn_view_v1: row-major float64 view (ffi.ts:15-19 TensorView)."""

    _fields_ = [
        ("data", ctypes.POINTER(ctypes.c_double)),
        ("ndim", ctypes.c_int32),
        ("shape", ctypes.c_int64 * 2),
        ("length", ctypes.c_int64),
    ]


class Problem(ctypes.Structure):
    _fields_ = [
        ("B", ctypes.c_int64),
        ("d1", ctypes.c_int64),
        ("d2", ctypes.c_int64),
        ("cost_kind", ctypes.c_int32),
        ("grid_nx", ctypes.c_int32),
        ("grid_ny", ctypes.c_int32),
        ("grid_hx", ctypes.c_float),
        ("grid_hy", ctypes.c_float),
    ]


class Options(ctypes.Structure):
    _fields_ = [
        ("lam", ctypes.c_double),
        ("max_iters", ctypes.c_int32),
        ("check_interval", ctypes.c_int32),
        ("tolerance", ctypes.c_double),
        ("flags", ctypes.c_uint32),
    ]


# double (*)(double local_max, void* user)
REDUCER = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.c_double, ctypes.c_void_p)
# void (*)(float* data, int64_t count, int32_t op, void* stream, void* user)
ALLREDUCE = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                             ctypes.c_void_p, ctypes.c_void_p)
REDUCE_SUM = 0

_lock = threading.Lock()
_lib = None

P = ctypes.c_void_p
VP = ctypes.POINTER(View)


def _declare(lib):
    i32, i64, f64, sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t
    sig = {
        "sinkhorn_forward_v1": (i32, [VP, VP, VP, f64, i32, f64, VP, VP, VP]),
        "sinkhorn_backward_v1": (i32, [VP, VP, f64, VP, VP, VP]),
        "sinkhorn_workspace_bytes_v1": (sz, [ctypes.POINTER(Problem)]),
        "sinkhorn_forward_device_v1": (
            i32, [ctypes.POINTER(Problem), ctypes.POINTER(Options), P, P, P, P, P, P,
                  ctypes.POINTER(ctypes.c_int32), P, P, sz, P]),
        "sinkhorn_forward_warm_device_v1": (
            i32, [ctypes.POINTER(Problem), ctypes.POINTER(Options), P, P, P, P, P, P, P,
                  ctypes.POINTER(ctypes.c_int32), P, P, sz, P]),
        "sinkhorn_backward_device_v1": (
            i32, [i64, i64, i64, f64, P, P, P, P, P, ctypes.POINTER(ctypes.c_int32), P, sz, P]),
        "sinkhorn_workspace_bytes_f64_v1": (sz, [ctypes.POINTER(Problem)]),
        "sinkhorn_forward_f64_device_v1": (
            i32, [ctypes.POINTER(Problem), ctypes.POINTER(Options), P, P, P, P, P, P,
                  ctypes.POINTER(ctypes.c_int32), P, P, sz, P]),
        "sinkhorn_backward_f64_device_v1": (
            i32, [i64, i64, i64, f64, P, P, P, P, P, ctypes.POINTER(ctypes.c_int32), P, sz, P]),
        "sinkhorn_half_sweep_workspace_bytes_v1": (sz, [i64, i64, i64]),
        "sinkhorn_half_sweep_device_v1": (i32, [i64, i64, i64, f64, P, P, P, P, P, P, P, sz, P]),
        "sinkhorn_plan_grad_device_v1": (i32, [ctypes.POINTER(Problem), f64, P, P, P, P, P, P]),
        "sinkhorn_plan_grad_workspace_bytes_v1": (sz, [ctypes.POINTER(Problem)]),
        "sinkhorn_plan_grad_ws_device_v1": (
            i32, [ctypes.POINTER(Problem), f64, P, P, P, P, P, P, sz, P]),
        "sinkhorn_e0_partial_device_v1": (i32, [i64, i64, i64, f64, P, P, P, P, P, sz, P]),
        "sinkhorn_set_residual_reducer_v1": (None, [REDUCER, P]),
        "sinkhorn_forward_async_device_v1": (
            i32, [ctypes.POINTER(Problem), ctypes.POINTER(Options), P, P, P, P, P, P, P, P, P, sz,
                  P]),
        "sinkhorn_forward_rows_device_v1": (
            i32, [ctypes.POINTER(Problem), ctypes.POINTER(Options), P, P, P, P, P, P,
                  ctypes.POINTER(ctypes.c_int32), P, ALLREDUCE, P, P, sz, P]),
        "sinkhorn_last_error": (ctypes.c_char_p, []),
        "sinkhorn_version": (ctypes.c_char_p, []),
        "sinkhorn_launch_count_v1": (ctypes.c_ulonglong, []),
        "sinkhorn_exact_reruns_v1": (ctypes.c_ulonglong, []),
        "sinkhorn_last_loop_ms_v1": (ctypes.c_float, []),
        "sinkhorn_last_kernel_ms_v1": (ctypes.c_float, [ctypes.POINTER(ctypes.c_int32)]),
        "sinkhorn_last_path_v1": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def load():
    """Load the sm_100a library (no fallback); raises ImportError when absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("SINKHORN_B200_LIB") or lib_path()   # override: experiments
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: the B200 kernels are not built. "
                "Run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(nvcc, sm_100a). There is no CPU fallback.")
        lib = ctypes.CDLL(path, mode=ctypes.RTLD_LOCAL)
        missing = [s for s in EXPORTED_SYMBOLS if not hasattr(lib, s)]
        if missing:
            raise ImportError(f"{path} lacks symbols {missing}")
        _declare(lib)
        _lib = lib
        return lib


def last_error() -> str:
    return load().sinkhorn_last_error().decode("utf-8", "replace")


def version() -> str:
    return load().sinkhorn_version().decode()
