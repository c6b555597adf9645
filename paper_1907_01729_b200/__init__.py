"""B200-native batched log-domain Sinkhorn loss (arXiv 1907.01729).

Public API (mirrors the reference's ``sinkhornLoss`` node and the
``sinkloss.batch`` engine):

* :func:`sinkhorn_loss` -- differentiable per-lane E0 loss (loss.ts:59-131);
* :func:`solve` -- forward only, returning potentials / iterations / residuals;
* :func:`batch_forward`, :func:`batch_backward`, :func:`fused_log_reduction`,
  :class:`SinkhornConfig` -- the ``sinkloss.batch`` surface (batch.py);
* :class:`GridCost` -- on-the-fly squared-Euclidean grid cost; a 3-D cost
  tensor selects per-sample costs; :class:`PointCloudCost` -- squared
  Euclidean between point clouds (x.y on the tensor cores).

All compute runs in the sm_100a library ``_lib/libsinkhorn_b200.so`` behind
the C ABI declared in ``include/sinkhorn_b200.h``; importing this package
does not load it, the first call does (and fails loudly if it is missing).
"""

from .batch import (
    BatchLossResult,
    SinkhornConfig,
    batch_backward,
    batch_forward,
    fused_log_reduction,
    partial_log_reduction,
)
from .errors import (
    DeviceError,
    InvalidConfig,
    InvalidCost,
    InvalidHistogram,
    NaNProduced,
    ShapeMismatch,
    SinklossError,
    ZeroMassGradient,
)
from .loss import GridCost, PointCloudCost, SinkhornLossFunction, SolveResult, plan_gradient, \
    potentials_backward, sinkhorn_loss, solve, solve_streamed

__version__ = "0.1.0"

__all__ = [
    "BatchLossResult", "DeviceError", "GridCost", "InvalidConfig", "InvalidCost", "PointCloudCost",
    "InvalidHistogram", "NaNProduced", "ShapeMismatch", "SinkhornConfig",
    "SinkhornLossFunction", "SinklossError", "SolveResult", "ZeroMassGradient",
    "batch_backward", "batch_forward", "fused_log_reduction", "partial_log_reduction",
    "plan_gradient", "potentials_backward", "sinkhorn_loss", "solve", "solve_streamed",
]
