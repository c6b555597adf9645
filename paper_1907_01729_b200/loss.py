"""PyTorch-facing Sinkhorn loss over the sm_100a C ABI.

Mirrors the reference's differentiable node ``sinkhornLoss``
(pkg/frontend/src/loss.ts:59-131): forward solves every lane through the
C-ABI forward and saves only the final log potentials (loss.ts:104);
backward turns them into mean-zero gradients through the C-ABI backward
without re-running anything (loss.ts:105-128), so autograd memory does not
depend on the iteration count.

PyTorch supplies device memory (the caching allocator backs the solver
workspace), the stream, and autograd; every arithmetic operation on the
path is one of the library's kernels.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from .errors import InvalidConfig, ShapeMismatch, raise_for_status


@dataclass(frozen=True)
class GridCost:
    """Squared Euclidean cost on an nx x ny grid, recomputed on the fly.

    Point k sits at ((k % nx) * hx, (k // nx) * hy); the default spacing
    1/(n-1) puts the grid on the unit square (BASELINE config 3).
    """

    nx: int
    ny: int
    hx: float | None = None
    hy: float | None = None

    @property
    def d(self) -> int:
        return self.nx * self.ny

    def spacing(self) -> tuple[float, float]:
        hx = self.hx if self.hx is not None else 1.0 / max(self.nx - 1, 1)
        hy = self.hy if self.hy is not None else 1.0 / max(self.ny - 1, 1)
        return float(hx), float(hy)

    def materialize(self, device=None, dtype=torch.float64) -> torch.Tensor:
        """The (d, d) matrix this descriptor stands for (tests / dC only)."""
        hx, hy = self.spacing()
        k = torch.arange(self.d, device=device)
        x = (k % self.nx).to(dtype) * hx
        y = (k // self.nx).to(dtype) * hy
        return (x[:, None] - x[None, :]) ** 2 + (y[:, None] - y[None, :]) ** 2


@dataclass(frozen=True)
class PointCloudCost:
    """Squared Euclidean cost between point clouds: c_ij = |x_i - y_j|^2.

    x (d1, D) and y (d2, D) are the histograms' support points.  The library
    evaluates |x|^2 + |y|^2 - 2 x.y with the x.y contraction on the tensor
    cores (3xTF32) and then solves with the materialised cost (PAPER.md:147,
    SPEC.md:13).
    """

    x: torch.Tensor
    y: torch.Tensor

    @property
    def dim(self) -> int:
        return int(self.x.shape[1])

    def packed(self, device) -> torch.Tensor:
        """[x; y] as one contiguous float32 (d1 + d2, D) device tensor."""
        x = torch.as_tensor(self.x).to(device=device, dtype=torch.float32)
        y = torch.as_tensor(self.y).to(device=device, dtype=torch.float32)
        return torch.cat([x, y], dim=0).contiguous()

    def materialize(self, device=None, dtype=torch.float64) -> torch.Tensor:
        """The (d1, d2) matrix this descriptor stands for (tests only)."""
        x = torch.as_tensor(self.x).to(device=device, dtype=dtype)
        y = torch.as_tensor(self.y).to(device=device, dtype=dtype)
        return ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)


@dataclass
class SolveResult:
    """Per-lane E0 costs plus the complete backward state (batch.py:237-253)."""

    cost_e0: torch.Tensor     # (B,)
    log_u: torch.Tensor       # (B, d1)
    log_v: torch.Tensor       # (B, d2)
    lam: float
    iterations_run: int
    residuals: torch.Tensor   # (B,)
    loop_ms: float = -1.0     # iteration-loop time (CUDA events) when solve(time_loop=True)
    path: str = ""            # solver path taken ("small", "tiled", "persistent", "lane")
    kernel_ms: float = -1.0   # dominant kernel's launches (CUDA events), solve(time_kernel=True)
    kernel_launches: int = 0
    device_status: torch.Tensor | None = None   # solve(asynchronous=True): int32 on the device

    def check(self) -> "SolveResult":
        """An asynchronous solve's device status -> the reference's exception
        (waits for the solve).  A no-op for synchronous solves."""
        if self.device_status is not None:
            st = int(self.device_status.item())
            if st != 0:
                _lib.load()
                from .errors import _BY_STATUS, DeviceError

                raise _BY_STATUS.get(st, DeviceError)(f"asynchronous solve: device status {st}")
        return self


def _stream_handle(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


_WS_CACHE: dict = {}


def _workspace(dev: torch.device, nbytes: int) -> torch.Tensor:
    """Per-(device, stream) workspace, grown on demand and reused across calls
    (stream-ordered reuse is safe; calls on other streams get their own)."""
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    ws = _WS_CACHE.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 256), device=dev, dtype=torch.uint8)
        _WS_CACHE[key] = ws
    return ws


_AUX_STREAMS: dict = {}


def _aux_stream(dev: torch.device, k: int) -> torch.cuda.Stream:
    """Long-lived extra compute streams (their workspaces are cached per stream)."""
    key = (dev, k)
    if key not in _AUX_STREAMS:
        _AUX_STREAMS[key] = torch.cuda.Stream(dev)
    return _AUX_STREAMS[key]


def _as_f32_cuda(x, device=None) -> torch.Tensor:
    t = torch.as_tensor(x)
    if device is None:
        device = t.device if t.is_cuda else torch.device("cuda", torch.cuda.current_device())
    return t.to(device=device, dtype=torch.float32).contiguous()


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _problem(B: int, d1: int, d2: int, cost) -> _lib.Problem:
    pr = _lib.Problem()
    pr.B, pr.d1, pr.d2 = B, d1, d2
    if isinstance(cost, GridCost):
        hx, hy = cost.spacing()
        pr.cost_kind = _lib.COST_GRID2D
        pr.grid_nx, pr.grid_ny = cost.nx, cost.ny
        pr.grid_hx, pr.grid_hy = hx, hy
    elif isinstance(cost, PointCloudCost):
        pr.cost_kind = _lib.COST_POINTS
        pr.grid_nx = cost.dim
    elif cost.dim() == 3:
        pr.cost_kind = _lib.COST_PER_SAMPLE
    else:
        pr.cost_kind = _lib.COST_SHARED
    return pr


def _check_shapes(mu: torch.Tensor, nu: torch.Tensor, cost) -> tuple[int, int, int]:
    if mu.dim() != 2 or nu.dim() != 2:
        raise ShapeMismatch("mu and nu must be 2-D (batch, dim)")
    B, d1 = mu.shape
    if nu.shape[0] != B:
        raise ShapeMismatch(f"batch sizes differ: mu has {B}, nu has {nu.shape[0]}")
    d2 = nu.shape[1]
    if isinstance(cost, PointCloudCost):
        if cost.x.dim() != 2 or cost.y.dim() != 2 or cost.x.shape[1] != cost.y.shape[1]:
            raise ShapeMismatch("point clouds must be (d1, D) and (d2, D)")
        if cost.x.shape[0] != d1 or cost.y.shape[0] != d2:
            raise ShapeMismatch(f"point clouds have {cost.x.shape[0]} and {cost.y.shape[0]} points "
                                f"but histograms have d1={d1}, d2={d2}")
    elif isinstance(cost, GridCost):
        if cost.d != d1 or cost.d != d2:
            raise ShapeMismatch(f"grid has {cost.d} points but histograms have d1={d1}, d2={d2}")
    elif cost.dim() == 2:
        if tuple(cost.shape) != (d1, d2):
            raise ShapeMismatch(f"cost is {tuple(cost.shape)} but histograms have d1={d1}, d2={d2}")
    elif cost.dim() == 3:
        if tuple(cost.shape) != (B, d1, d2):
            raise ShapeMismatch(f"per-sample cost is {tuple(cost.shape)}, need ({B}, {d1}, {d2})")
    else:
        raise ShapeMismatch("cost must be (d1, d2), (B, d1, d2) or a GridCost")
    return B, d1, d2


def solve(mu, nu, cost, lam: float, max_iters: int = 1000, tolerance: float = 0.0,
          check_interval: int = 10, validate: bool = True, time_loop: bool = False,
          exact_max: bool = False, mufu_only: bool = False,
          persistent: bool = False, tiled_only: bool = False,
          dense_grid: bool = False, init_log_u=None, fused: bool = True,
          fp64: bool = False, gemm: bool | None = None,
          time_kernel: bool = False, asynchronous: bool = False,
          force_rerun: bool = False, out=None) -> SolveResult:
    """batch_forward (batch.py:264-349) on the GPU.

    mu (B, d1), nu (B, d2) histograms; cost a (d1, d2) tensor shared by all
    lanes, a (B, d1, d2) per-sample tensor, or a GridCost.  Inputs are cast
    to contiguous float32 on the current CUDA device.  ``exact_max`` forces
    the two-pass chunk reduction (no previous-iteration lse estimate).
    ``init_log_u`` (B, d1) warm-starts the iteration from a previous solve's
    log_u instead of 0 on the support (no reference API; batch.py:295).
    ``fused=False`` runs shared costs as two half-sweeps per iteration instead
    of the fused row->column pass (sweep_fused.cuh).  ``fp64=True`` runs the
    reference's float64 iteration on the device (sweep_f64.cuh): float64
    outputs, reaches the reference's default tolerance 1e-9; path "fp64".
    ``gemm``: None (default) takes the two-GEMM iteration (sweep_gemm.cuh) for
    shared costs larger than the fused pass handles; True forces it for any
    shared cost, False never takes it.  ``time_kernel`` records CUDA events
    around every launch of the solve's dominant kernel (``kernel_ms``,
    ``kernel_launches``; measurement only -- the events break the launch
    overlap).  ``asynchronous=True`` (tolerance 0): the call returns once the
    solve is enqueued on the current stream -- no host synchronisation; the
    estimate-guard rerun is decided on the device; device-detected errors are
    raised by ``result.check()`` (``iterations_run`` is ``max_iters``).
    ``force_rerun`` (diagnostics) exercises the exact-rerun machinery.
    ``out``: optional preallocated (cost (B,), log_u (B, d1), log_v (B, d2),
    residuals (B,)) float32 device tensors to write into.
    """
    if fp64:
        return _solve_f64(mu, nu, cost, lam, max_iters, tolerance, check_interval, validate)
    mu, nu = torch.as_tensor(mu), torch.as_tensor(nu)
    if not isinstance(cost, (GridCost, PointCloudCost)):
        cost = torch.as_tensor(cost)
    B, d1, d2 = _check_shapes(mu, nu, cost)   # host-side, before touching the device
    mu = _as_f32_cuda(mu)
    dev = mu.device
    nu = _as_f32_cuda(nu, dev)
    if isinstance(cost, GridCost):
        cost_buf = None                      # recomputed on the fly
    elif isinstance(cost, PointCloudCost):
        cost_buf = cost.packed(dev)          # [x; y]
    else:
        cost = cost_buf = _as_f32_cuda(cost, dev)
    lib = _lib.load()
    pr = _problem(B, d1, d2, cost)
    op = _lib.Options()
    op.lam, op.max_iters, op.check_interval, op.tolerance = float(lam), int(max_iters), \
        int(check_interval), float(tolerance)
    op.flags = (0 if validate else _lib.FLAG_SKIP_VALIDATION) | \
        (_lib.FLAG_TIME_LOOP if time_loop else 0) | (_lib.FLAG_EXACT_MAX if exact_max else 0) | \
        (_lib.FLAG_MUFU_ONLY if mufu_only else 0) | (_lib.FLAG_PERSISTENT if persistent else 0) | \
        (_lib.FLAG_TILED_ONLY if tiled_only else 0) | (_lib.FLAG_DENSE_GRID if dense_grid else 0) | \
        (0 if fused else _lib.FLAG_NO_FUSED) | \
        (_lib.FLAG_FORCE_GEMM if gemm else 0) | (_lib.FLAG_NO_GEMM if gemm is False else 0) | \
        (_lib.FLAG_TIME_KERNEL if time_kernel else 0) | \
        (_lib.FLAG_FORCE_RERUN if force_rerun else 0)
    if out is not None:
        out_cost, log_u, log_v, residuals = out
        for t, shp in zip(out, ((B,), (B, d1), (B, d2), (B,))):
            if tuple(t.shape) != shp or t.dtype != torch.float32 or not t.is_contiguous() \
                    or t.device != dev:
                raise ShapeMismatch(f"out tensor must be contiguous float32 {shp} on {dev}")
    else:
        out_cost = torch.empty(B, device=dev, dtype=torch.float32)
        log_u = torch.empty(B, d1, device=dev, dtype=torch.float32)
        log_v = torch.empty(B, d2, device=dev, dtype=torch.float32)
        residuals = torch.empty(B, device=dev, dtype=torch.float32)
    with torch.cuda.device(dev):
        nbytes = lib.sinkhorn_workspace_bytes_v1(ctypes.byref(pr))
        ws = _workspace(dev, nbytes)
        iters = ctypes.c_int32(0)
        if asynchronous:
            if init_log_u is not None:
                raise ValueError("asynchronous solves start from u = 0 (no warm start)")
            dstat = torch.empty(1, device=dev, dtype=torch.int32)
            st = lib.sinkhorn_forward_async_device_v1(
                ctypes.byref(pr), ctypes.byref(op), _ptr(mu), _ptr(nu),
                _ptr(cost_buf), _ptr(out_cost), _ptr(log_u),
                _ptr(log_v), _ptr(residuals), _ptr(dstat), _ptr(ws), ws.numel(),
                _stream_handle(dev))
            raise_for_status(st, "sinkhorn_forward_async_device_v1")
            return SolveResult(out_cost, log_u, log_v, float(lam), int(max_iters), residuals,
                               -1.0, lib.sinkhorn_last_path_v1().decode(), device_status=dstat)
        if init_log_u is not None:
            init = _as_f32_cuda(init_log_u, dev)
            if tuple(init.shape) != (B, d1):
                raise ShapeMismatch(f"init_log_u must be ({B}, {d1}), got {tuple(init.shape)}")
            st = lib.sinkhorn_forward_warm_device_v1(
                ctypes.byref(pr), ctypes.byref(op), _ptr(mu), _ptr(nu),
                _ptr(cost_buf), _ptr(init), _ptr(out_cost),
                _ptr(log_u), _ptr(log_v), ctypes.byref(iters), _ptr(residuals), _ptr(ws),
                ws.numel(), _stream_handle(dev))
        else:
            st = lib.sinkhorn_forward_device_v1(
                ctypes.byref(pr), ctypes.byref(op), _ptr(mu), _ptr(nu),
                _ptr(cost_buf), _ptr(out_cost), _ptr(log_u),
                _ptr(log_v), ctypes.byref(iters), _ptr(residuals), _ptr(ws), ws.numel(),
                _stream_handle(dev))
    raise_for_status(st, "sinkhorn_forward_device_v1")
    loop_ms = float(lib.sinkhorn_last_loop_ms_v1()) if time_loop else -1.0
    path = lib.sinkhorn_last_path_v1().decode()
    kms, kn = -1.0, 0
    if time_kernel:
        n = ctypes.c_int32(0)
        kms, kn = float(lib.sinkhorn_last_kernel_ms_v1(ctypes.byref(n))), int(n.value)
    return SolveResult(out_cost, log_u, log_v, float(lam), int(iters.value), residuals, loop_ms,
                       path, kms, kn)


def solve_streamed(mu, nu, cost, lam: float, max_iters: int = 1000, tolerance: float = 0.0,
                   check_interval: int = 10, chunks=8, device=None,
                   validate: bool = True, compute_streams: int = 2) -> SolveResult:
    """``solve`` from host tensors, overlapping the host->device upload with the solve.

    mu (B, d1), nu (B, d2) and cost -- shared (d1, d2), per-sample (B, d1, d2),
    a GridCost or a PointCloudCost -- in host memory (pin it for full PCIe
    bandwidth).  At tolerance 0 the lanes are independent (test_batch.py:46-63),
    so the batch is solved in ``chunks`` lane groups through three rotating
    device buffers: group k+1 and k+2's histograms and per-sample costs are
    copied on a second stream while group k solves, and the solves are
    asynchronous (no host synchronisation until the end), so the copy engine
    never waits for the host.  With tolerance > 0 the lockstep stopping rule
    couples every lane (batch.py:318-322): one group, synchronous.
    ``chunks`` is a group count (equal groups) or a list of group sizes summing
    to B -- the pipeline's exposed ends are the first group's upload and the
    last group's solve, so short groups there shorten the step.  Consecutive
    groups alternate over ``compute_streams`` streams (each with its own
    workspace), so one group's kernel tails overlap the next one's.
    """
    mu, nu = torch.as_tensor(mu), torch.as_tensor(nu)
    grid = isinstance(cost, (GridCost, PointCloudCost))   # small descriptors: passed through
    if not grid:
        cost = torch.as_tensor(cost)
    B, d1, d2 = _check_shapes(mu, nu, cost)
    dev = torch.device(device) if device is not None else \
        torch.device("cuda", torch.cuda.current_device())
    per_sample = (not grid) and cost.dim() == 3
    asynchronous = tolerance == 0 and B > 0
    if not asynchronous:
        chunks = 1
    if isinstance(chunks, int):
        chunks = max(1, min(int(chunks), B if B else 1))
        bounds = [(B * k // chunks, B * (k + 1) // chunks) for k in range(chunks)]
    else:   # explicit lane-group sizes (e.g. a short first and last group)
        sizes = [int(n) for n in chunks if int(n) > 0]
        if sum(sizes) != B:
            raise InvalidConfig("solve_streamed: lane-group sizes must sum to B")
        edges = [sum(sizes[:k]) for k in range(len(sizes) + 1)]
        bounds = list(zip(edges[:-1], edges[1:]))
    chunks = len(bounds)
    nbuf = min(3, chunks)
    gmax = max(hi - lo for lo, hi in bounds) if B else 0
    compute = torch.cuda.current_stream(dev)
    streams = [compute] + [_aux_stream(dev, k) for k in range(
        max(0, min(int(compute_streams), chunks) - 1) if asynchronous else 0)]
    copy = torch.cuda.Stream(dev)
    f32 = dict(device=dev, dtype=torch.float32)
    bufs = [(torch.empty(gmax, d1, **f32), torch.empty(gmax, d2, **f32),
             torch.empty(gmax, d1, d2, **f32) if per_sample else None) for _ in range(nbuf)]
    shared = None if (grid or per_sample) else cost.to(**f32, non_blocking=True)
    ready = [torch.cuda.Event() for _ in range(nbuf)]
    free = [torch.cuda.Event() for _ in range(nbuf)]
    out_cost = torch.empty(B, **f32)
    log_u = torch.empty(B, d1, **f32)
    log_v = torch.empty(B, d2, **f32)
    residuals = torch.empty(B, **f32)

    def upload(k):
        lo, hi = bounds[k]
        m, n, c = bufs[k % nbuf]
        with torch.cuda.stream(copy):
            if k >= nbuf:
                copy.wait_event(free[k % nbuf])   # group k - nbuf has finished with it
            m[: hi - lo].copy_(mu[lo:hi], non_blocking=True)
            n[: hi - lo].copy_(nu[lo:hi], non_blocking=True)
            if c is not None:
                c[: hi - lo].copy_(cost[lo:hi], non_blocking=True)
            ready[k % nbuf].record(copy)

    iters, checks = 0, []
    with torch.cuda.device(dev):
        for k in range(min(nbuf, chunks)):
            upload(k)
        start = torch.cuda.Event()
        start.record(compute)   # the caller's prior work on its stream comes first
        for s_ in streams[1:]:
            s_.wait_event(start)
        if shared is not None:
            shared_ready = torch.cuda.Event()
            shared_ready.record(compute)
        for k, (lo, hi) in enumerate(bounds):
            m, n, c = bufs[k % nbuf]
            st = streams[k % len(streams)]
            st.wait_event(ready[k % nbuf])
            if shared is not None and st is not compute:
                st.wait_event(shared_ready)
            g = hi - lo
            cg = cost if grid else (c[:g] if per_sample else shared)
            # results straight into the slices of the outputs (contiguous lane ranges)
            with torch.cuda.stream(st):
                r = solve(m[:g], n[:g], cg, lam, max_iters, tolerance, check_interval,
                          validate=validate, asynchronous=asynchronous,
                          out=(out_cost[lo:hi], log_u[lo:hi], log_v[lo:hi], residuals[lo:hi]))
            checks.append(r)
            iters = max(iters, r.iterations_run)
            free[k % nbuf].record(st)
            if k + nbuf < chunks:
                upload(k + nbuf)
        for s_ in streams[1:]:   # the outputs are complete on the caller's stream
            done = torch.cuda.Event()
            done.record(s_)
            compute.wait_event(done)
    for r in checks:
        r.check()
    return SolveResult(out_cost, log_u, log_v, float(lam), iters, residuals, -1.0,
                       _lib.load().sinkhorn_last_path_v1().decode())


def _solve_f64(mu, nu, cost, lam, max_iters, tolerance, check_interval, validate) -> SolveResult:
    """The float64 parity mode: sinkhorn_forward_f64_device_v1 (sweep_f64.cuh)."""
    mu, nu = torch.as_tensor(mu), torch.as_tensor(nu)
    if not isinstance(cost, GridCost):
        cost = torch.as_tensor(cost)
    B, d1, d2 = _check_shapes(mu, nu, cost)
    dev = mu.device if mu.is_cuda else torch.device("cuda", torch.cuda.current_device())
    f64 = dict(device=dev, dtype=torch.float64)
    mu, nu = mu.to(**f64).contiguous(), nu.to(**f64).contiguous()
    if not isinstance(cost, GridCost):
        cost = cost.to(**f64).contiguous()
    lib = _lib.load()
    pr = _problem(B, d1, d2, cost)
    op = _lib.Options()
    op.lam, op.max_iters, op.check_interval, op.tolerance = float(lam), int(max_iters), \
        int(check_interval), float(tolerance)
    op.flags = 0 if validate else _lib.FLAG_SKIP_VALIDATION
    out_cost = torch.empty(B, **f64)
    log_u = torch.empty(B, d1, **f64)
    log_v = torch.empty(B, d2, **f64)
    residuals = torch.empty(B, **f64)
    iters = ctypes.c_int32(0)
    with torch.cuda.device(dev):
        ws = _workspace(dev, lib.sinkhorn_workspace_bytes_f64_v1(ctypes.byref(pr)))
        st = lib.sinkhorn_forward_f64_device_v1(
            ctypes.byref(pr), ctypes.byref(op), _ptr(mu), _ptr(nu),
            None if isinstance(cost, GridCost) else _ptr(cost), _ptr(out_cost), _ptr(log_u),
            _ptr(log_v), ctypes.byref(iters), _ptr(residuals), _ptr(ws), ws.numel(),
            _stream_handle(dev))
    raise_for_status(st, "sinkhorn_forward_f64_device_v1")
    return SolveResult(out_cost, log_u, log_v, float(lam), int(iters.value), residuals, -1.0,
                       lib.sinkhorn_last_path_v1().decode())


def potentials_backward(log_u: torch.Tensor, log_v: torch.Tensor, lam: float,
                        upstream: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """batch_backward (batch.py:352-375): up[b] * lam * (x - mean_i x).
    float64 potentials (the fp64 mode) are differentiated in float64."""
    dev = log_u.device
    if log_u.dtype == torch.float64:
        return _potentials_backward_f64(log_u, log_v, lam, upstream)
    log_u = _as_f32_cuda(log_u, dev)
    log_v = _as_f32_cuda(log_v, dev)
    up = _as_f32_cuda(upstream, dev).reshape(-1)
    B, d1 = log_u.shape
    d2 = log_v.shape[1]
    if log_v.shape[0] != B or up.numel() != B:
        raise ShapeMismatch(f"upstream must have shape ({B},), got {tuple(upstream.shape)}")
    g_mu = torch.empty_like(log_u)
    g_nu = torch.empty_like(log_v)
    if B == 0:
        return g_mu, g_nu
    lib = _lib.load()
    ws = torch.empty(64, device=dev, dtype=torch.uint8)
    lane = ctypes.c_int32(-1)
    with torch.cuda.device(dev):
        st = lib.sinkhorn_backward_device_v1(B, d1, d2, float(lam), _ptr(log_u), _ptr(log_v),
                                             _ptr(up), _ptr(g_mu), _ptr(g_nu),
                                             ctypes.byref(lane), _ptr(ws), ws.numel(),
                                             _stream_handle(dev))
    raise_for_status(st, "sinkhorn_backward_device_v1", lane=lane.value)
    return g_mu, g_nu


def _potentials_backward_f64(log_u, log_v, lam, upstream):
    dev = log_u.device
    f64 = dict(device=dev, dtype=torch.float64)
    log_u, log_v = log_u.to(**f64).contiguous(), log_v.to(**f64).contiguous()
    up = torch.as_tensor(upstream).to(**f64).reshape(-1).contiguous()
    B, d1 = log_u.shape
    d2 = log_v.shape[1]
    if log_v.shape[0] != B or up.numel() != B:
        raise ShapeMismatch(f"upstream must have shape ({B},), got {tuple(up.shape)}")
    g_mu, g_nu = torch.empty_like(log_u), torch.empty_like(log_v)
    if B == 0:
        return g_mu, g_nu
    lib = _lib.load()
    ws = torch.empty(64, device=dev, dtype=torch.uint8)
    lane = ctypes.c_int32(-1)
    with torch.cuda.device(dev):
        st = lib.sinkhorn_backward_f64_device_v1(B, d1, d2, float(lam), _ptr(log_u), _ptr(log_v),
                                                 _ptr(up), _ptr(g_mu), _ptr(g_nu),
                                                 ctypes.byref(lane), _ptr(ws), ws.numel(),
                                                 _stream_handle(dev))
    raise_for_status(st, "sinkhorn_backward_f64_device_v1", lane=lane.value)
    return g_mu, g_nu


def plan_gradient(log_u: torch.Tensor, log_v: torch.Tensor, cost: torch.Tensor, lam: float,
                  upstream: torch.Tensor) -> torch.Tensor:
    """dC = sum_b up_b P_b (shared) or up_b P_b (per-sample); P from core.py:363-368."""
    dev = log_u.device
    cost = _as_f32_cuda(cost, dev)
    up = _as_f32_cuda(upstream, dev).reshape(-1)
    B, d1 = log_u.shape
    d2 = log_v.shape[1]
    pr = _problem(B, d1, d2, cost)
    out = torch.empty_like(cost)
    lib = _lib.load()
    with torch.cuda.device(dev):
        # shared costs: the tensor-core contraction over the lanes (workspace variant)
        ws = _workspace(dev, lib.sinkhorn_plan_grad_workspace_bytes_v1(ctypes.byref(pr)))
        st = lib.sinkhorn_plan_grad_ws_device_v1(ctypes.byref(pr), float(lam),
                                                 _ptr(log_u.float().contiguous()),
                                                 _ptr(log_v.float().contiguous()), _ptr(cost),
                                                 _ptr(up), _ptr(out), _ptr(ws), ws.numel(),
                                                 _stream_handle(dev))
    raise_for_status(st, "sinkhorn_plan_grad_ws_device_v1")
    return out


class SinkhornLossFunction(torch.autograd.Function):
    """Custom node: forward = C-ABI forward, backward = C-ABI backward (loss.ts:59-131)."""

    @staticmethod
    def forward(ctx, mu, nu, cost, lam, max_iters, tolerance, check_interval):
        grid = cost if isinstance(cost, (GridCost, PointCloudCost)) else None
        res = solve(mu.detach(), nu.detach(), grid if grid is not None else cost.detach(), lam,
                    max_iters, tolerance, check_interval)
        # the complete backward state: final potentials only (loss.ts:104)
        if grid is None and ctx.needs_input_grad[2]:
            ctx.save_for_backward(res.log_u, res.log_v, cost.detach())
        else:
            ctx.save_for_backward(res.log_u, res.log_v)
        ctx.lam = float(lam)
        ctx.in_dtypes = (mu.dtype, nu.dtype, None if grid is not None else cost.dtype)
        ctx.iterations_run = res.iterations_run
        return res.cost_e0.to(mu.dtype)

    @staticmethod
    def backward(ctx, grad_out):
        saved = ctx.saved_tensors
        log_u, log_v = saved[0], saved[1]
        g_mu = g_nu = g_c = None
        if ctx.needs_input_grad[0] or ctx.needs_input_grad[1]:
            gm, gn = potentials_backward(log_u, log_v, ctx.lam, grad_out.detach())
            g_mu = gm.to(ctx.in_dtypes[0]) if ctx.needs_input_grad[0] else None
            g_nu = gn.to(ctx.in_dtypes[1]) if ctx.needs_input_grad[1] else None
        if len(saved) == 3 and ctx.needs_input_grad[2]:
            g_c = plan_gradient(log_u, log_v, saved[2], ctx.lam, grad_out.detach())
            g_c = g_c.to(ctx.in_dtypes[2])
        return g_mu, g_nu, g_c, None, None, None, None


def sinkhorn_loss(mu, nu, cost, lam: float, max_iters: int = 1000, tolerance: float = 0.0,
                  check_interval: int = 10) -> torch.Tensor:
    """Per-lane E0 transport loss, shape (B,) (loss.ts:59-131).

    Defaults follow the reference node: max_iters 1000, tolerance 0
    (loss.ts:76-77).  1-D histograms are treated as a batch of one
    (loss.ts:41-49).  Gradients reach whichever of mu / nu (/ cost) require them.
    """
    if mu.dim() == 1:
        mu = mu.unsqueeze(0)
    if nu.dim() == 1:
        nu = nu.unsqueeze(0)
    return SinkhornLossFunction.apply(mu, nu, cost, lam, max_iters, tolerance, check_interval)
