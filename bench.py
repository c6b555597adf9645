"""Benchmark: B*d1*d2*iters/s of the log-domain Sinkhorn forward + analytic backward.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5] [--impl ours|reference]

Default workload (N=1): BASELINE.json configs[3] ("config 4") -- the config the
metric is quoted on at 1/2/4/8 B200 that fits one GPU: per-sample U[0,1) cost
matrices d1=d2=1024, B=1024 lanes per GPU (4.3 GB of costs streamed from HBM
every iteration), lambda=0.05, 100 iterations, tolerance 0 (like the
reference's own bench, cli.py:293-297), forward + analytic backward.
Synthetic inputs generated on the device.  A "step" is one forward (100
iterations + the fused residual/E0 tail) plus the backward over the batch.
`--gpus N` runs N ranks (it launches torchrun itself when not already under
it): the batch is sharded (weak scaling, B lanes per GPU) with one final NCCL
all-gather of the per-lane losses per step; config 5 is row-sharded.

Prints ONE JSON line (rank 0).  `--impl reference` times the reference
implementation itself (the `sinkloss` package installed in baseline/_ref,
kind "reference") on the host cores instead; the CPU oracle port (oracle/,
kind "port") stands in only when baseline/_ref is absent.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "B·d1·d2·iters/sec, log-Sinkhorn fwd+bwd"
UNIT = "cell*iter/s"
MUFU_PER_SM_CLK = 16     # ex2 results per SM per clock (sm_100 SFU)

CONFIGS = {
    1: dict(workload="config1: 1-D histograms d=100, B=32, |i-j|^2/99^2 shared cost, lambda=0.1",
            B=32, d=100, cost="index", lam=0.1, iters=100),
    2: dict(workload="config2: 28x28 grid histograms d=784, B=256 per GPU, shared stored "
                     "squared-Euclidean cost, lambda=0.05",
            B=256, d=784, cost="grid_stored", nx=28, lam=0.05, iters=100),
    3: dict(workload="config3: 64x64 grid histograms d=4096, B=512 per GPU, on-the-fly "
                     "squared-Euclidean cost, lambda=1e-3",
            B=512, d=4096, cost="grid_fly", nx=64, lam=1e-3, iters=100),
    4: dict(workload="config4: per-sample U[0,1) costs d1=d2=1024, B=1024 per GPU "
                     "(streamed from HBM), lambda=0.05",
            B=1024, d=1024, cost="per_sample", lam=0.05, iters=100),
    5: dict(workload="config5: d=65536 shared stored |i-j|^2/(d-1)^2 cost, B=64, lambda=0.05",
            B=64, d=65536, cost="index", lam=0.05, iters=100),
}


def load_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md "clocks" line)

class ClockSampler:
    """Clock and throttle-reason sampling during the timed region.

    In-process NVML queries from a background thread (ctypes calls release the
    GIL): unlike an ``nvidia-smi -lms`` child, which re-enumerates the devices
    on every sample and can hold the driver lock for tens of milliseconds
    while the solver enqueues its launches.  Falls back to nvidia-smi when
    NVML is unavailable."""

    REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index: int, interval_ms: int = 500):
        self.gpu = gpu_index
        self.interval_ms = interval_ms
        self.window = None   # wall-clock (start, end) of the timed region
        self.rows = []       # (ts, sm_mhz, sm_max_mhz, {reason: active})
        self._stop = None
        self._thread = None
        self._proc = None
        self._path = None

    def mark(self, t0: float, t1: float) -> None:
        """The timed region; samples within one interval of it are reported.
        (Sampling starts before the warm-up steps.)"""
        self.window = (t0, t1)

    def _nvml_handle(self):
        import pynvml
        import torch

        pynvml.nvmlInit()
        try:
            prop = torch.cuda.get_device_properties(self.gpu)
            bus = f"{prop.pci_domain_id:08X}:{prop.pci_bus_id:02X}:{prop.pci_device_id:02X}.0"
            return pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(self.gpu)

    def _loop(self, h):
        import pynvml

        bits = (pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap)
        while not self._stop.is_set():
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                mask = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((time.time(), float(sm), float(smax),
                                  {n: bool(mask & b) for n, b in zip(self.REASONS, bits)}))
            except Exception:
                pass
            self._stop.wait(self.interval_ms * 1e-3)

    def __enter__(self):
        import threading

        try:
            h = self._nvml_handle()
            self._stop = threading.Event()
            self._thread = threading.Thread(target=self._loop, args=(h,), daemon=True)
            self._thread.start()
            return self
        except Exception:
            pass
        try:   # fallback: an nvidia-smi child process
            self._path = tempfile.mktemp(prefix="clocks_", suffix=".csv")
            self._fh = open(self._path, "w")
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits",
                 "-lms", str(self.interval_ms)], stdout=self._fh, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except (OSError, FileNotFoundError):
            self._proc = None
        return self

    def __exit__(self, *exc):
        if self._thread is not None:
            self._stop.set()
            self._thread.join(timeout=5)
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._proc.kill()
            self._fh.close()
            try:   # no timestamps from this fallback: every row counts
                with open(self._path) as f:
                    for line in f:
                        v = [x.strip() for x in line.split(",")]
                        if len(v) >= 6 and v[0].replace(".", "").isdigit():
                            self.rows.append((None, float(v[0]), float(v[1]),
                                              {n: v[2 + k] == "Active"
                                               for k, n in enumerate(self.REASONS)}))
            except OSError:
                pass

    def summary(self) -> dict:
        rows = self.rows
        if self.window is not None and rows:
            pad = self.interval_ms * 1e-3
            t0, t1 = self.window[0] - pad, self.window[1] + pad
            near = [r for r in rows if r[0] is None or t0 <= r[0] <= t1]
            rows = near or rows[-1:]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        smax = max(r[2] for r in rows)
        sm = [r[1] for r in rows]
        load = [x for x in sm if x > 0.5 * smax] or sm
        reasons = sorted({n for r in rows for n, on in r[3].items() if on})
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# synthetic inputs (on the device)

def make_inputs(cfg: dict, device, seed: int):
    import torch

    from paper_1907_01729_b200 import GridCost

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    B, d = cfg["B"], cfg["d"]

    def hist(n):
        m = torch.rand(n, d, generator=g, device=device, dtype=torch.float64) + 0.5
        return (m / m.sum(dim=1, keepdim=True)).float()

    mu, nu = hist(B), hist(B)
    kind = cfg["cost"]
    if kind == "index":
        i = torch.arange(d, device=device, dtype=torch.float64)
        cost = ((i[:, None] - i[None, :]).abs() / max(d - 1, 1)) ** 2
        cost = cost.float()
    elif kind == "grid_stored":
        cost = GridCost(cfg["nx"], cfg["nx"]).materialize(device=device).float()
    elif kind == "grid_fly":
        cost = GridCost(cfg["nx"], cfg["nx"])
    elif kind == "per_sample":
        cost = torch.rand(B, d, d, generator=g, device=device, dtype=torch.float32)
    elif kind == "none":
        cost = None
    else:
        raise ValueError(kind)
    return mu, nu, cost


def index_cost_rows(d: int, r0: int, rows: int, device):
    """Rows [r0, r0 + rows) of the |i - j|^2 / (d - 1)^2 cost, built in blocks."""
    import torch

    out = torch.empty(rows, d, device=device, dtype=torch.float32)
    j = torch.arange(d, device=device, dtype=torch.float64)
    for a in range(0, rows, 1024):
        i = torch.arange(r0 + a, r0 + min(a + 1024, rows), device=device, dtype=torch.float64)
        out[a:a + len(i)] = (((i[:, None] - j[None, :]).abs() / max(d - 1, 1)) ** 2).float()
    return out


def work_units(cfg: dict) -> float:
    return float(cfg["B"]) * cfg["d"] * cfg["d"] * cfg["iters"]


KERNEL_OF_PATH = {
    "fused": "fused_ps_kernel (per-sample: one fused row->column pass per iteration, C_b read "
             "once) / fgemm_pass_kernel (shared: two register-blocked fp32 GEMMs per 16-row block)",
    "gemm": "umma_gemm_kernel (tcgen05 3xTF32 contraction streaming K or K^T from HBM; two per "
            "iteration, S = K X and T = K^T a)",
    "tiled": "tiled_sweep_kernel (stream-K online-LSE half-sweep)",
    "small": "small_solve_kernel (whole solve in one launch, cost in shared memory)",
    "persistent": "persistent_solve_kernel (cooperative whole loop)",
    "lane": "lane_col_kernel / lane_row_kernel (per-sample sweep)",
    "separable": "sep_sweep_kernel (separable grid LSE: two nested 1-D LSE-GEMMs per sweep)",
    "row-sharded-gemm": "umma_gemm_kernel on this rank's kernel-matrix rows (whole step incl. "
                        "the NCCL all-reduce of the column sums)",
}


def roofline(cfg: dict, kernel_ms: float, peaks: dict, clocks: dict, traffic, path: str,
             share: float = 1.0) -> dict:
    """Roofline of the dominant kernel from its measured average launch time
    (CUDA events around each launch, SINKHORN_FLAG_TIME_KERNEL) and the
    ALGORITHMIC work one launch does (DESIGN.md section 4 states both):

    * per-sample fused pass: reads C_b once per iteration, 4 B per cell
      (bound hbm); the survey's 8 B per cell-iteration (two half-sweeps that
      each read C) is reported beside it;
    * GEMM iteration: one contraction streams the d1 x d2 kernel matrix once,
      4 B per matrix element (bound hbm); its 3xTF32 tensor work is reported
      beside it;
    * shared fused block pass: two fp32 GEMMs, 4 FLOP per cell (bound fp32
      FMA pipe);
    * tiled / separable / small: ex2 per cell (bound mufu).
    """
    B, d = float(cfg["B"]), float(cfg["d"])
    cells = B * d * d * share          # cells one launch covers (this GPU)
    t = kernel_ms * 1e-3
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    fmax = float(peaks.get("sm_max_mhz", 1965.0))
    sms = 148
    hbm_src = ("MEASURED_PEAKS.json hbm_gbs (measured copy)" if "hbm_gbs" in peaks
               else "fallback 6650 GB/s (B200_PROFILING.md)")
    base = {"traffic": traffic, "kernel": KERNEL_OF_PATH.get(path, path),
            "kernel_ms_per_launch": kernel_ms}
    if cfg["cost"] == "per_sample" and path == "fused":
        read = 4 * cells
        a = read / t / 1e9
        return {"bound": "hbm", "achieved": a, "peak": hbm, "unit": "GB/s", "frac": a / hbm, **base,
                "algorithmic_per_launch": f"{read:.4g} B (C_b read once per iteration: 4 B per cell)",
                "peak_source": hbm_src,
                "survey_8B_per_cell": {"achieved": 2 * a, "frac": 2 * a / hbm,
                                       "note": "SURVEY 8(d) counts two half-sweeps that each read "
                                               "C_b (8 B per cell-iteration); the fused pass reads "
                                               "it once"}}
    if path in ("gemm", "row-sharded-gemm"):
        mat = d * d * share                              # kernel-matrix elements per launch
        read = 4 * mat
        a = read / t / 1e9
        tf = 6 * B * mat / t / 1e12                      # 3 tf32 products x 2 FLOP
        tf_peak = float(peaks.get("bf16_tflops", 1606.6)) / 2
        return {"bound": "hbm", "achieved": a, "peak": hbm, "unit": "GB/s", "frac": a / hbm, **base,
                "algorithmic_per_launch": f"{read:.4g} B (the d1 x d2 kernel matrix, 4 B per "
                                          "element, streamed once per contraction)",
                "peak_source": hbm_src,
                "tensor_tf32": {"achieved_tflops": tf, "peak_tflops": tf_peak,
                                "frac": tf / tf_peak,
                                "note": "3xTF32: 3 MMA products x 2 FLOP per B-lane x element; "
                                        "peak = measured bf16 / 2 (tf32 runs at half the bf16 rate)"}}
    if path == "fused":
        flop = 4 * cells
        a = flop / t / 1e12
        peak = sms * 128 * 2 * fmax * 1e6 / 1e12
        return {"bound": "fp32", "achieved": a, "peak": peak, "unit": "TFLOP/s", "frac": a / peak,
                **base, "algorithmic_per_launch": f"{flop:.4g} FLOP (two GEMMs, 4 FLOP per cell "
                                                  "per iteration)",
                "peak_source": f"nominal 148 SM x 128 FFMA/clk x 2 x sm_max_mhz {fmax:.0f}",
                "ex2_equivalent": {"frac": 2 * cells / t / (sms * MUFU_PER_SM_CLK * fmax * 1e6),
                                   "note": "the direct log-domain method's 2 ex2 per "
                                           "cell-iteration (SURVEY 8(d)) vs the MUFU peak; the "
                                           "block pass evaluates none per cell"}}
    if path == "separable":
        ex2 = B * d * (2 * cfg["nx"])                    # nested 1-D LSEs per sweep
        what = f"{ex2:.4g} ex2 (B*d*(nx+ny), separable)"
    elif path == "small":
        ex2 = cells * 2 * cfg["iters"]                   # the whole solve in one launch
        what = f"{ex2:.4g} ex2 (whole solve: 2 per cell-iteration)"
    else:
        ex2 = cells
        what = f"{ex2:.4g} ex2 (1 per cell per half-sweep)"
    a = ex2 / t / 1e12
    peak = sms * MUFU_PER_SM_CLK * fmax * 1e6 / 1e12
    out = {"bound": "mufu", "achieved": a, "peak": peak, "unit": "Tex2/s", "frac": a / peak, **base,
           "algorithmic_per_launch": what,
           "peak_source": f"148 SM x {MUFU_PER_SM_CLK} ex2/clk x sm_max_mhz {fmax:.0f}"}
    if clocks.get("sm_mhz"):
        out["frac_at_measured_clock"] = a / (sms * MUFU_PER_SM_CLK * clocks["sm_mhz"] * 1e-6)
    return out


def load_traffic(cfg_id: int, path: str):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed ncu capture of this config and solver path (profiles/), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            data = json.load(f)
    except (OSError, ValueError):
        return None
    entry = data.get(f"config{cfg_id}", {})
    if entry.get("path") == path:
        return entry.get("dram_bytes_per_sweep_launch")
    return entry.get(f"{path}_path", {}).get("dram_bytes_per_sweep_launch")


# ---------------------------------------------------------------------------
# CPU baseline: the reference itself (baseline/_ref), bounded samples

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_package():
    """The reference's own `sinkloss` package installed in baseline/_ref
    (pip --target), or None when it is absent."""
    if not os.path.isfile(os.path.join(REF_DIR, "sinkloss", "batch.py")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import sinkloss  # noqa: F401

    return sinkloss


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _ref_hist(rng, d):
    """random_histogram (oracle.py:152-155): U(0.5, 1.5) normalised."""
    m = rng.uniform(0.5, 1.5, d)
    return m / m.sum()


def _ref_lane_job(args):
    """One per-sample lane through the reference's public API: batch_forward
    with B = 1 and the lane's own cost (the reference has no per-sample API,
    SPEC.md:323; lanes are independent at tolerance 0, test_batch.py:46-63),
    then batch_backward.  Returns the solve's seconds."""
    seed, lane, d, lam, iters = args
    reference_package()
    from sinkloss import batch, core

    rng = np.random.default_rng([seed, lane])
    mu, nu = _ref_hist(rng, d), _ref_hist(rng, d)
    c = rng.random((d, d), dtype=np.float32).astype(np.float64)
    cfg = core.SinkhornConfig(lam=lam, max_iters=iters, tolerance=0.0)
    hb = batch.validate_histogram_batch
    t0 = time.perf_counter()
    r = batch.batch_forward(hb(mu[None]), hb(nu[None]), core.CostMatrix(c), cfg, workers=1)
    batch.batch_backward(r, np.ones(1))
    return time.perf_counter() - t0


def _ref_shared_cost(cfg, d):
    from sinkloss import core, oracle

    if cfg["cost"] == "index":
        return oracle.index_grid_cost(d, power=2)
    n = int(math.isqrt(d))   # 2-D grids (configs 2, 3): coordinates (col, row)/(n-1)
    k = np.arange(n * n)
    x, y = (k % n) / max(n - 1, 1), (k // n) / max(n - 1, 1)
    return core.CostMatrix(cost=(x[:, None] - x[None, :]) ** 2 + (y[:, None] - y[None, :]) ** 2)


def reference_cpu_sample(cfg: dict, seed: int = 0, runs: int = 3, light: bool = False) -> dict:
    """Time the reference implementation (baseline/_ref sinkloss) on the host cores.

    Forward (batch_forward, workers = os.cpu_count()) + batch_backward at k1
    and k2 iterations, median of `runs` runs each (cli.py:299-306 with fewer
    repetitions); the per-iteration slope and the fixed tail (final residual
    + E0) extrapolate to the configured iteration count (lanes independent at
    tolerance 0, every iteration costs the same).  Per-sample costs (config 4)
    run one lane per process over a pool of os.cpu_count() processes.
    """
    sl = reference_package()
    if sl is None:
        return port_cpu_sample(cfg, seed)
    from sinkloss import batch, core

    threads = os.cpu_count() or 1
    B, d, lam, iters = cfg["B"], cfg["d"], cfg["lam"], cfg["iters"]
    k1, k2 = (2, 4) if light else (5, 10)
    if cfg["cost"] != "per_sample" and min(cfg["d"], 4096) >= 4096:
        k1, k2 = 1, 2   # ~4 s per iteration at d = 4096 on the reference's streaming loop
    if cfg["cost"] == "per_sample":
        from concurrent.futures import ProcessPoolExecutor

        lanes = threads
        with ProcessPoolExecutor(max_workers=threads) as ex:
            list(ex.map(_ref_lane_job, [(seed, b, d, lam, 1) for b in range(lanes)]))  # warm

            def run(k):
                ts = list(ex.map(_ref_lane_job, [(seed, b, d, lam, k) for b in range(lanes)]))
                return max(ts)     # the lanes run concurrently, one per process
            t1 = statistics.median(run(k1) for _ in range(runs))
            t2 = statistics.median(run(k2) for _ in range(runs))
        cells = float(lanes) * d * d
        sample = (f"reference sinkloss.batch_forward(B=1)+batch_backward, {lanes} per-sample lanes "
                  f"d={d} on {threads} processes, {k1} and {k2} iterations, median of {runs}")
    else:
        dd = min(d, 4096)
        Bs = B if dd == d and B * dd * dd <= 256 * 784 * 784 else min(B, 64)
        rng = np.random.default_rng(seed)
        hb = batch.validate_histogram_batch
        mu = hb(np.stack([_ref_hist(rng, dd) for _ in range(Bs)]))
        nu = hb(np.stack([_ref_hist(rng, dd) for _ in range(Bs)]))
        c = _ref_shared_cost(cfg, dd)
        if d <= 100:
            k1, k2 = iters // 2, iters

        def one(k):
            conf = core.SinkhornConfig(lam=lam, max_iters=k, tolerance=0.0)
            t0 = time.perf_counter()
            r = batch.batch_forward(mu, nu, c, conf, workers=threads)
            batch.batch_backward(r, np.ones(Bs))
            return time.perf_counter() - t0
        one(1)
        t1 = statistics.median(one(k1) for _ in range(runs))
        t2 = statistics.median(one(k2) for _ in range(runs))
        cells = float(Bs) * dd * dd
        sample = (f"reference sinkloss.batch_forward+batch_backward, workers={threads}, B={Bs} "
                  f"d={dd}, {k1} and {k2} iterations, median of {runs}"
                  + (f"; per-cell rate extrapolated to d={d} (the reference's fp64 copies of "
                     f"a d={d} cost exceed host RAM)" if dd != d else ""))
    per_iter = max((t2 - t1) / (k2 - k1), 1e-9)
    tail = max(t1 - k1 * per_iter, 0.0)
    t_full = tail + iters * per_iter
    rate = cells * iters / t_full
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": sample + f"; extrapolated to {iters} iterations (slope + fixed tail)",
            "cpu": cpu_model(), "seconds_per_iteration": per_iter, "tail_seconds": tail,
            "ms_per_step_full": t_full * 1e3 * (float(B) * d * d / cells)}


def port_cpu_sample(cfg: dict, seed: int = 0) -> dict:
    """Fallback when baseline/_ref is absent: the oracle port (oracle/, kind "port")."""
    from oracle import sinkhorn_oracle as orc

    rng = np.random.default_rng(seed)
    B, d, lam, iters = cfg["B"], cfg["d"], cfg["lam"], cfg["iters"]
    threads = os.cpu_count() or 1
    dd = min(d, 1024)
    mu = orc.random_histogram_batch(1, dd, rng)[0]
    nu = orc.random_histogram_batch(1, dd, rng)[0]
    c = (orc.per_sample_cost(1, 0, dd, dd).astype(np.float64) if cfg["cost"] == "per_sample"
         else orc.index_grid_cost(dd))

    def run(k):
        t0 = time.perf_counter()
        r = orc.dense_forward(mu, nu, c, lam, k)
        orc.batch_backward(r.log_u, r.log_v, lam, np.ones(1))
        return time.perf_counter() - t0
    t1, t2 = run(1), run(2)
    per_iter = max(t2 - t1, 1e-9)
    tail = max(t1 - per_iter, 0.0)
    t_full = tail + iters * per_iter
    return {"value": float(dd) * dd * iters / t_full, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"oracle port dense single lane d={dd}, 1 and 2 iterations (baseline/_ref absent)",
            "cpu": cpu_model(), "ms_per_step_full": t_full * 1e3 * B * (d / dd) ** 2}


# ---------------------------------------------------------------------------

def init_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def config_dict(cfg: dict, world: int, row: bool) -> dict:
    """The `config` object both arms print (same keys, same values)."""
    jobs = 1 if row else world
    out = {"workload": cfg["workload"], "B_per_gpu": cfg["B"], "global_batch": cfg["B"] * jobs,
           "d1": cfg["d"], "d2": cfg["d"], "iters": cfg["iters"], "lambda": cfg["lam"],
           "tolerance": 0.0,
           "parallelism": (f"row-sharded cost over {world} GPU(s), one NCCL all-reduce of the "
                           "column sums per iteration") if row else f"batch-sharded dp{world}",
           "l2": ("flushed between steps (256 MiB write outside the timed events); config-4 / "
                  "config-5 inputs (4.3 / 17.2 GB) also exceed L2")}
    return out


def run_reference(args, cfg, world, rank):
    """`--impl reference`: the reference's own CPU implementation on this
    host's cores, rank 0 only (the other ranks exit without work)."""
    if rank != 0:
        return
    heavy = cfg["cost"] != "per_sample" and cfg["d"] > 100
    for _ in range(max(0, min(args.warmup, 1))):
        reference_cpu_sample(cfg, seed=99, runs=1, light=True)
    vals, ms, r = [], [], None
    t0 = time.perf_counter()
    for s in range(args.steps):
        r = reference_cpu_sample(cfg, seed=s, runs=1, light=heavy)
        vals.append(r["value"])
        ms.append(r["ms_per_step_full"])
        if time.perf_counter() - t0 > args.reference_budget_s:   # bounded CPU work
            break
    value = statistics.median(vals)
    row = args.config == 5 and world > 1
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(ms), "higher_is_better": True,
        "scaling": "strong" if row else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": config_dict(cfg, world, row),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
                         "sample": r["sample"] + f"; one sample per step, median of {len(vals)} "
                                                 f"(of {args.steps} requested; CPU budget "
                                                 f"{args.reference_budget_s:.0f} s)",
                         "cpu": r["cpu"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def run_ours(args, cfg, world, rank, local):
    import torch
    import torch.distributed as dist

    import paper_1907_01729_b200 as skb
    from paper_1907_01729_b200 import _lib

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if args.sharding is None:
        args.sharding = "row" if (args.config == 5 and world > 1) else "batch"
    lib = _lib.load()
    peaks = load_peaks()
    B, d, lam, iters = cfg["B"], cfg["d"], cfg["lam"], cfg["iters"]
    row = args.sharding == "row"
    if row:
        # BASELINE config 5: the cost's rows are sharded over the ranks; every
        # column sweep merges (max, sum-exp) pairs across ranks
        if not dist.is_initialized():   # also for a 1-rank run outside torchrun
            if "RANK" not in os.environ:
                import socket

                with socket.socket() as sk:
                    sk.bind(("127.0.0.1", 0))
                    os.environ.setdefault("MASTER_PORT", str(sk.getsockname()[1]))
                os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("nccl", device_id=dev)
        from paper_1907_01729_b200 import distributed as D

        if d % world:
            raise SystemExit(f"row sharding needs d % world == 0 (d={d}, world={world})")
        mu, nu, _ = make_inputs(dict(cfg, cost="none"), dev, seed=1234)
        rows = d // world
        r0 = rank * rows
        cost = index_cost_rows(d, r0, rows, dev)
        mu_l = mu[:, r0:r0 + rows].contiguous()
        backend = None if args.row_backend == "gemm" else D.CudaShardBackend(cost)
    else:
        mu, nu, cost = make_inputs(cfg, dev, seed=1234 + rank)
    up = torch.ones(B, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, device=dev, dtype=torch.float32)
    gathered = torch.empty(B * world, device=dev) if (world > 1 and not row) else None

    def step():
        if row:
            if backend is None:   # the library's loop: one NCCL sum per column sweep
                res = D.row_sharded_solve_device(mu_l, nu, cost, lam, iters, 0.0, 10,
                                                 time_loop=True)
            else:
                res = D.row_sharded_solve(mu_l, nu, backend, lam, iters, 0.0, 10, d1_total=d)
                res.loop_ms, res.path = -1.0, "row-sharded"
            D.row_sharded_backward(res.log_u, res.log_v, lam, up, d1_total=d)
            return res
        res = skb.solve(mu, nu, cost, lam, iters, 0.0, 10, validate=True, time_loop=True)
        gm, gn = skb.potentials_backward(res.log_u, res.log_v, lam, up)
        if world > 1:   # the single final loss collective of a batch-sharded step
            dist.all_gather_into_tensor(gathered, res.cost_e0)
        return res

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    loop_ms = []
    with ClockSampler(local, args.clock_interval_ms) as clk:
        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        launches0 = lib.sinkhorn_launch_count_v1()
        reruns0 = lib.sinkhorn_exact_reruns_v1()
        torch.cuda.synchronize()
        t_wall0 = time.time()
        for s in range(args.steps):
            flush.zero_()                       # L2 flush between steps (outside the events)
            starts[s].record()
            res = step()
            ends[s].record()
            loop_ms.append(res.loop_ms)
            path = res.path
        torch.cuda.synchronize()
        clk.mark(t_wall0, time.time())
    launches = lib.sinkhorn_launch_count_v1() - launches0
    reruns = lib.sinkhorn_exact_reruns_v1() - reruns0
    # the dominant kernel's average launch time: one more solve (untimed by the
    # step clock) with CUDA events around each of its launches
    if row and backend is None:
        kr = D.row_sharded_solve_device(mu_l, nu, cost, lam, iters, 0.0, 10, time_kernel=True)
        kernel_ms = kr.kernel_ms / max(kr.kernel_launches, 1)
    elif row:
        kernel_ms = None
    else:
        kr = skb.solve(mu, nu, cost, lam, iters, 0.0, 10, validate=True, time_kernel=True)
        kernel_ms = kr.kernel_ms / max(kr.kernel_launches, 1)
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
    ms = sum(step_ms) / len(step_ms)
    step_stats = {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms)}
    if kernel_ms is None:   # row sharding: the step's share per contraction (2 per iteration)
        kernel_ms = statistics.median(step_ms) / (2 * iters)
    t = torch.tensor([ms, kernel_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, kernel_ms = float(t[0]), float(t[1])
    # batch sharding: every rank solves its own B lanes (weak scaling);
    # row sharding: the ranks share one B x d x d problem (strong scaling)
    jobs = 1 if row else world
    value = jobs * work_units(cfg) / (ms * 1e-3)

    # ---- end to end through the public / reference-facing API with host buffers ----
    if row:
        e2e = run_e2e_row(args, step, mu_l, nu, dev)
    else:
        e2e = run_e2e(args, cfg, mu, nu, cost, lam, iters, dev)
    if world > 1:
        te = torch.tensor([e2e["seconds_per_step"]], device=dev, dtype=torch.float64)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e["seconds_per_step"] = float(te[0])
    e2e_value = jobs * work_units(cfg) / e2e["seconds_per_step"]

    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if row else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": config_dict(cfg, world, row),
        "solver_path": path,
        "roofline": roofline(cfg, kernel_ms, peaks, clocks, load_traffic(args.config, path), path,
                             share=(1.0 / world) if row else 1.0),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": e2e["h2d"],
                "d2h_bytes_per_step": e2e["d2h"], "path": e2e["path"]},
        "gpu_launches": int(launches),
        "exact_reruns": int(reruns),
        "clocks": clocks,
        "step_ms_stats": step_stats,
        "loop_ms_median": statistics.median(loop_ms) if loop_ms and loop_ms[0] > 0 else None,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = reference_cpu_sample(cfg, runs=3 if cfg["cost"] == "per_sample" else 1,
                                  light=cfg["cost"] != "per_sample" and d > 100)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu")}
    if rank == 0:
        emit(line)
    if dist.is_initialized():
        dist.destroy_process_group()


def run_e2e_row(args, step_fn, mu_l, nu, dev):
    """Row-sharded e2e: this rank's histogram columns and nu from pinned host
    buffers into the same device tensors, the step, the losses back."""
    import torch

    h_mu, h_nu = mu_l.cpu().pin_memory(), nu.cpu().pin_memory()
    h_loss = torch.empty(nu.shape[0]).pin_memory()
    steps = max(1, min(args.steps, 3))

    def one():
        mu_l.copy_(h_mu, non_blocking=True)
        nu.copy_(h_nu, non_blocking=True)
        res = step_fn()
        h_loss.copy_(res.cost_e0, non_blocking=True)
        torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    dt = (time.perf_counter() - t0) / steps
    return {"seconds_per_step": dt, "h2d": 4 * (mu_l.numel() + nu.numel()),
            "d2h": 4 * nu.shape[0],
            "path": "row_sharded_solve()+row_sharded_backward() from pinned host tensors"}


def pinned_copy(t):
    """A page-locked host copy of device tensor t, allocated pinned directly
    (no pageable intermediate: config 5's cost is 17 GB); pageable if the host
    cannot lock that much."""
    import torch

    try:
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    except RuntimeError:
        return t.cpu()
    h.copy_(t)
    return h


def run_e2e(args, cfg, mu, nu, cost, lam, iters, dev):
    """Host buffers in, host results out, copies inside the timed region."""
    import ctypes

    import torch

    import paper_1907_01729_b200 as skb
    from paper_1907_01729_b200 import _lib

    B, d = cfg["B"], cfg["d"]
    steps = max(1, min(args.steps, 10))
    if cfg["cost"] in ("index", "grid_stored") and d <= 8192:
        # the reference-facing C ABI: sinkhorn_forward_v1 / sinkhorn_backward_v1 (ffi.ts:80-191)
        lib = _lib.load()

        def pinned(shape, src=None):   # numpy views of page-locked host memory
            t = torch.empty(shape, dtype=torch.float64).pin_memory()
            if src is not None:
                t.copy_(src.double().cpu())
            return t.numpy()
        h_mu, h_nu, h_c = pinned((B, d), mu), pinned((B, d), nu), pinned((d, d), cost)
        o_cost, o_lu, o_lv = pinned((B,)), pinned((B, d)), pinned((B, d))
        up, g_mu, g_nu = pinned((B,)), pinned((B, d)), pinned((B, d))
        up[:] = 1.0

        def view(a):
            v = _lib.View()
            v.data = a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
            v.ndim = a.ndim
            v.shape[0] = a.shape[0]
            v.shape[1] = a.shape[1] if a.ndim == 2 else 0
            v.length = a.size
            return v
        vs = [view(a) for a in (h_mu, h_nu, h_c, o_cost, o_lu, o_lv, up, g_mu, g_nu)]

        def one():
            st = lib.sinkhorn_forward_v1(ctypes.byref(vs[0]), ctypes.byref(vs[1]),
                                         ctypes.byref(vs[2]), lam, iters, 0.0,
                                         ctypes.byref(vs[3]), ctypes.byref(vs[4]),
                                         ctypes.byref(vs[5]))
            assert st == 0, (st, _lib.last_error())
            st = lib.sinkhorn_backward_v1(ctypes.byref(vs[4]), ctypes.byref(vs[5]), lam,
                                          ctypes.byref(vs[6]), ctypes.byref(vs[7]),
                                          ctypes.byref(vs[8]))
            assert st == 0, (st, _lib.last_error())
        h2d = 8 * (2 * B * d + d * d) + 8 * (2 * B * d + B)
        d2h = 8 * (B + 2 * B * d) + 8 * (2 * B * d)
        path = ("C ABI sinkhorn_forward_v1 + sinkhorn_backward_v1, host float64 views in "
                "pinned memory")
    else:
        h_mu = mu.cpu().pin_memory()
        h_nu = nu.cpu().pin_memory()
        grid = isinstance(cost, skb.GridCost)
        h_c = None if grid else pinned_copy(cost)
        h_loss = torch.empty(B).pin_memory()
        h_gm = torch.empty(B, d).pin_memory()
        h_gn = torch.empty(B, d).pin_memory()
        per_sample = (not grid) and cost.dim() == 3
        chunks = args.e2e_chunks if per_sample else 1

        def one():
            # solve_streamed: lane groups of histograms (+ per-sample costs) are
            # uploaded on a copy stream while the previous group solves
            res = skb.solve_streamed(h_mu, h_nu, cost if grid else h_c, lam, iters, 0.0,
                                     chunks=chunks, device=dev)
            gm, gn = skb.potentials_backward(res.log_u, res.log_v, lam, torch.ones(B, device=dev))
            h_loss.copy_(res.cost_e0, non_blocking=True)
            h_gm.copy_(gm, non_blocking=True)
            h_gn.copy_(gn, non_blocking=True)
            torch.cuda.synchronize()
        h2d = 4 * (2 * B * d + (0 if grid else cost.numel()))
        d2h = 4 * (B + 2 * B * d)
        path = (f"torch API solve_streamed(chunks={chunks})+potentials_backward() from pinned "
                "host tensors" + (" (uploads overlap the solve)" if chunks > 1 else ""))
    one()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    dt = (time.perf_counter() - t0) / steps
    return {"seconds_per_step": dt, "h2d": h2d, "d2h": d2h, "path": path}


_JSON_OUT = None   # the process's original stdout (see quiet_stdout)


def quiet_stdout() -> None:
    """stdout carries exactly one JSON line: from here on anything else that
    writes to file descriptor 1 -- NCCL's version banner, library prints --
    lands on stderr, and emit() writes to the saved original stdout."""
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(obj) -> None:
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(obj) + "\n")
    out.flush()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default per config: ~0.3-1 s of timed work, 3 for config 5)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--clock-interval-ms", type=int, default=100)
    ap.add_argument("--row-backend", choices=["gemm", "lse"], default="gemm",
                    help="row sharding: the library's GEMM loop (default) or the exact "
                         "log-domain half-sweep shards")
    ap.add_argument("--sharding", choices=["batch", "row"], default=None,
                    help="multi-GPU split (default: row for config 5 on N>1, else batch)")
    ap.add_argument("--probe-ranks", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--reference-budget-s", type=float, default=150.0,
                    help="--impl reference: stop sampling after this many seconds of CPU work")
    ap.add_argument("--e2e-chunks", type=int, default=16,
                    help="e2e leg, per-sample costs: lane groups whose upload overlaps the solve")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: relaunch under torchrun (the driver's own launch
        # sets WORLD_SIZE and lands in the branch below instead)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        raise SystemExit(subprocess.call(cmd))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}: "
                         "launch N ranks for --gpus N")
    quiet_stdout()   # a worker (or the single process): the launcher above keeps its stdout
    if args.steps is None:
        # enough steps that a rare host-side stall (seen on the boxes: one
        # step in ~100 takes 5-100 ms longer, with or without our sampler)
        # does not dominate the mean
        args.steps = {1: 50, 2: 30, 3: 30, 4: 10, 5: 3}[args.config]
    world, rank, local = init_dist()
    if args.probe_ranks:   # launcher check (tests/test_bench_cpu.py): gloo, no GPU work
        import torch
        import torch.distributed as dist

        dist.init_process_group("gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        if rank == 0:
            emit({"probe": "ranks", "world": world, "ranks_seen": int(t.item()),
                  "gpus_arg": args.gpus})
        dist.destroy_process_group()
        return
    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
    else:
        run_ours(args, cfg, world, rank, local)


if __name__ == "__main__":
    main()
