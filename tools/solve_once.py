"""Run a few forward solves of one bench config (for ncu captures; no timing).

    python tools/solve_once.py --config 3 --reps 2 [--iters 10] [--dense-grid] [--tiled-only]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1907_01729_b200 as skb  # noqa: E402
from bench import CONFIGS, make_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--iters", type=int, default=None)
ap.add_argument("--dense-grid", action="store_true")
ap.add_argument("--tiled-only", action="store_true")
ap.add_argument("--mufu-only", action="store_true")
ap.add_argument("--no-fused", action="store_true")
ap.add_argument("--gemm", choices=["auto", "on", "off"], default="auto")
ap.add_argument("--B", type=int, default=None, help="override the config's batch")
ap.add_argument("--d", type=int, default=None, help="override the config's support size")
a = ap.parse_args()
cfg = dict(CONFIGS[a.config])
if a.B:
    cfg["B"] = a.B
if a.d:
    cfg["d"] = a.d
dev = torch.device("cuda", 0)
mu, nu, cost = make_inputs(cfg, dev, 1)
import time  # noqa: E402

up = torch.ones(cfg["B"], device=dev)
for _ in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = skb.solve(mu, nu, cost, cfg["lam"], a.iters or cfg["iters"], 0.0, 10,
                  dense_grid=a.dense_grid, tiled_only=a.tiled_only, time_loop=True,
                  mufu_only=a.mufu_only, fused=not a.no_fused,
                  gemm={"auto": None, "on": True, "off": False}[a.gemm])
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    skb.potentials_backward(r.log_u, r.log_v, cfg["lam"], up)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cells = cfg["B"] * cfg["d"] ** 2 * 2 * (a.iters or cfg["iters"])
    print(f"B {cfg['B']} cells/s {cells / (r.loop_ms * 1e-3):.3e} config {a.config} path {r.path} loop_ms {r.loop_ms:.3f} solve_ms "
          f"{1e3 * (t1 - t0):.3f} backward_ms {1e3 * (t2 - t1):.3f} E0[0] {float(r.cost_e0[0]):.6g}")
