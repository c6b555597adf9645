"""Fused vs tiled on a golden case, per iteration count (diagnostic).

    SKB_NO_RERUN=1 python tools/debug_fused.py [golden-name]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402

import paper_1907_01729_b200 as skb  # noqa: E402
from paper_1907_01729_b200 import _lib  # noqa: E402
from conftest import golden_cost, load_golden  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config2_subset"
g = load_golden(name)
dev = torch.device("cuda", 0)
c = torch.tensor(golden_cost(g), dtype=torch.float32, device=dev)
mu, nu = torch.tensor(g["mu"], device=dev), torch.tensor(g["nu"], device=dev)
lib = _lib.load()
for it in [1, 2, 3, 5, 10, 30]:
    r0 = lib.sinkhorn_exact_reruns_v1()
    f = skb.solve(mu, nu, c, float(g["lam"]), it, 0.0, 10, tiled_only=True)
    r1 = lib.sinkhorn_exact_reruns_v1()
    t = skb.solve(mu, nu, c, float(g["lam"]), it, 0.0, 10, tiled_only=True, fused=False)
    fin = torch.isfinite(t.log_v)
    dv = (f.log_v[fin] - t.log_v[fin]).abs().max().item()
    du = (f.log_u[torch.isfinite(t.log_u)] - t.log_u[torch.isfinite(t.log_u)]).abs().max().item()
    de = ((f.cost_e0 - t.cost_e0).abs() / t.cost_e0).max().item()
    print(f"iters {it} path {f.path} reruns {r1 - r0} dlog_v {dv:.3e} dlog_u {du:.3e} dE0 {de:.3e} "
          f"nan_v {int(torch.isnan(f.log_v).sum())} nan_u {int(torch.isnan(f.log_u).sum())}")
