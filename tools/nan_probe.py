"""What each solver path returns for the reference's NaNProduced instance
(c = 1e30 everywhere, lambda = 1e-300: A = -c/lambda = -inf)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1907_01729_b200 as skb  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(6)
B, d = 3, 64
m = torch.rand(B, d, generator=g, device=dev, dtype=torch.float64) + 0.5
mu = (m / m.sum(1, keepdim=True)).float()
m = torch.rand(B, d, generator=g, device=dev, dtype=torch.float64) + 0.5
nu = (m / m.sum(1, keepdim=True)).float()
c = torch.full((d, d), 1.0e30, device=dev)
for name, kw in (("small", {}), ("fused", {"tiled_only": True}),
                 ("tiled", {"tiled_only": True, "fused": False, "gemm": False}),
                 ("gemm", {"tiled_only": True, "gemm": True})):
    try:
        r = skb.solve(mu, nu, c, 1e-300, 20, 0.0, **kw)
        print(name, "NO ERROR", r.path, r.cost_e0.tolist(), r.log_u[0, :3].tolist(),
              r.log_v[0, :3].tolist())
    except Exception as e:
        print(name, type(e).__name__, str(e)[:120])
