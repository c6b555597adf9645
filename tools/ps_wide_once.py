"""One per-sample solve with 4096-column rows (the two-warps-per-lane fused
pass), for ncu captures.   python tools/ps_wide_once.py [d] [B]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1907_01729_b200 as skb  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
m = torch.rand(B, d, generator=g, device=dev, dtype=torch.float64) + 0.5
mu = (m / m.sum(1, keepdim=True)).float()
nu = mu.flip(0).contiguous()
c = torch.rand(B, d, d, generator=g, device=dev)
r = skb.solve(mu, nu, c, 0.05, 6, 0.0)
torch.cuda.synchronize()
print(r.path, float(r.cost_e0[0]))
