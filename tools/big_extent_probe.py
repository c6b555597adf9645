"""Extents whose cell counts pass 2^31 (32-bit index overflow guard): a shared
d = 46341 cost (gemm vs tiled paths) and per-sample lanes of 33000^2 cells
(lane path) against single-lane solves.   python tools/big_extent_probe.py
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1907_01729_b200 as skb  # noqa: E402

dev = torch.device("cuda", 0)


def hist(B, d, g):
    m = torch.rand(B, d, generator=g, device=dev, dtype=torch.float64) + 0.5
    return (m / m.sum(1, keepdim=True)).float()


g = torch.Generator(device=dev)
g.manual_seed(0)
d = 46341
mu, nu = hist(2, d, g), hist(2, d, g)
i = torch.arange(d, device=dev, dtype=torch.float32) / (d - 1)
c = torch.empty(d, d, device=dev)
for a in range(0, d, 4096):
    c[a:a + 4096] = (i[a:a + 4096, None] - i[None, :]) ** 2
r1 = skb.solve(mu, nu, c, 0.05, 3, 0.0, tiled_only=True, gemm=True)
r2 = skb.solve(mu, nu, c, 0.05, 3, 0.0, tiled_only=True, fused=False, gemm=False)
rel = float(((r1.cost_e0.double() - r2.cost_e0.double()).abs() / r2.cost_e0.double()).max())
print("shared d=46341", r1.path, r2.path, "rel", rel, "OK" if rel < 1e-5 else "MISMATCH")
del c, r1, r2
torch.cuda.empty_cache()
d = 33000
mu, nu = hist(2, d, g), hist(2, d, g)
c = torch.rand(2, d, d, generator=g, device=dev)
r = skb.solve(mu, nu, c, 0.05, 3, 0.0)
one = skb.solve(mu[1:], nu[1:], c[1:], 0.05, 3, 0.0)
rel = abs(float(one.cost_e0[0]) - float(r.cost_e0[1])) / float(one.cost_e0[0])
print("per-sample 2 x 33000^2", r.path, "rel", rel, "OK" if rel < 1e-6 else "MISMATCH")
