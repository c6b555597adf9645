"""Few-lane problems: which path is fastest per loop (auto vs forced).
    python tools/small_batch_bench.py
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1907_01729_b200 as skb  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
for B, d, kind in [(1, 784, "shared"), (4, 784, "shared"), (16, 784, "shared"), (1, 2048, "shared"),
                   (4, 4096, "shared"), (1, 1024, "per_sample"), (8, 1024, "per_sample"),
                   (2, 4096, "grid")]:
    m = torch.rand(B, d, generator=g, device=dev, dtype=torch.float64) + 0.5
    mu = (m / m.sum(1, keepdim=True)).float()
    nu = mu.flip(0).contiguous()
    if kind == "shared":
        i = torch.arange(d, device=dev, dtype=torch.float32) / (d - 1)
        c = (i[:, None] - i[None, :]) ** 2
        opts = (("auto", {}), ("fused", {"tiled_only": True}),
                ("gemm", {"tiled_only": True, "gemm": True}),
                ("tiled", {"tiled_only": True, "fused": False, "gemm": False}))
    elif kind == "per_sample":
        c = torch.rand(B, d, d, generator=g, device=dev)
        opts = (("auto", {}), ("lane", {"fused": False}))
    else:
        c = skb.GridCost(64, 64)
        opts = (("auto", {}), ("dense", {"dense_grid": True}))
    row = [f"{kind} B={B} d={d}:"]
    for name, kw in opts:
        for _ in range(3):
            r = skb.solve(mu, nu, c, 0.05, 100, 0.0, time_loop=True, **kw)
        row.append(f"{name}({r.path}) {r.loop_ms:.2f}")
    print(" | ".join(row), flush=True)
