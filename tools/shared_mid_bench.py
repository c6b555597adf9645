"""Shared costs between the fused block pass (d <= 1024) and config 5: the
tcgen05 GEMM iteration against the MUFU tiled sweeps.  python tools/shared_mid_bench.py
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1907_01729_b200 as skb  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
for B, d in [(256, 1024), (256, 1100), (256, 1536), (256, 2048), (64, 4096), (256, 4096),
             (64, 8192)]:
    m = torch.rand(B, d, generator=g, device=dev, dtype=torch.float64) + 0.5
    mu = (m / m.sum(1, keepdim=True)).float()
    nu = mu.flip(0).contiguous()
    i = torch.arange(d, device=dev, dtype=torch.float32) / (d - 1)
    c = (i[:, None] - i[None, :]) ** 2
    row = [f"B={B} d={d}:"]
    for name, kw in (("auto", {}), ("gemm", {"tiled_only": True, "gemm": True}),
                     ("tiled", {"tiled_only": True, "fused": False, "gemm": False})):
        if name != "auto" and d <= 1024 and name == "gemm":
            pass
        r = skb.solve(mu, nu, c, 0.05, 50, 0.0, time_loop=True, **kw)
        r = skb.solve(mu, nu, c, 0.05, 50, 0.0, time_loop=True, **kw)
        row.append(f"{name}({r.path}) {r.loop_ms:.2f} ms")
    print(" | ".join(row), flush=True)
