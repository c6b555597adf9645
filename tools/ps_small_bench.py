"""Per-sample costs with short rows: fused pass vs lane half-sweeps at equal
bytes (~1 GB of costs).   python tools/ps_small_bench.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1907_01729_b200 as skb  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
for d in (16, 32, 64, 128, 256, 512):
    B = (1 << 28) // (d * d)
    m = torch.rand(B, d, generator=g, device=dev, dtype=torch.float64) + 0.5
    mu = (m / m.sum(1, keepdim=True)).float()
    nu = mu.flip(0).contiguous()
    c = torch.rand(B, d, d, generator=g, device=dev)
    row = [f"B={B} d={d}:"]
    for name, kw in (("auto", {}), ("lane", {"fused": False})):
        for _ in range(3):
            r = skb.solve(mu, nu, c, 0.05, 50, 0.0, time_loop=True, **kw)
        gbs = 4.0 * B * d * d * 50 / (r.loop_ms * 1e-3) / 1e9
        row.append(f"{name}({r.path}) {r.loop_ms:.2f} ms = {gbs:.0f} GB/s of C per iteration")
    print(" | ".join(row), flush=True)
    del c
    torch.cuda.empty_cache()
