"""Per-sample costs with rows of 1024-2048 columns: the fused pass (one read of
C_b per iteration) against the two lane half-sweeps.  python tools/ps_wide_bench.py
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1907_01729_b200 as skb  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
for B, d in [(1024, 1024), (448, 1536), (256, 2048), (300, 1800), (1024, 1023), (256, 2047),
             (110, 3100), (64, 4096), (64, 4095), (180, 2500), (42, 5000), (16, 8192),
             (20, 7001), (8, 12000), (4, 16384)]:
    m = torch.rand(B, d, generator=g, device=dev, dtype=torch.float64) + 0.5
    mu = (m / m.sum(1, keepdim=True)).float()
    nu = mu.flip(0).contiguous()
    c = torch.rand(B, d, d, generator=g, device=dev)
    out = []
    for kw in ({}, {"fused": False}):
        for _ in range(3):   # eager, graph capture, replay (the capture call's loop
            # timing includes the host's capture)
            r = skb.solve(mu, nu, c, 0.05, 100, 0.0, time_loop=True, **kw)
        out.append((r.path, r.loop_ms, r.cost_e0))
    gbs = [4.0 * B * d * d * 100 / (ms * 1e-3) / 1e9 for _, ms, _ in out]
    rel = float(((out[0][2].double() - out[1][2].double()).abs() / out[1][2].double()).max())
    print(f"B={B} d={d}: {out[0][0]} {out[0][1]:.1f} ms ({gbs[0]:.0f} GB/s of C per iteration) | "
          f"{out[1][0]} {out[1][1]:.1f} ms | rel {rel:.1e}", flush=True)
    del c
    torch.cuda.empty_cache()
