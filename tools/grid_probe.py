"""Grid costs of many aspect ratios and sizes on the separable / dense paths:
each against the materialised stored cost (tiled path).   python tools/grid_probe.py
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1907_01729_b200 as skb  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
for nx, ny in [(1, 1), (1, 50), (50, 1), (3, 300), (300, 3), (100, 100), (128, 128), (150, 140),
               (200, 200), (256, 64), (33, 257), (160, 170), (300, 250), (400, 33)]:
    d = nx * ny
    B = 4
    m = torch.rand(B, d, generator=g, device=dev, dtype=torch.float64) + 0.5
    mu = (m / m.sum(1, keepdim=True)).float()
    nu = mu.flip(0).contiguous()
    gc = skb.GridCost(nx, ny)
    try:
        r = skb.solve(mu, nu, gc, 0.01, 10, 0.0, time_loop=True)
        dn = skb.solve(mu, nu, gc, 0.01, 10, 0.0, time_loop=True, dense_grid=True)
        cm = gc.materialize(device=dev).float()
        ref = skb.solve(mu, nu, cm, 0.01, 10, 0.0, tiled_only=True, fused=False, gemm=False)
        diff = (r.cost_e0.double() - ref.cost_e0.double()).abs()
        rel = float((diff / ref.cost_e0.double().clamp_min(1e-300)).max())
        print(nx, ny, r.path, f"rel {rel:.2e}", "OK" if rel < 1e-5 else "MISMATCH",
              f"loop {r.loop_ms:.2f} ms (dense {dn.loop_ms:.2f})", flush=True)
        del cm
    except Exception as e:
        print(nx, ny, "ERROR", repr(e)[:160], flush=True)
