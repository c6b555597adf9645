"""Batches above the grid.y limit (65535 lanes) on every path: the batch solve
equals single-lane solves at both ends.   python tools/big_batch_probe.py
"""
import sys, torch
sys.path.insert(0, ".")
import paper_1907_01729_b200 as skb
dev = torch.device("cuda", 0)
for B, d, kind, kw in [(70000, 16, "shared", {}), (70000, 16, "shared", {"tiled_only": True}),
                       (70000, 16, "shared", {"tiled_only": True, "fused": False, "gemm": False}),
                       (70000, 32, "shared", {"tiled_only": True, "gemm": True}),
                       (70000, 16, "per_sample", {}), (70000, 16, "per_sample", {"fused": False}),
                       (70000, 16, "grid", {}), (70000, 16, "shared", {"fp64": True}),
                       (70000, 16, "per_sample", {"fp64": True})]:
    g = torch.Generator(device=dev); g.manual_seed(0)
    m = torch.rand(B, d, generator=g, device=dev, dtype=torch.float64) + 0.5
    mu = (m / m.sum(1, keepdim=True)).float()
    nu = mu.flip(0).contiguous()
    if kind == "shared":
        c = torch.rand(d, d, generator=g, device=dev)
    elif kind == "per_sample":
        c = torch.rand(B, d, d, generator=g, device=dev)
    else:
        c = skb.GridCost(4, 4)
    try:
        r = skb.solve(mu, nu, c, 0.1, 20, 0.0, **kw)
        # compare lanes 0 and B-1 with single-lane solves
        ok = True
        for b in (0, B - 1):
            cb = c[b:b+1] if kind == "per_sample" else c
            one = skb.solve(mu[b:b+1], nu[b:b+1], cb, 0.1, 20, 0.0, **kw)
            ok &= abs(float(one.cost_e0[0]) - float(r.cost_e0[b])) <= 1e-5 * abs(float(one.cost_e0[0]))
        print(B, d, kind, kw, r.path, "OK" if ok else "MISMATCH")
    except Exception as e:
        print(B, d, kind, kw, "ERROR", repr(e)[:200])
