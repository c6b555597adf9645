"""Feature x shape probe: point-cloud costs (odd D, d1 != d2, B > 64), warm
start, lockstep tolerance, asynchronous solves, dC and the fp64 mode, each on
odd shapes, checked against an independent route (materialised cost, cold
start, synchronous solve, direct plan sum, fp32 path).
    python tools/feature_probe.py
"""
import sys
import traceback

import torch

sys.path.insert(0, ".")
import paper_1907_01729_b200 as skb  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
fails = 0


def hist(B, d):
    m = torch.rand(B, d, generator=g, device=dev, dtype=torch.float64) + 0.5
    return (m / m.sum(1, keepdim=True)).float()


def rel(a, b):
    a, b = a.double(), b.double()
    return float(((a - b).abs() / b.abs().clamp_min(1e-300)).max())


def report(name, ok, info=""):
    global fails
    fails += 0 if ok else 1
    print(("OK   " if ok else "FAIL ") + name, info, flush=True)


def run(name, fn):
    try:
        fn()
    except Exception:
        report(name, False, traceback.format_exc().splitlines()[-1][:200])


# point clouds
for (B, d1, d2, D) in [(3, 50, 70, 1), (2, 129, 33, 3), (70, 64, 64, 17), (4, 300, 1100, 65),
                       (2, 1500, 700, 200), (1, 5, 5, 2)]:
    def f(B=B, d1=d1, d2=d2, D=D):
        x = torch.rand(d1, D, generator=g, device=dev)
        y = torch.rand(d2, D, generator=g, device=dev)
        pc = skb.PointCloudCost(x, y)
        mu, nu = hist(B, d1), hist(B, d2)
        r = skb.solve(mu, nu, pc, 0.1, 20, 0.0)
        ref = skb.solve(mu, nu, pc.materialize(device=dev).float(), 0.1, 20, 0.0)
        e = rel(r.cost_e0, ref.cost_e0)
        report(f"points B={B} {d1}x{d2} D={D} path={r.path}", e < 2e-5, f"rel {e:.1e}")
    run(f"points {B} {d1} {d2} {D}", f)

# warm start + lockstep tolerance + async + fp64 per path on odd shapes
paths = {"auto": {}, "tiled": {"tiled_only": True, "fused": False, "gemm": False},
         "fused": {"tiled_only": True}, "gemm": {"tiled_only": True, "gemm": True}}
for (B, d1, d2) in [(5, 37, 53), (3, 300, 129), (66, 70, 90), (2, 1100, 1030)]:
    mu, nu = hist(B, d1), hist(B, d2)
    c = torch.rand(d1, d2, generator=g, device=dev)
    for pname, kw in paths.items():
        def f(kw=kw, pname=pname, mu=mu, nu=nu, c=c, B=B, d1=d1, d2=d2):
            full = skb.solve(mu, nu, c, 0.1, 40, 0.0, **kw)
            half = skb.solve(mu, nu, c, 0.1, 20, 0.0, **kw)
            warm = skb.solve(mu, nu, c, 0.1, 20, 0.0, init_log_u=half.log_u, **kw)
            e = rel(warm.cost_e0, full.cost_e0)
            report(f"warm {pname} {B}x{d1}x{d2}", e < 2e-5, f"rel {e:.1e}")
            a = skb.solve(mu, nu, c, 0.1, 40, 0.0, asynchronous=True, **kw).check()
            e = rel(a.cost_e0, full.cost_e0)
            report(f"async {pname} {B}x{d1}x{d2}", e < 1e-6, f"rel {e:.1e}")
            t = skb.solve(mu, nu, c, 0.1, 2000, 1e-5, **kw)
            t64 = skb.solve(mu, nu, c, 0.1, 2000, 1e-5, fp64=True)
            report(f"tol {pname} {B}x{d1}x{d2}", abs(t.iterations_run - t64.iterations_run) <= 10
                   and rel(t.cost_e0, t64.cost_e0) < 2e-5,
                   f"iters {t.iterations_run} vs fp64 {t64.iterations_run}")
        run(f"{pname} {B} {d1} {d2}", f)
    def fdc(mu=mu, nu=nu, c=c, B=B, d1=d1, d2=d2):
        r = skb.solve(mu, nu, c, 0.1, 30, 0.0)
        up = torch.randn(B, generator=g, device=dev)
        dc = skb.plan_gradient(r.log_u, r.log_v, c, 0.1, up)
        P = torch.exp(r.log_u.double()[:, :, None] + r.log_v.double()[:, None, :]
                      - c.double()[None] / 0.1)
        want = (up.double()[:, None, None] * P).sum(0)
        e = float((dc.double() - want).abs().max() / want.abs().max())
        report(f"dC shared {B}x{d1}x{d2}", e < 1e-5, f"rel-to-max {e:.1e}")
    run(f"dC {B} {d1} {d2}", fdc)
print("FAILURES", fails)
