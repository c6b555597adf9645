import sys, torch
sys.path.insert(0, ".")
import paper_1907_01729_b200 as skb
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(0)
d = 16384
i = torch.arange(d, device=dev, dtype=torch.float32) / (d - 1)
c = (i[:, None] - i[None, :]) ** 2
for B in (64, 128, 256, 512):
    m = torch.rand(B, d, generator=g, device=dev, dtype=torch.float64) + 0.5
    mu = (m / m.sum(1, keepdim=True)).float(); nu = mu.flip(0).contiguous()
    for _ in range(3):
        r = skb.solve(mu, nu, c, 0.05, 20, 0.0, time_loop=True)
    print(B, r.path, f"{r.loop_ms/20:.3f} ms/iter", f"{2*4*d*d/(r.loop_ms/20*1e-3)/1e9:.0f} GB/s of K per iteration (2 reads)", flush=True)
