"""Host-side overhead probe: wall time of solve()+backward vs the device loop time."""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1907_01729_b200 as skb
from paper_1907_01729_b200 import _lib
from bench import CONFIGS, make_inputs

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
if os.environ.get("NO_GC"):
    gc.disable()
dev = torch.device("cuda", 0)
mu, nu, cost = make_inputs(cfg, dev, 1)
up = torch.ones(cfg["B"], device=dev)
lib = _lib.load()
for _ in range(3):
    r = skb.solve(mu, nu, cost, cfg["lam"], cfg["iters"], 0.0, time_loop=True)
torch.cuda.synchronize()
for _ in range(n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0 = lib.sinkhorn_exact_reruns_v1()
    t0 = time.perf_counter()
    e0.record()
    r = skb.solve(mu, nu, cost, cfg["lam"], cfg["iters"], 0.0, time_loop=True)
    t1 = time.perf_counter()
    g = skb.potentials_backward(r.log_u, r.log_v, cfg["lam"], up)
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"solve host {1e3*(t1-t0):.2f} ms, step wall {1e3*(t2-t0):.2f} ms, "
          f"step events {e0.elapsed_time(e1):.2f} ms, loop events {r.loop_ms:.2f} ms, "
          f"exact reruns {lib.sinkhorn_exact_reruns_v1() - r0}")
