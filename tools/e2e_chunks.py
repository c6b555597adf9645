"""Config-4 e2e step time against the lane-group schedule of solve_streamed.

  python tools/e2e_chunks.py            (on the GPU box)

Prints ms per step (upload + solve + backward + readback, as bench.py's e2e
leg) for equal groups and for ramped schedules (short first / last groups).
"""
import json
import sys
import time

sys.path.insert(0, ".")

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1907_01729_b200 as skb  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    cfg = bench.CONFIGS[4]
    mu, nu, cost = bench.make_inputs(cfg, dev, 0)
    lam, iters = cfg["lam"], cfg["iters"]
    B = cfg["B"]
    h_mu, h_nu = bench.pinned_copy(mu), bench.pinned_copy(nu)
    h_c = bench.pinned_copy(cost)
    # device-resident solve time per lane-group size (the pipeline's compute side)
    for g in (32, 64, 128, 256, 1024):
        for _ in range(2):
            skb.solve(mu[:g], nu[:g], cost[:g], lam, iters, 0.0, asynchronous=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            skb.solve(mu[:g], nu[:g], cost[:g], lam, iters, 0.0, asynchronous=True)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / 3 * 1e3
        print(f"device solve B={g}: {ms:.2f} ms, {ms / g * 1024:.1f} ms per 1024 lanes", flush=True)
    del cost
    torch.cuda.empty_cache()
    h_loss = torch.empty(B).pin_memory()
    h_gm = torch.empty(B, cfg["d"]).pin_memory()
    h_gn = torch.empty(B, cfg["d"]).pin_memory()

    def step(chunks, ns=2):
        res = skb.solve_streamed(h_mu, h_nu, h_c, lam, iters, 0.0, chunks=chunks, device=dev,
                                 compute_streams=ns)
        gm, gn = skb.potentials_backward(res.log_u, res.log_v, lam, torch.ones(B, device=dev))
        h_loss.copy_(res.cost_e0, non_blocking=True)
        h_gm.copy_(gm, non_blocking=True)
        h_gn.copy_(gn, non_blocking=True)
        torch.cuda.synchronize()

    schedules = {"equal8_1stream": (8, 1), "equal8_2streams": (8, 2), "equal16_2streams": (16, 2),
                 "equal16_3streams": (16, 3), "equal24_2streams": (24, 2),
                 "equal32_2streams": (32, 2), "equal32_3streams": (32, 3)}
    out = {}
    for name, (ch, ns) in schedules.items():
        step(ch, ns)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            step(ch, ns)
            ts.append((time.perf_counter() - t0) * 1e3)
        ts.sort()
        out[name] = {"ms_median": ts[2], "ms_min": ts[0]}
        print(name, f"{ts[2]:.2f} ms (min {ts[0]:.2f})", flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
