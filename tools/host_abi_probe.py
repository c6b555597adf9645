"""The reference-facing host ABI (sinkhorn_forward_v1 / sinkhorn_backward_v1,
float64 host views) on odd shapes against the float64 oracle.
    python tools/host_abi_probe.py
"""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import sinkhorn_oracle as orc  # noqa: E402
from paper_1907_01729_b200 import _lib  # noqa: E402

lib = _lib.load()


def view(a):
    v = _lib.View()
    v.data = a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    v.ndim = a.ndim
    v.shape[0] = a.shape[0]
    v.shape[1] = a.shape[1] if a.ndim == 2 else 0
    v.length = a.size
    return v


fails = 0
for B, d1, d2 in [(1, 1, 1), (3, 7, 1), (2, 1025, 3), (5, 129, 130), (70000, 4, 4), (2, 1500, 900)]:
    rng = np.random.default_rng(B + d1 + d2)
    mu = orc.random_histogram_batch(B, d1, rng)
    nu = orc.random_histogram_batch(B, d2, rng)
    c = rng.random((d1, d2))
    lam, iters = 0.1, 20
    oc, ou, ov = np.zeros(B), np.zeros((B, d1)), np.zeros((B, d2))
    vs = [view(a) for a in (mu, nu, c, oc, ou, ov)]
    st = lib.sinkhorn_forward_v1(*(ctypes.byref(v) for v in vs[:3]), lam, iters, 0.0,
                                 *(ctypes.byref(v) for v in vs[3:]))
    up = np.ones(B)
    gm, gn = np.zeros((B, d1)), np.zeros((B, d2))
    vb = [view(a) for a in (ou, ov, up, gm, gn)]
    st2 = lib.sinkhorn_backward_v1(ctypes.byref(vb[0]), ctypes.byref(vb[1]), lam,
                                   ctypes.byref(vb[2]), ctypes.byref(vb[3]), ctypes.byref(vb[4]))
    if B <= 8:
        ref = orc.batch_forward(mu, nu, c, lam, iters, 0.0, workers=4)
        gref, _ = orc.batch_backward(ref.log_u, ref.log_v, lam, up)
        rel = float(np.max(np.abs(oc - ref.cost_e0) / np.maximum(np.abs(ref.cost_e0), 1e-300)))
        gerr = float(np.max(np.abs(gm - gref)))
    else:   # lanes 0 and B-1 against one-lane oracle solves
        rel = gerr = 0.0
        for b in (0, B - 1):
            r = orc.batch_forward(mu[b:b + 1], nu[b:b + 1], c, lam, iters, 0.0, workers=1)
            g, _ = orc.batch_backward(r.log_u, r.log_v, lam, np.ones(1))
            rel = max(rel, abs(oc[b] - r.cost_e0[0]) / max(abs(r.cost_e0[0]), 1e-300))
            gerr = max(gerr, float(np.max(np.abs(gm[b] - g[0]))))
    ok = st == 0 and st2 == 0 and rel <= 1e-5 and gerr <= 1e-4
    fails += not ok
    print("OK  " if ok else "FAIL", B, d1, d2, "status", st, st2, f"rel {rel:.1e} grad {gerr:.1e}",
          flush=True)
print("FAILURES", fails)
