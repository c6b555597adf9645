"""Time the sections of loss.solve() to locate sporadic host stalls (diagnostic)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1907_01729_b200 as skb
from paper_1907_01729_b200 import _lib, loss as L
from bench import CONFIGS, make_inputs
cfg = CONFIGS[2]
dev = torch.device("cuda", 0)
mu, nu, cost = make_inputs(cfg, dev, 1)
up = torch.ones(256, device=dev)
lib = _lib.load()
for i in range(12):
    T = [time.perf_counter()]
    pr = L._problem(256, 784, 784, cost)
    op = _lib.Options(); op.lam = 0.05; op.max_iters = 100; op.check_interval = 10
    op.tolerance = 0.0; op.flags = _lib.FLAG_TIME_LOOP
    T.append(time.perf_counter())
    out_cost = torch.empty(256, device=dev); log_u = torch.empty(256, 784, device=dev)
    log_v = torch.empty(256, 784, device=dev); res = torch.empty(256, device=dev)
    T.append(time.perf_counter())
    nbytes = lib.sinkhorn_workspace_bytes_v1(ctypes.byref(pr))
    ws = L._workspace(dev, nbytes)
    T.append(time.perf_counter())
    it = ctypes.c_int32(0)
    st = lib.sinkhorn_forward_device_v1(ctypes.byref(pr), ctypes.byref(op), mu.data_ptr(),
        nu.data_ptr(), cost.data_ptr(), out_cost.data_ptr(), log_u.data_ptr(), log_v.data_ptr(),
        ctypes.byref(it), res.data_ptr(), ws.data_ptr(), ws.numel(), L._stream_handle(dev))
    T.append(time.perf_counter())
    g = skb.potentials_backward(log_u, log_v, 0.05, up)
    T.append(time.perf_counter())
    d = [1e3 * (b - a) for a, b in zip(T, T[1:])]
    print("sections ms: prob %.3f alloc %.3f ws %.3f forward %.2f backward %.2f | loop %.2f" %
          (*d, lib.sinkhorn_last_loop_ms_v1()))
