import os, sys, time, ctypes
sys.path.insert(0, "/root/repo")
import torch
import paper_1907_01729_b200 as skb
from paper_1907_01729_b200 import _lib, loss as L
from bench import CONFIGS, make_inputs
cfg = CONFIGS[2]
dev = torch.device("cuda", 0)
mu, nu, cost = make_inputs(cfg, dev, 1)
lib = _lib.load()
pr = L._problem(256, 784, 784, cost)
op = _lib.Options(); op.lam=0.05; op.max_iters=100; op.check_interval=10; op.tolerance=0.0; op.flags=_lib.FLAG_TIME_LOOP
nbytes = lib.sinkhorn_workspace_bytes_v1(ctypes.byref(pr))
ws = torch.empty(nbytes, device=dev, dtype=torch.uint8)
oc = torch.empty(256, device=dev); lu = torch.empty(256,784,device=dev); lv = torch.empty(256,784,device=dev); rs=torch.empty(256,device=dev)
st = torch.cuda.current_stream(dev).cuda_stream
it = ctypes.c_int32(0)
for i in range(14):
    t0 = time.perf_counter()
    s = lib.sinkhorn_forward_device_v1(ctypes.byref(pr), ctypes.byref(op), mu.data_ptr(), nu.data_ptr(), cost.data_ptr(), oc.data_ptr(), lu.data_ptr(), lv.data_ptr(), ctypes.byref(it), rs.data_ptr(), ws.data_ptr(), ws.numel(), st)
    t1 = time.perf_counter()
    print(f"raw C call {1e3*(t1-t0):.2f} ms loop {lib.sinkhorn_last_loop_ms_v1():.2f} status {s}")
