"""Shape probe through the raw C ABI of any library build (regression hunting):
    python tools/iso_probe_raw.py LIB d1 d2 flags"""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from paper_1907_01729_b200 import _lib as L

lib = ctypes.CDLL(sys.argv[1])
d1, d2, flags = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
B = 6
dev = torch.device('cuda', 0)
rng = np.random.default_rng(0)
mu = torch.tensor(rng.uniform(0.5, 1.5, (B, d1)), dtype=torch.float64); mu = (mu / mu.sum(1, keepdim=True)).float().to(dev)
nu = torch.tensor(rng.uniform(0.5, 1.5, (B, d2)), dtype=torch.float64); nu = (nu / nu.sum(1, keepdim=True)).float().to(dev)
c = torch.rand(d1, d2, device=dev)
pr = L.Problem(); pr.B, pr.d1, pr.d2, pr.cost_kind = B, d1, d2, 0
op = L.Options(); op.lam, op.max_iters, op.check_interval, op.tolerance, op.flags = 0.1, 60, 10, 0.0, flags
lib.sinkhorn_workspace_bytes_v1.restype = ctypes.c_size_t
nb = lib.sinkhorn_workspace_bytes_v1(ctypes.byref(pr))
ws = torch.empty(nb, dtype=torch.uint8, device=dev)
oc = torch.empty(B, device=dev); lu = torch.empty(B, d1, device=dev); lv = torch.empty(B, d2, device=dev)
it = ctypes.c_int32(0); res = torch.empty(B, device=dev)
P = ctypes.c_void_p
st = lib.sinkhorn_forward_device_v1(ctypes.byref(pr), ctypes.byref(op), P(mu.data_ptr()), P(nu.data_ptr()), P(c.data_ptr()),
    P(oc.data_ptr()), P(lu.data_ptr()), P(lv.data_ptr()), ctypes.byref(it), P(res.data_ptr()), P(ws.data_ptr()), ctypes.c_size_t(nb), P(torch.cuda.current_stream().cuda_stream))
lib.sinkhorn_last_error.restype = ctypes.c_char_p
lib.sinkhorn_last_path_v1.restype = ctypes.c_char_p
print(sys.argv[1].split('/')[-1], d1, d2, flags, 'status', st, lib.sinkhorn_last_path_v1(), lib.sinkhorn_last_error()[:80] if st else '', oc[:2].tolist() if st == 0 else '')
