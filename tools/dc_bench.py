"""dC = sum_b up_b P_b (shared cost): the tensor-core contraction vs the direct
per-cell sum, CUDA-event timed.   python tools/dc_bench.py B d"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1907_01729_b200 as skb  # noqa: E402
from paper_1907_01729_b200 import _lib  # noqa: E402

B, d = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
lu = torch.randn(B, d, generator=g, device=dev) * 0.1 - 6.0
lv = torch.randn(B, d, generator=g, device=dev) * 0.1 - 6.0
i = torch.arange(d, device=dev, dtype=torch.float32)
c = ((i[:, None] - i[None, :]).abs() / (d - 1)) ** 2
up = torch.randn(B, generator=g, device=dev)
lib = _lib.load()
pr = _lib.Problem()
pr.B, pr.d1, pr.d2, pr.cost_kind = B, d, d, _lib.COST_SHARED
out = torch.empty_like(c)
st = torch.cuda.current_stream().cuda_stream


def direct():
    lib.sinkhorn_plan_grad_device_v1(ctypes.byref(pr), 0.05, lu.data_ptr(), lv.data_ptr(),
                                     c.data_ptr(), up.data_ptr(), out.data_ptr(), st)


def tensor_core():
    skb.plan_gradient(lu, lv, c, 0.05, up)


for name, fn in (("direct", direct), ("tensor-core", tensor_core)):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"dC B={B} d={d} {name}: {e0.elapsed_time(e1) / 5:.3f} ms")
