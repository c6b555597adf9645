"""Per-sample dC = up_b P_b (config-4 shape, HBM-bound), CUDA-event timed.

    python tools/dc_per_sample_bench.py
"""
import ctypes, sys, torch
sys.path.insert(0, ".")
from paper_1907_01729_b200 import _lib
B, d = 1024, 1024
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(0)
lu = torch.randn(B, d, generator=g, device=dev) * 0.1 - 6.0
lv = torch.randn(B, d, generator=g, device=dev) * 0.1 - 6.0
c = torch.rand(B, d, d, generator=g, device=dev)
up = torch.randn(B, generator=g, device=dev)
out = torch.empty_like(c)
lib = _lib.load(); pr = _lib.Problem(); pr.B, pr.d1, pr.d2, pr.cost_kind = B, d, d, _lib.COST_PER_SAMPLE
st = torch.cuda.current_stream().cuda_stream
def run():
    assert lib.sinkhorn_plan_grad_device_v1(ctypes.byref(pr), 0.05, lu.data_ptr(), lv.data_ptr(), c.data_ptr(), up.data_ptr(), out.data_ptr(), st) == 0
run(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): run()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"per-sample dC B={B} d={d}: {ms:.3f} ms, {2 * 4 * B * d * d / (ms * 1e-3) / 1e9:.0f} GB/s")
ref = up[:, None, None] * torch.exp(lu[:, :, None] + lv[:, None, :] - c / 0.05)
print("max rel err", float(((out - ref).abs() / ref.abs().clamp_min(1e-30)).max()))
