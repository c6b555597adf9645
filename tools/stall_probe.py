"""Step-time outliers under different clock samplers (diagnostic).

    python tools/stall_probe.py [none|smi|nvml] [steps]
"""
import os
import statistics
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1907_01729_b200 as skb  # noqa: E402
from bench import CONFIGS, make_inputs  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "none"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 60
cfg = CONFIGS[2]
dev = torch.device("cuda", 0)
mu, nu, cost = make_inputs(cfg, dev, 1)
for _ in range(3):
    skb.solve(mu, nu, cost, cfg["lam"], cfg["iters"], 0.0, 10)
stop = threading.Event()
proc = None
if mode in ("smi", "smi_full", "smi_nopower"):
    fields = {"smi": "clocks.sm,clocks.max.sm",
              "smi_full": "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                          "clocks_event_reasons.hw_thermal_slowdown,"
                          "clocks_event_reasons.sw_thermal_slowdown,"
                          "clocks_event_reasons.sw_power_cap,timestamp",
              "smi_nopower": "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                             "clocks_event_reasons.hw_thermal_slowdown,"
                             "clocks_event_reasons.sw_thermal_slowdown,"
                             "clocks_event_reasons.sw_power_cap,timestamp"}[mode]
    proc = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={fields}",
                             "--format=csv,noheader", "-lms", "100"], stdout=subprocess.DEVNULL)
    time.sleep(1.0)
elif mode == "nvml":
    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)

    def loop():
        while not stop.is_set():
            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            time.sleep(0.1)
    threading.Thread(target=loop, daemon=True).start()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
      for _ in range(steps)]
torch.cuda.synchronize()
for a, b in ev:
    a.record()
    skb.solve(mu, nu, cost, cfg["lam"], cfg["iters"], 0.0, 10)
    b.record()
torch.cuda.synchronize()
stop.set()
if proc:
    proc.terminate()
ms = [a.elapsed_time(b) for a, b in ev]
print(f"{mode}: mean {statistics.mean(ms):.3f} median {statistics.median(ms):.3f} "
      f"max {max(ms):.3f} >11ms: {sum(m > 11 for m in ms)}/{steps}")
