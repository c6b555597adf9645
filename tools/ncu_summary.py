"""Summarise ncu reports / launch lists into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py report gpurun_out/prof.ncu-rep > profiles/rNN_x.md
    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/rNN_launches.md
    python tools/ncu_summary.py traffic gpurun_out/prof.ncu-rep config2   # -> profiles/ncu_summary.json
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_active.avg", "sm__cycles_active.max", "sm__cycles_elapsed.max",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
]


def raw(rep: str):
    """The raw page of a report, or an exported `ncu -i rep --page raw --csv` file."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return [dict(zip(r[0], row)) for row in r[2:]], dict(zip(r[0], r[1]))


def report(rep: str) -> None:
    rows, units = raw(rep)
    print(f"# ncu --set full summary: `{os.path.basename(rep)}`\n")
    for i, d in enumerate(rows):
        print(f"## launch {i}: {d.get('Kernel Name', '')[:120]}\n")
        for k in KEYS:
            if k in d:
                print(f"- `{k}`: {d[k]} {units.get(k, '')}")
        stalls = []
        for h, v in d.items():
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith(
                    "per_issue_active.ratio"):
                try:
                    stalls.append((float(v), h.split("stalled_")[1].split("_per")[0]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("- top stall reasons (warps per issue): " +
              ", ".join(f"{n} {v:.2f}" for v, n in stalls[:6]))
        print()


def launches(path: str) -> None:
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"])
        unit = d.get("Metric Unit", "nsecond")
        v *= {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}.get(unit, 1.0)
        name = d["Kernel Name"].split("(")[0][:90]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values()) or 1.0
    print(f"# launch list `{os.path.basename(path)}` (ncu gpu__time_duration, cold, serialised)\n")
    print("| launches | total us | share | kernel |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {v[0]} | {v[1] / 1e3:.1f} | {100 * v[1] / tot:.1f}% | `{k}` |")


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def traffic(rep: str, cfg: str) -> None:
    rows, units = raw(rep)
    vals = []
    for d in rows:
        try:
            vals.append(sum(float(d[k].replace(",", "")) * SCALE.get(units.get(k, "byte"), 1.0)
                            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum")))
        except (KeyError, ValueError):
            pass
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "ncu_summary.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data[cfg] = {"dram_bytes_per_sweep_launch": sum(vals) / max(len(vals), 1),
                 "source": os.path.basename(rep)}
    json.dump(data, open(path, "w"), indent=1)
    print(json.dumps(data[cfg]))


if __name__ == "__main__":
    {"report": lambda: report(sys.argv[2]), "launches": lambda: launches(sys.argv[2]),
     "traffic": lambda: traffic(sys.argv[2], sys.argv[3])}[sys.argv[1]]()
