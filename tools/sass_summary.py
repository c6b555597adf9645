"""Per-kernel SASS mnemonic counts of the built library (cuobjdump -sass), the
evidence that the hot kernels use tcgen05 (UTC*MMA, LDTM/STTM), TMA
(UTMALDG / UBLKCP) and packed fp32 (FFMA2/FADD2).

    python tools/sass_summary.py > profiles/r02_sass_summary.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1907_01729_b200", "_lib", "libsinkhorn_b200.so")
WATCH = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTCATOMSWS", "LDTM", "STTM", "UTMALDG", "UBLKCP",
         "SYNCS", "FFMA2", "FADD2", "FMUL2", "FFMA", "MUFU.EX2", "MUFU.LG2", "LDS", "LDG", "STG",
         "HMMA", "BAR"]
KERNELS = ["umma_gemm_kernel", "umma_fixup_kernel", "umma_kernel_matrices", "fused_ps_kernel",
           "fgemm_pass_kernel", "fused_merge_kernel", "tiled_sweep_kernel", "sep_sweep_kernel",
           "small_solve_kernel", "lane_col_kernel"]

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)
print("# SASS mnemonic counts (static instruction counts per kernel)\n")
print(f"`cuobjdump -sass {os.path.relpath(LIB, ROOT)}`; one row per instantiation of the hot kernels.\n")
print("| kernel | " + " | ".join(WATCH) + " |")
print("|---|" + "---|" * len(WATCH))
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    if not any(k in dem for k in KERNELS):
        continue
    ops = collections.Counter()
    for line in f.splitlines():
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m:
            ops[m.group(1)] += 1
    def count(key):
        return sum(v for k, v in ops.items() if k == key or k.startswith(key + "."))
    short = dem.split("(")[0].replace("skb::", "")
    print(f"| `{short[:70]}` | " + " | ".join(str(count(k)) for k in WATCH) + " |")
