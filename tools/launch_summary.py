"""Summarise an ncu launch-list CSV (--metrics gpu__time_duration.sum) of one
bench step as markdown: python tools/launch_summary.py launches.csv title > x.md"""
import csv
import sys

path = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else path
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h = rows[0]
ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
data = [r for r in rows[1:] if r[ki].startswith("void mq::")]
step = data[-8:]  # last step: 4 x (K1, K2)
print(f"# ncu launch list — {title}\n")
print("`ncu --metrics gpu__time_duration.sum --clock-control none -c 400` — cold-cache and serialised "
      "(no PDL overlap), so compare SHARES, not absolute times.\n")
print("One step = 4 x (K1 act_quant_eal + K2 mixed_gemm) for qkv (6144x4096), o (4096x4096), "
      "gate_up (28672x4096), down (4096x14336), M=16.\n")
print("| # | kernel | grid | us |\n|---|---|---|---|")
tot = k2 = 0.0
for i, r in enumerate(step):
    us = float(r[vi]) / 1e3
    tot += us
    name = r[ki].split("(")[0]
    if "mixed_gemm" in name:
        k2 += us
    print(f"| {i} | `{name}` | {r[gi]} | {us:.2f} |")
print(f"\nK2 share of the step (serialised): {k2:.1f} of {tot:.1f} us = {100 * k2 / tot:.0f}%")
