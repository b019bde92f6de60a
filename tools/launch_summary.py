"""Summarise an ncu launch-list CSV (--metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum])
of one bench step as markdown: python tools/launch_summary.py launches.csv title [traffic.json] > x.md
With dram metrics, also writes the K2 DRAM traffic per step (read + write of the step's 4 K2 launches) to
traffic.json — bench.py reports it as roofline.traffic."""
import csv
import json
import sys

path = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else path
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h = rows[0]
ki, vi, gi, ni, ii = (h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size"), h.index("Metric Name"),
                      h.index("ID"))
mets = {}
for r in rows[1:]:
    if r[ki].startswith("void mq::"):
        mets.setdefault(r[ii], {"name": r[ki], "grid": r[gi]})[r[ni]] = float(r[vi].replace(",", ""))
data = [mets[k] for k in sorted(mets, key=int)]
step = data[-8:]  # last step: 4 x (K1, K2)
print(f"# ncu launch list — {title}\n")
print("`ncu --metrics gpu__time_duration.sum --clock-control none -c 400` — cold-cache and serialised "
      "(no PDL overlap), so compare SHARES, not absolute times.\n")
print("One step = 4 x (K1 act_quant_eal + K2 mixed_gemm) for qkv (6144x4096), o (4096x4096), "
      "gate_up (28672x4096), down (4096x14336), M=16.\n")
tot = k2 = 0.0
traffic = 0.0
has_dram = all("dram__bytes_read.sum" in r for r in step)
if has_dram:
    print("| # | kernel | grid | us | DRAM read MB | DRAM write MB |\n|---|---|---|---|---|---|")
else:
    print("| # | kernel | grid | us |\n|---|---|---|---|")
for i, r in enumerate(step):
    us = r["gpu__time_duration.sum"] / 1e3
    tot += us
    name = r["name"].split("(")[0]
    extra = ""
    if has_dram:
        rd, wr = r["dram__bytes_read.sum"], r["dram__bytes_write.sum"]
        extra = f" {rd / 1e6:.2f} | {wr / 1e6:.2f} |"
        if "mixed_gemm" in name:
            traffic += rd + wr
    if "mixed_gemm" in name:
        k2 += us
    print(f"| {i} | `{name}` | {r['grid']} | {us:.2f} |" + extra)
print(f"\nK2 share of the step (serialised): {k2:.1f} of {tot:.1f} us = {100 * k2 / tot:.0f}%")
if has_dram:
    print(f"\nK2 DRAM traffic per step (read + write, 4 launches): {traffic / 1e6:.2f} MB")
    if len(sys.argv) > 3:
        json.dump({"k2_dram_bytes_per_step": traffic, "source": path,
                   "note": "ncu dram__bytes_read.sum + dram__bytes_write.sum of the step's 4 K2 launches "
                           "(serialised replay, cold L2)"}, open(sys.argv[3], "w"), indent=1)
