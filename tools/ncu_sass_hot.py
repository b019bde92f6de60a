"""Hottest CUDA source lines of an ncu report by warp instructions executed and by
warp-stall samples: python tools/ncu_sass_hot.py rep.ncu-rep [n] [inst|stall]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
by = sys.argv[3] if len(sys.argv) > 3 else "inst"
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = next(i for i, r in enumerate(rows) if r and r[0] in ("Address", "# Address", "Line No"))
h = rows[hi]
col = h.index("Instructions Executed" if by == "inst" else "Warp Stall Sampling (All Samples)")
cur = None
agg = defaultdict(int)
total = 0
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    if r[0].isdigit() and not r[0].startswith("0x"):  # a CUDA source line header
        cur = (r[0], r[1].strip()[:90])
        continue
    try:
        v = int(float(r[col]))
    except ValueError:
        continue
    total += v
    agg[cur] += v
print(f"total {by} {total}")
for (k, v) in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{v / max(total, 1) * 100:5.1f}%  {v:9d}  L{k[0] if k else '?'}: {k[1] if k else ''}")
