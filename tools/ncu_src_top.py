"""Top stall lines (CUDA source) of an ncu report: python tools/ncu_src_top.py rep.ncu-rep [n]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
# find header row with "Line No"/"# Address"
hi = next(i for i, r in enumerate(rows) if r and ("Line No" in r[0] or "#" in r[0] or "Source" in r))
h = rows[hi]
data = [dict(zip(h, r)) for r in rows[hi + 1:] if len(r) == len(h)]
def f(x):
    try: return float(x)
    except: return 0.0
key = "Warp Stall Sampling (All Samples)"
tot = sum(f(d.get(key, 0)) for d in data) or 1
print("columns:", [c for c in h][:6], "total samples", tot)
for d in sorted(data, key=lambda d: -f(d.get(key, 0)))[:n]:
    print(f"{f(d.get(key,0))/tot*100:5.1f}%  L{d.get('Line No', d.get('#',''))}: {d.get('Source','')[:110]}")
