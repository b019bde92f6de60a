"""Top stall SASS instructions of an ncu report: python tools/ncu_sass_top.py rep.ncu-rep [n] [grep]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
pat = sys.argv[3] if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) >= len(h) - 1]
def f(x):
    try: return float(x)
    except: return 0.0
key = "Warp Stall Sampling (All Samples)"
tot = sum(f(d.get(key, 0)) for d in data) or 1
stalls = [c for c in h if c.startswith("stall_")]
print("total samples", tot, "instructions", len(data))
sel = [d for d in data if (pat is None or pat in d["Source"])]
for d in sorted(sel, key=lambda d: -f(d.get(key, 0)))[:n]:
    top = sorted(((f(d[c]), c[6:]) for c in stalls), reverse=True)[:3]
    print(f"{f(d.get(key,0))/tot*100:5.1f}% {d['Address'][-5:]} {d['Source'].strip()[:60]:60s} ex={d['Instructions Executed']:>8s} l2sec={d.get('L2 Theoretical Sectors Global','')} " + " ".join(f"{c}:{v:.0f}" for v, c in top if v))
