"""Per-CTA timeline of one K2 launch (globaltimer stamps of the -DMQ_DEV build):
python tools/trace_k2.py N K M [pdl]   with MQ_LIB=build_var/libmq_dev.so MQ_DBG=32.
The traced launch is the last of 6 back-to-back launches (steady state)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi

N, K, M = (int(x) for x in sys.argv[1:4])
pdl = len(sys.argv) <= 4 or sys.argv[4] != "0"
W, A, prom = mq.bench_inputs(M, N, K, 0.1, 1)
L = mq.partition_and_quantize(W, prom)
dls = [mq.DeviceLayer(L) for _ in range(2)]
dA = torch.from_numpy(A).cuda()
Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
opts = mq.exec_opts(capi.MQ_FAST, 128, pdl=pdl, ksplit=int(os.environ.get("KSPLIT", "0")))
wss = [d.quantize_ws(dA, opts) for d in dls]
for i in range(6):
    dls[i % 2].forward_ws(M, wss[i % 2], out=Y, opts=opts)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (148 * 8 + 1024))()
capi.lib().mq_debug_trace(buf)
raw = np.array(buf, dtype=np.float64)
a = raw[:148 * 8].reshape(148, 8)
ok = a[:, 0] > 0
base = a[ok, 0].min()
a = np.where(a > 0, a - base, np.nan) / 1000.0
names = ["start", "prod_all_issued", "prod_enter", "epi_first_tfull", "epi_units_done", "epi_exit", "end",
         "prod_first_issue"]
print(f"N={N} K={K} M={M} pdl={pdl}: {int(ok.sum())} CTAs traced (us from the first CTA start)")
for i in (0, 2, 7, 1, 3, 4, 5, 6):
    col = a[:, i]
    if np.all(np.isnan(col)):
        continue
    print(f"  {names[i]:16s} min {np.nanmin(col):6.2f} med {np.nanmedian(col):6.2f} max {np.nanmax(col):6.2f}")
if int(os.environ.get("MQ_DBG", "0")) & 64:
    ch = raw[148 * 8:].reshape(16, 64)
    t0 = ch[14, 0]
    print(f"CTA {int(os.environ['MQ_DBG']) >> 8} chunk timeline (kcycles from CTA start; end at {(ch[15, 0] - t0) / 1e3:.2f}):")
    ev = [(0, "w_issue"), (10, "x_issue"), (5, "conv_full"), (6, "conv_slot"), (3, "conv_done"), (7, "mma_w"),
          (8, "mma_x"), (9, "mma_a"), (1, "mma_go"), (2, "mma_commit"), (13, "epi_full"), (4, "epi_done"),
          (11, "st_begin"), (12, "st_end")]
    print("  producer prologue (kcycles): " + " ".join(f"{(ch[15, i] - t0) / 1e3:.2f}" for i in range(1, 6)))
    print("  last join sums loaded at: " + (f"{(ch[15, 8] - t0) / 1e3:.2f}" if ch[15, 8] > 0 else "-"))
    print("  n " + " ".join(f"{nm:>10s}" for _, nm in ev))
    for n in range(64):
        row = [ch[e, n] for e, _ in ev]
        if not any(v > 0 for v in row):
            continue
        print(f"{n:3d} " + " ".join(f"{(v - t0) / 1e3:10.2f}" if v > 0 else "         -" for v in row))
