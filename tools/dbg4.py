import sys, os, ctypes as C
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi
N, K, M = (int(x) for x in sys.argv[1:4])
W, A, prom = mq.bench_inputs(M, N, K, 0.1, 1)
L = mq.partition_and_quantize(W, prom)
dl = mq.DeviceLayer(L)
dA = torch.from_numpy(A).cuda()
Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
opts = mq.exec_opts(capi.MQ_FAST, 128, pdl=False, ksplit=int(os.environ.get("KSPLIT", "0")))
ws = dl.quantize_ws(dA, opts)
for _ in range(3): dl.forward_ws(M, ws, out=Y, opts=opts)
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record(); dl.forward_ws(M, ws, out=Y, opts=opts); t1.record(); torch.cuda.synchronize()
print("event us", t0.elapsed_time(t1) * 1e3)
buf = (C.c_ulonglong * (148 * 8 + 1024))()
n = capi.lib().mq_debug_trace(buf)
raw = np.array(buf, dtype=np.float64)
a = raw[:148*8].reshape(148, 8)
base = a[:, 0][a[:, 0] > 0].min()
a = np.where(a > 0, a - base, np.nan) / 1000.0
names = ["start", "prod_all_issued", "prod_enter", "epi_first_tfull", "epi_unit_done", "epi_exit", "end", "prod_first_issue"]
for i, nm in enumerate(names):
    col = a[:, i]
    print(f"{nm:16s} min {np.nanmin(col):7.2f} med {np.nanmedian(col):7.2f} max {np.nanmax(col):7.2f} us")

order = np.argsort(-np.nan_to_num(a[:, 5], nan=-1))[:6]
print("slowest CTAs (epi_exit):", [(int(i), round(float(a[i, 5]), 2), round(float(a[i, 4]), 2)) for i in order])
ch = raw[148*8:].reshape(16, 64)
b = min(v for v in ch[:8].reshape(-1) if v > 0)
print("CTA chunk timeline (kcycles): issue / mma_start / mma_commit / conv_done / epi_done / conv_full / conv_waits / mma_wfull / mma_wx / mma_wa / xprod_issue / store_begin / store_end / epi_start")
for n in range(int(os.environ.get('NCH', '40'))):
    row = ch[:14, n]
    if row[1] == 0 and row[11] == 0: continue
    print(n, " ".join(f"{(v-b)/1000:7.2f}" if v > 0 else "    -  " for v in row))
