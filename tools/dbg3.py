import sys, os
sys.path.insert(0, "/root/repo")
import torch
import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi
N, K, M = (int(x) for x in sys.argv[1:4])
W, A, prom = mq.bench_inputs(M, N, K, 0.1, 1)
L = mq.partition_and_quantize(W, prom)
reps = 4
layers = [mq.DeviceLayer(L) for _ in range(reps)]
dA = torch.from_numpy(A).cuda()
Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
opts = mq.exec_opts(capi.MQ_FAST, 128, ksplit=int(os.environ.get("KSPLIT", "0")), pdl=os.environ.get("NOPDL", "0") != "1")
ws = layers[0].quantize_ws(dA, opts)
for dl in layers: dl.forward_ws(M, ws, out=Y, opts=opts)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(20): layers[i % reps].forward_ws(M, ws, out=Y, opts=opts)
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
print(f"dbg={os.environ.get('MQ_DBG','0')} nopdl={os.environ.get('NOPDL','0')} ksplit={os.environ.get('KSPLIT','0')} N={N} K={K} M={M}: {us:.2f} us/launch  {layers[0].info.weight_stream_bytes/us/1e3:.0f} GB/s(weights)")
