"""Device time of the bench stack (K1 + K2 per projection, CUDA graph, PDL), the
bench's `value` step without the harness: python tools/stack_time.py [M]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi

M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
SH = [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)]
reps = []
for r in range(2):
    layers = []
    for i, (N, K) in enumerate(SH):
        W, _, prom = mq.bench_inputs(1, N, K, 0.1, 1 + i)
        layers.append(mq.DeviceLayer(mq.partition_and_quantize(W, prom)))
    reps.append(layers)
xs = [torch.randn((M, K), device="cuda") for (_, K) in SH]
ys = [torch.empty((M, N), dtype=torch.float16, device="cuda") for (N, _) in SH]
opts = mq.exec_opts(capi.MQ_FAST, 128)
gs = []
for r in range(2):
    for i in range(4):
        reps[r][i].forward(xs[i], out=ys[i], opts=opts)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(4):
            reps[r][i].forward(xs[i], out=ys[i], opts=opts)
    gs.append(g)
for k in range(20):
    gs[k % 2].replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for k in range(100):
    gs[k % 2].replay()
e1.record()
torch.cuda.synchronize()
print(f"M={M}: {e0.elapsed_time(e1) * 10:.2f} us per stack step", flush=True)
