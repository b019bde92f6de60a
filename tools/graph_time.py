"""Per-launch device time of K2 inside a CUDA graph (no host overhead), PDL on:
20 back-to-back launches alternating 2 weight replicas (> L2 for big shapes).
python tools/graph_time.py [M]   (MQ_DBG / MQ_LIB select development variants)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi

M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
SH = [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)]
for (N, K) in SH:
    W, A, prom = mq.bench_inputs(M, N, K, float(os.environ.get("FRAC", "0.1")), 1)
    L = mq.partition_and_quantize(W, prom)
    reps = [mq.DeviceLayer(L) for _ in range(2)]
    dA = torch.from_numpy(A).cuda()
    opts = mq.exec_opts(capi.MQ_FAST, 128, ksplit=int(os.environ.get("KSPLIT", "0")), schedule=int(os.environ.get("SCHED", "0")), pdl=os.environ.get("NOPDL") is None, token_tile=int(os.environ.get("TT", "0")))
    wss = [r.quantize_ws(dA, opts) for r in reps]
    Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
    for i in range(4):
        reps[i % 2].forward_ws(M, wss[i % 2], out=Y, opts=opts)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(20):
            reps[i % 2].forward_ws(M, wss[i % 2], out=Y, opts=opts)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 200
    wb = reps[0].info.weight_stream_bytes
    print(f"sched={os.environ.get('SCHED', '0')} ks={os.environ.get('KSPLIT', '0')} dbg={os.environ.get('MQ_DBG', '0'):>3s} frac={os.environ.get('FRAC', '0.1')} N={N} K={K} M={M}: {us:6.2f} us/launch  {wb / us / 1e3:6.0f} GB/s", flush=True)
