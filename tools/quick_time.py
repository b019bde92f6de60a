"""Quick device timing of the engine on a few shapes (development aid)."""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi


def bench(n, k, m, mode, act_group=128, iters=50, reps=8, token_tile=0, ksplit=0):
    W, A, prom = mq.bench_inputs(m, n, k, 0.1, 1)
    L = mq.partition_and_quantize(W, prom)
    layers = [mq.DeviceLayer(L) for _ in range(reps)]  # rotate > L2 for big shapes
    dA = torch.from_numpy(A).cuda()
    opts = mq.exec_opts(mode, act_group, ksplit=ksplit, token_tile=token_tile)
    ws = layers[0].quantize_ws(dA, opts)
    Y = torch.empty((m, n), dtype=torch.float16, device="cuda")
    for dl in layers:
        dl.forward_ws(m, ws, out=Y, opts=opts)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        layers[i % reps].forward_ws(m, ws, out=Y, opts=opts)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / iters * 1e3
    info = layers[0].info
    byts = info.weight_stream_bytes + m * k + m * 4 * ((k + 127) // 128) + m * n * 2
    print(f"N={n} K={k} M={m} mode={mode} ag={act_group}: {us:.2f} us  {byts/us/1e3:.0f} GB/s  {2*m*n*k/us/1e6:.1f} TOPS", flush=True)


if __name__ == "__main__" and not (len(sys.argv) > 1 and sys.argv[1] == "prefill"):
    for m in (1, 16, 64, 128, 256, 512):
        bench(4096, 4096, m, capi.MQ_FAST)
    for m in (16, 512):
        bench(4096, 4096, m, capi.MQ_EXACT)
        bench(4096, 4096, m, capi.MQ_FAST, act_group=4096)
    for m in (16, 512):
        bench(14336, 4096, m, capi.MQ_FAST, reps=4)
        bench(28672, 8192, m, capi.MQ_FAST, reps=2)
if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "prefill":
    for m in (256, 512, 1024, 2048):
        bench(14336, 4096, m, capi.MQ_FAST, reps=4, iters=20)
    bench(4096, 4096, 1024, capi.MQ_FAST, iters=20)
    bench(4096, 14336, 1024, capi.MQ_FAST, reps=4, iters=20)
if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "decode":
    for (n, k) in ((6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336), (28672, 8192), (8192, 28672)):
        bench(n, k, 16, capi.MQ_FAST, reps=4)
