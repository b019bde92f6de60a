"""Device time of the bench stack (K1 + K2 per projection, CUDA graph, PDL), the
bench's `value` step without the harness: python tools/stack_time.py [M ...]
env PF=<MB>: each projection prefetches the next one's weights into L2 (0 = auto
size, unset = off); REPS: weight replicas rotated between steps (default 3);
K2ONLY=1: activations quantized once outside the graph (the K2 launches alone,
chained as in the stack: the K1 share of the step is the difference)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi

SH = [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)]
R = int(os.environ.get("REPS", "3"))
reps = []
for r in range(R):
    layers = []
    for i, (N, K) in enumerate(SH):
        W, _, prom = mq.bench_inputs(1, N, K, 0.1, 1 + i)
        layers.append(mq.DeviceLayer(mq.partition_and_quantize(W, prom)))
    reps.append(layers)
pf = os.environ.get("PF")
for M in [int(a) for a in sys.argv[1:]] or [16]:
    xs = [torch.randn((M, K), device="cuda") for (_, K) in SH]
    ys = [torch.empty((M, N), dtype=torch.float16, device="cuda") for (N, _) in SH]
    gs = []
    for r in range(R):
        nxt = [reps[r][i + 1] for i in range(3)] + [reps[(r + 1) % R][0]]
        opts = [mq.exec_opts(capi.MQ_FAST, 128, prefetch_next=nxt[i] if pf is not None else None,
                             prefetch_bytes=int(float(pf) * 2**20) if pf else 0) for i in range(4)]
        k2only = os.environ.get("K2ONLY") is not None
        wss = [reps[r][i].quantize_ws(xs[i], opts[i]) for i in range(4)] if k2only else None

        def step():
            for i in range(4):
                if k2only:
                    reps[r][i].forward_ws(M, wss[i], out=ys[i], opts=opts[i])
                else:
                    reps[r][i].forward(xs[i], out=ys[i], opts=opts[i])
        step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        gs.append(g)
    for k in range(20):
        gs[k % R].replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(120):
        gs[k % R].replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"M={M} PF={pf}: {e0.elapsed_time(e1) * 1e3 / 120:.2f} us per stack step", flush=True)
