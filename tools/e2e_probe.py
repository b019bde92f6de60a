"""e2e copy-overlap variants for the bench stack (development aid):
python tools/e2e_probe.py  -> ms per step for: serial 1+1 copies, 2+2 split, per-layer 4+4."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi
SH = [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)]
M = 16
dev = torch.device("cuda", 0)
host = []
for i, (N, K) in enumerate(SH):
    W, A, prom = mq.bench_inputs(1, N, K, 0.1, 1 + i)
    host.append(mq.partition_and_quantize(W, prom))
reps = [[mq.DeviceLayer(L) for L in host] for _ in range(2)]
layers = reps[0]
opts = mq.exec_opts(capi.MQ_FAST, 128)
nx = [M * K for (_, K) in SH]
ny = [M * N for (N, _) in SH]
hx = torch.randn(sum(nx)).pin_memory()
hy = torch.empty(sum(ny), dtype=torch.float16).pin_memory()
dx = torch.empty(sum(nx), device=dev)
dy = torch.empty(sum(ny), dtype=torch.float16, device=dev)
xv = [v.view(M, K) for v, (_, K) in zip(torch.split(dx, nx), SH)]
yv = [v.view(M, N) for v, (N, _) in zip(torch.split(dy, ny), SH)]
s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def groups(n, cuts):  # contiguous element ranges of layer groups
    offs = [0]
    for v in n:
        offs.append(offs[-1] + v)
    return [(offs[a], offs[b]) for a, b in cuts]


def make(in_cuts, out_cuts, rep=0):
    gi = groups(nx, in_cuts)
    go = groups(ny, out_cuts)
    def step():
        main = torch.cuda.current_stream(dev)
        fork = torch.cuda.Event(); fork.record(main)
        s_in.wait_event(fork); s_out.wait_event(fork)
        ready = {}
        with torch.cuda.stream(s_in):
            for (a, b), (lo, hi) in zip(in_cuts, gi):
                dx[lo:hi].copy_(hx[lo:hi], non_blocking=True)
                ev = torch.cuda.Event(); ev.record(s_in)
                for i in range(a, b):
                    ready[i] = ev
        oc = {b - 1: (lo, hi) for (a, b), (lo, hi) in zip(out_cuts, go)}
        for i in range(len(SH)):
            main.wait_event(ready[i])
            reps[rep][i].forward(xv[i], out=yv[i], opts=opts)
            if i in oc:
                lo, hi = oc[i]
                done = torch.cuda.Event(); done.record(main)
                s_out.wait_event(done)
                with torch.cuda.stream(s_out):
                    hy[lo:hi].copy_(dy[lo:hi], non_blocking=True)
        join = torch.cuda.Event(); join.record(s_out); main.wait_event(join)
        join2 = torch.cuda.Event(); join2.record(s_in); main.wait_event(join2)
    return step


def serial():
    dx.copy_(hx, non_blocking=True)
    for i in range(len(SH)):
        layers[i].forward(xv[i], out=yv[i], opts=opts)
    hy.copy_(dy, non_blocking=True)


variants = {
    "serial 1+1": serial,
    "split 2+2 (x0|x1-3, y0-2|y3)": make([(0, 1), (1, 4)], [(0, 3), (3, 4)]),
    "split 2+2 (x0|x1-3, y0-1|y2-3)": make([(0, 1), (1, 4)], [(0, 2), (2, 4)]),
    "split 3+2 (x0|x1|x2-3, y0-2|y3)": make([(0, 1), (1, 2), (2, 4)], [(0, 3), (3, 4)]),
    "per-layer 4+4": make([(i, i + 1) for i in range(4)], [(i, i + 1) for i in range(4)]),
}
variants["per-layer 4+4, 2 replicas"] = [make([(i, i + 1) for i in range(4)], [(i, i + 1) for i in range(4)], r) for r in range(2)]
for name, fn in variants.items():
    fns = fn if isinstance(fn, list) else [fn]
    gs = []
    for f in fns:
        f(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f()
        gs.append(g)
    for k in range(10): gs[k % len(gs)].replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(50): gs[k % len(gs)].replay()
    e1.record(); torch.cuda.synchronize()
    print(f"{name:36s} {e0.elapsed_time(e1) / 50 * 1e3:8.1f} us/step", flush=True)
