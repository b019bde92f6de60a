"""Where the e2e step's time goes (bench.py e2e): host<->device copy rates at the
step's sizes and the overlapped step vs its parts. python tools/e2e_probe.py [M]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
SH = [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)]
dev = torch.device("cuda:0")


def tm(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


nx = [M * K for (_, K) in SH]
ny = [M * N for (N, _) in SH]
hx = torch.randn(sum(nx)).pin_memory()
dx = torch.empty(sum(nx), device=dev)
hy = torch.empty(sum(ny), dtype=torch.float16).pin_memory()
dy = torch.empty(sum(ny), dtype=torch.float16, device=dev)
print(f"M={M}: H2D {hx.numel() * 4 / 1e6:.2f} MB, D2H {hy.numel() * 2 / 1e6:.2f} MB")
us = tm(lambda: dx.copy_(hx, non_blocking=True))
print(f"one H2D copy of all inputs: {us:.1f} us = {hx.numel() * 4 / us / 1e3:.1f} GB/s")
hxs, dxs = list(torch.split(hx, nx)), list(torch.split(dx, nx))
us = tm(lambda: [d.copy_(h, non_blocking=True) for d, h in zip(dxs, hxs)])
print(f"4 H2D copies: {us:.1f} us")
us = tm(lambda: hy.copy_(dy, non_blocking=True))
print(f"one D2H copy of all outputs: {us:.1f} us = {hy.numel() * 2 / us / 1e3:.1f} GB/s")
big = torch.randn(1 << 24).pin_memory()
dbig = torch.empty(1 << 24, device=dev)
us = tm(lambda: dbig.copy_(big, non_blocking=True), 10)
print(f"H2D 64 MB: {us:.1f} us = {big.numel() * 4 / us / 1e3:.1f} GB/s")
s1 = torch.cuda.Stream()
def both():
    with torch.cuda.stream(s1):
        hy.copy_(dy, non_blocking=True)
    dx.copy_(hx, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
us = tm(both)
print(f"H2D + D2H on two streams: {us:.1f} us")

# ---- the bench's e2e step and variants, on the real engine
import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi
layers = []
for i, (N, K) in enumerate(SH):
    W, _, prom = mq.bench_inputs(1, N, K, 0.1, 1 + i)
    layers.append(mq.DeviceLayer.replicas(mq.partition_and_quantize(W, prom), 4))
opts = mq.exec_opts(capi.MQ_FAST, 128)
xv = [d.view(M, K) for d, (_, K) in zip(dxs, SH)]
dys = list(torch.split(dy, ny))
hys = list(torch.split(hy, ny))
yv = [d.view(M, N) for d, (N, _) in zip(dys, SH)]
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
s_in2, s_out2 = torch.cuda.Stream(), torch.cuda.Stream()


def step_e2e2(r, order=(0, 1, 2, 3)):
    """H2D split over two streams (copy engines), D2H over two streams."""
    main = torch.cuda.current_stream()
    fork = torch.cuda.Event()
    fork.record(main)
    for st in (s_in, s_in2, s_out, s_out2):
        st.wait_event(fork)
    ready = [None] * 4
    for k, i in enumerate(order):
        st = (s_in, s_in2)[k % 2]
        with torch.cuda.stream(st):
            dxs[i].copy_(hxs[i], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(st)
            ready[i] = ev
    for i in range(4):
        main.wait_event(ready[i])
        layers[i][r].forward(xv[i], out=yv[i], opts=opts)
        done = torch.cuda.Event()
        done.record(main)
        so = (s_out, s_out2)[i % 2]
        so.wait_event(done)
        with torch.cuda.stream(so):
            hys[i].copy_(dys[i], non_blocking=True)
    for st in (s_out, s_out2, s_in, s_in2):
        j = torch.cuda.Event()
        j.record(st)
        main.wait_event(j)


def step_dev(r):
    for i in range(4):
        layers[i][r].forward(xv[i], out=yv[i], opts=opts)


def step_e2e(r, h2d=True, d2h=True, per_layer=True):
    main = torch.cuda.current_stream()
    fork = torch.cuda.Event()
    fork.record(main)
    s_in.wait_event(fork)
    s_out.wait_event(fork)
    ready = []
    with torch.cuda.stream(s_in):
        if h2d and not per_layer:
            dx.copy_(hx, non_blocking=True)
        for i in range(4):
            if h2d and per_layer:
                dxs[i].copy_(hxs[i], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s_in)
            ready.append(ev)
    for i in range(4):
        main.wait_event(ready[i] if per_layer else ready[-1])
        layers[i][r].forward(xv[i], out=yv[i], opts=opts)
        if d2h and per_layer:
            done = torch.cuda.Event()
            done.record(main)
            s_out.wait_event(done)
            with torch.cuda.stream(s_out):
                hys[i].copy_(dys[i], non_blocking=True)
    if d2h and not per_layer:
        hy.copy_(dy, non_blocking=True)
    for st in (s_out, s_in):
        j = torch.cuda.Event()
        j.record(st)
        main.wait_event(j)


def graphs(fn):
    gs = []
    for r in range(4):
        fn(r)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn(r)
        gs.append(g)
    return gs


def tg(gs, reps=60):
    k = [0]
    def one():
        gs[k[0] % len(gs)].replay()
        k[0] += 1
    return tm(one, reps)


print(f"device-resident step: {tg(graphs(step_dev)):.1f} us")
for name, kw in (("e2e (bench)", {}), ("e2e H2D only", {"d2h": False}), ("e2e D2H only", {"h2d": False}),
                 ("e2e, one H2D + one D2H (no per-layer overlap)", {"per_layer": False})):
    print(f"{name}: {tg(graphs(lambda r, kw=kw: step_e2e(r, **kw))):.1f} us")


def host_view(t):
    """A CUDA-tensor view of pinned host memory (UVA: the device reads it over PCIe)."""
    class _A:
        __cuda_array_interface__ = {"shape": tuple(t.shape), "typestr": "<f4" if t.dtype == torch.float32 else "<f2",
                                    "data": (t.data_ptr(), False), "version": 3, "strides": None}
    return torch.as_tensor(_A(), device=dev)


hxv = [host_view(h).view(M, K) for h, (_, K) in zip(hxs, SH)]
hyv = [host_view(h).view(M, N) for h, (N, _) in zip(hys, SH)]


def step_zc(r, zc_in=(0, 1, 2, 3), kern_out=(3,)):
    """K1 reads the zero-copy inputs straight from pinned host memory; the other
    inputs by copy engine; outputs in kern_out leave through a kernel writing pinned
    host memory, the others by copy engine."""
    main = torch.cuda.current_stream()
    fork = torch.cuda.Event()
    fork.record(main)
    s_in.wait_event(fork)
    s_out.wait_event(fork)
    ready = [None] * 4
    with torch.cuda.stream(s_in):
        for i in range(4):
            if i not in zc_in:
                dxs[i].copy_(hxs[i], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s_in)
                ready[i] = ev
    for i in range(4):
        if ready[i] is not None:
            main.wait_event(ready[i])
        layers[i][r].forward(hxv[i] if i in zc_in else xv[i], out=yv[i], opts=opts)
        if i in kern_out:
            torch.add(yv[i], 0, out=hyv[i])  # a kernel: stores over PCIe
        else:
            done = torch.cuda.Event()
            done.record(main)
            s_out.wait_event(done)
            with torch.cuda.stream(s_out):
                hys[i].copy_(dys[i], non_blocking=True)
    for st in (s_out, s_in):
        j = torch.cuda.Event()
        j.record(st)
        main.wait_event(j)




def step_v(r, zc=(0,), one_h2d=True, one_d2h=True):
    """zero-copy K1 reads for the layers in zc; the other inputs in ONE copy (they
    are contiguous); outputs of layers 0-2 in ONE copy after layer 2; the last
    layer's output through a kernel writing pinned host memory."""
    main = torch.cuda.current_stream()
    fork = torch.cuda.Event()
    fork.record(main)
    s_in.wait_event(fork)
    s_out.wait_event(fork)
    rest = [i for i in range(4) if i not in zc]
    ready = None
    if rest:
        with torch.cuda.stream(s_in):
            a0 = sum(nx[:rest[0]])
            n = sum(nx[i] for i in rest)
            dx[a0:a0 + n].copy_(hx[a0:a0 + n], non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(s_in)
    for i in range(4):
        if i in rest and ready is not None:
            main.wait_event(ready)
            ready = None
        layers[i][r].forward(hxv[i] if i in zc else xv[i], out=yv[i], opts=opts)
        if i == 2:
            done = torch.cuda.Event()
            done.record(main)
            s_out.wait_event(done)
            with torch.cuda.stream(s_out):
                n = sum(ny[:3])
                hy[:n].copy_(dy[:n], non_blocking=True)
        if i == 3:
            torch.add(yv[3], 0, out=hyv[3])
    for st in (s_out, s_in):
        j = torch.cuda.Event()
        j.record(st)
        main.wait_event(j)




def step_d2h(r, which):
    """device-resident inputs; D2H copy-engine transfers of the outputs in `which` only"""
    main = torch.cuda.current_stream()
    fork = torch.cuda.Event()
    fork.record(main)
    s_out.wait_event(fork)
    for i in range(4):
        layers[i][r].forward(xv[i], out=yv[i], opts=opts)
        if i in which:
            done = torch.cuda.Event()
            done.record(main)
            s_out.wait_event(done)
            with torch.cuda.stream(s_out):
                hys[i].copy_(dys[i], non_blocking=True)
    j = torch.cuda.Event()
    j.record(s_out)
    main.wait_event(j)


for w in ((), (3,), (0,), (0, 1, 2), (0, 1, 2, 3)):
    print(f"D2H of outputs {w}: {tg(graphs(lambda r, w=w: step_d2h(r, w))):.1f} us")


def step_out(r, zc_out=(0, 1, 2, 3), h2d=True):
    """bench-style inputs (layer 0 zero-copy, the others by copy engine, or all
    device-resident when h2d is False); the outputs of the layers in zc_out are
    written by K2's epilogue straight into pinned host memory (no copy), the
    others by copy engine (the last one by a copy kernel)."""
    main = torch.cuda.current_stream()
    fork = torch.cuda.Event()
    fork.record(main)
    s_in.wait_event(fork)
    s_out.wait_event(fork)
    ready = [None] * 4
    if h2d:
        with torch.cuda.stream(s_in):
            for i in range(1, 4):
                dxs[i].copy_(hxs[i], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s_in)
                ready[i] = ev
    for i in range(4):
        if ready[i] is not None:
            main.wait_event(ready[i])
        x = hxv[0] if (i == 0 and h2d) else xv[i]
        if i in zc_out:
            layers[i][r].forward(x, out=hyv[i], opts=opts)
            continue
        layers[i][r].forward(x, out=yv[i], opts=opts)
        if i == 3:
            torch.add(yv[i], 0, out=hyv[i])
            continue
        done = torch.cuda.Event()
        done.record(main)
        s_out.wait_event(done)
        with torch.cuda.stream(s_out):
            hys[i].copy_(dys[i], non_blocking=True)
    for st in (s_out, s_in):
        j = torch.cuda.Event()
        j.record(st)
        main.wait_event(j)


for w in ((), (3,), (2, 3), (0, 1, 2, 3)):
    print(f"epilogue-to-host outputs {w}: e2e {tg(graphs(lambda r, w=w: step_out(r, w))):.1f} us, "
          f"device inputs {tg(graphs(lambda r, w=w: step_out(r, w, h2d=False))):.1f} us")
