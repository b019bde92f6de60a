"""Time one prefill K2 launch under MQ_DBG stage bypasses (dev library)."""
import os, subprocess, sys
sys.path.insert(0, "/root/repo")
if len(sys.argv) > 1 and sys.argv[1] == "one":
    import torch
    import paper_2412_14590_b200 as mq
    from paper_2412_14590_b200 import capi
    N, K, M = (int(x) for x in sys.argv[2:5])
    W, A, prom = mq.bench_inputs(M, N, K, 0.1, 1)
    L = mq.partition_and_quantize(W, prom)
    dl = mq.DeviceLayer(L)
    dA = torch.from_numpy(A).cuda()
    Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
    opts = mq.exec_opts(capi.MQ_FAST, 128, pdl=os.environ.get("PDL", "0") == "1")
    ws = dl.quantize_ws(dA, opts)
    for _ in range(5): dl.forward_ws(M, ws, out=Y, opts=opts)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    R = 20
    t0.record()
    for _ in range(R): dl.forward_ws(M, ws, out=Y, opts=opts)
    t1.record(); torch.cuda.synchronize()
    us = t0.elapsed_time(t1) * 1e3 / R
    print(f"dbg={os.environ.get('MQ_DBG','0'):>3s} N={N} K={K} M={M}: {us:8.2f} us  {2*M*N*K/us/1e6:7.1f} TOPS")
    sys.exit(0)
SHAPES = [(14336, 4096, 512), (4096, 4096, 1024)]
DBGS = (0, 128, 129, 135)
if len(sys.argv) > 1 and sys.argv[1] == "floor":
    SHAPES = [(4096, 4096, 16), (28672, 4096, 16)]
    DBGS = (0, 135, 8, 24)
if len(sys.argv) > 1 and sys.argv[1] == "decode":
    SHAPES = [(6144, 4096, 16), (4096, 4096, 16), (28672, 4096, 16), (4096, 14336, 16)]
    DBGS = (0, 1, 4, 5, 7, 135)
for shape in SHAPES:
    for dbg in DBGS:
        env = dict(os.environ, MQ_DBG=str(dbg))
        subprocess.run([sys.executable, __file__, "one", *map(str, shape)], env=env, timeout=120)
