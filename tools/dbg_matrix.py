"""Isolation matrix for K2 failures: each config in its own subprocess.
usage: python tools/dbg_matrix.py            (runs the matrix)
       python tools/dbg_matrix.py one M N K P MODE AG TT  (one config)"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))


def one(M, N, K, P, mode, ag, tt):
    import numpy as np
    import torch
    import oracle_py as O
    import paper_2412_14590_b200 as mq
    from paper_2412_14590_b200 import capi
    W, A, prom = mq.bench_inputs(M, N, K, P, 1)
    L = mq.partition_and_quantize(W, prom)
    dl = mq.DeviceLayer(L)
    o = mq.exec_opts(capi.MQ_EXACT if mode == "exact" else capi.MQ_FAST, ag, token_tile=tt)
    Y = dl.forward(torch.from_numpy(A).cuda(), opts=o)
    torch.cuda.synchronize()
    y = Y.cpu().numpy()
    sub8 = O.QTensor(8, True, 128, L.sub8.rows, L.sub8.cols, L.sub8.payload, L.sub8.scales, None)
    sub4 = O.QTensor(4, False, 128, L.sub4.rows, L.sub4.cols, L.sub4.payload, L.sub4.scales, L.sub4.zero_points)
    ref, _, _ = O.mixed_linear(O.Layer(N, K, 128, L.index_map8, L.index_map4, sub8, sub4), A,
                               act_group=None if ag == 128 else ag)
    rel = float(np.abs(y - ref).max() / np.abs(ref).max())
    print(f"rel={rel:.3g} exact={np.array_equal(y, ref)}")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        a = sys.argv[2:]
        one(int(a[0]), int(a[1]), int(a[2]), float(a[3]), a[4], int(a[5]), int(a[6]))
        sys.exit(0)
    cfgs = []
    for mode in ("exact", "fast"):
        for (M, N, K, P) in [(16, 512, 256, 0.0), (16, 512, 256, 1.0), (16, 512, 256, 0.1), (16, 4096, 4096, 0.1)]:
            for tt in (16, 32, 64, 128):
                cfgs.append((M, N, K, P, mode, 128, tt))
    for c in cfgs:
        r = subprocess.run([sys.executable, __file__, "one", *map(str, c)], capture_output=True, text=True, timeout=120)
        tail = (r.stdout.strip().splitlines() or [""])[-1] if r.returncode == 0 else \
            [l for l in r.stderr.splitlines() if "Error" in l or "error" in l][-1:]
        print(c, "rc", r.returncode, tail, flush=True)
