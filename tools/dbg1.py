import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle")
import numpy as np, torch
import paper_2412_14590_b200 as mq, oracle_py as O
from paper_2412_14590_b200 import capi
for (m, n, k) in [(16, 512, 512), (16, 512, 4096)]:
    W, A, prom = mq.bench_inputs(m, n, k, 0.1, 1)
    L = mq.partition_and_quantize(W, prom)
    dl = mq.DeviceLayer(L)
    dA = torch.from_numpy(A).cuda()
    sub4 = O.QTensor(4, False, 128, L.sub4.rows, L.sub4.cols, L.sub4.payload, L.sub4.scales, L.sub4.zero_points)
    codes, scales = mq.quantize_act(dA, 128)
    rc, rs = O.quantize_acts(A, 128)
    p = dl.partials(codes, 1).cpu().numpy()
    r = O.group_partials(rc, sub4)
    bad = (p != r)
    print(m, n, k, "sub4 partial mismatches", bad.sum(), "of", bad.size)
    print(" per group", bad.sum(axis=(1, 2)).tolist())
    print(" per row-tile", [int(bad[:, :, t*128:(t+1)*128].sum()) for t in range((L.sub4.rows + 127)//128)])
    print(" per token", bad.sum(axis=(0, 2)).tolist())
    i = np.argwhere(bad)[:3]
    for g, mm, rr in i: print("  ", g, mm, rr, p[g, mm, rr], r[g, mm, rr])
    Y = dl.forward_codes(codes, scales, opts=mq.exec_opts(capi.MQ_EXACT, 128)).cpu().numpy()
    print(" Y sub8 cols nan", np.isnan(Y[:, L.index_map8]).sum(), "sub4 cols nan", np.isnan(Y[:, L.index_map4]).sum(),
          "sub8 max", np.abs(Y[:, L.index_map8]).max())
