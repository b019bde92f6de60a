import sys, os, time
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle")
import numpy as np, torch
import paper_2412_14590_b200 as mq, oracle_py as O
from paper_2412_14590_b200 import capi
M = int(sys.argv[1]); N = int(sys.argv[2]); K = int(sys.argv[3])
W, A, prom = mq.bench_inputs(M, N, K, 0.1, 9)
L = mq.partition_and_quantize(W, prom)
dl = mq.DeviceLayer(L)
dA = torch.from_numpy(A).cuda()
sub8 = O.QTensor(8, True, 128, L.sub8.rows, L.sub8.cols, L.sub8.payload, L.sub8.scales, None)
sub4 = O.QTensor(4, False, 128, L.sub4.rows, L.sub4.cols, L.sub4.payload, L.sub4.scales, L.sub4.zero_points)
OL = O.Layer(L.out_features, L.in_features, 128, L.index_map8, L.index_map4, sub8, sub4)
ref, rc, rs = O.mixed_linear(OL, A)
for name, o in [("exact tt64", mq.exec_opts(capi.MQ_EXACT, 128, token_tile=64)),
                ("exact tt128", mq.exec_opts(capi.MQ_EXACT, 128, token_tile=128)),
                ("exact tt128 nopdl", mq.exec_opts(capi.MQ_EXACT, 128, token_tile=128, pdl=False)),
                ("fast nosplit tt128", mq.exec_opts(capi.MQ_FAST, 128, token_tile=128, ksplit=1)),
                ("fast split tt64", mq.exec_opts(capi.MQ_FAST, 128, token_tile=64)),
                ("fast split tt128", mq.exec_opts(capi.MQ_FAST, 128, token_tile=128)),
                ("fast split tt32", mq.exec_opts(capi.MQ_FAST, 128, token_tile=32)),
                ]:
    t = time.time()
    Y = dl.forward(dA, opts=o); torch.cuda.synchronize()
    Y = Y.cpu().numpy()
    d = np.abs(Y - ref)
    print(f"{name}: eq={np.array_equal(Y, ref)} rel={d.max()/np.abs(ref).max():.3g} nan={np.isnan(Y).sum()} "
          f"bad_tokens={sorted(set(np.argwhere(d > 1e-3*np.abs(ref).max())[:,0].tolist()))[:8]} {time.time()-t:.2f}s", flush=True)
