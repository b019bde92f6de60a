import sys, os
sys.path.insert(0, "/root/repo")
import torch
import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi
N, K, M = (int(x) for x in sys.argv[1:4])
W, A, prom = mq.bench_inputs(M, N, K, 0.1, 1)
L = mq.partition_and_quantize(W, prom)
dl = mq.DeviceLayer(L)
dA = torch.from_numpy(A).cuda()
codes, scales = mq.quantize_act(dA, 128)
Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
opts = mq.exec_opts(capi.MQ_FAST, 128)
for _ in range(4): dl.forward_codes(codes, scales, out=Y, opts=opts)
torch.cuda.synchronize()
print("done")
