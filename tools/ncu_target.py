"""Small fixed workload for ncu captures: one 8B projection at batch M.
usage: python tools/ncu_target.py [N K M mode(fast|exact) act(group|token)]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi

N, K, M = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (14336, 4096, 16)))
mode = capi.MQ_EXACT if len(sys.argv) > 4 and sys.argv[4] == "exact" else capi.MQ_FAST
ag = K if len(sys.argv) > 5 and sys.argv[5] == "token" else 128
W, A, prom = mq.bench_inputs(M, N, K, 0.1, 1)
L = mq.partition_and_quantize(W, prom)
dl = mq.DeviceLayer(L)
dA = torch.from_numpy(A).cuda()
Y = torch.empty((M, N), dtype=torch.float16, device="cuda")
opts = mq.exec_opts(mode, ag, ksplit=int(os.environ.get("KSPLIT", "0")))
for _ in range(5):
    dl.forward(dA, out=Y, opts=opts)
torch.cuda.synchronize()
print("ok", dl.info.tiles8, dl.info.tiles4)
