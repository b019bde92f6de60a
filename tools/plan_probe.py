import sys; sys.path.insert(0, "/root/repo")
import torch, paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi
for (n, k) in ((4096, 4096), (14336, 4096), (28672, 4096), (6144, 4096)):
    W, A, prom = mq.bench_inputs(16, n, k, 0.1, 1)
    dl = mq.DeviceLayer(mq.partition_and_quantize(W, prom))
    print(n, k, dl.info.tiles8, dl.info.tiles4, flush=True)
    dl.forward(torch.from_numpy(A).cuda(), opts=mq.exec_opts(capi.MQ_FAST, 128))
    torch.cuda.synchronize()
