"""Column-sharded layers on the device, on one B200:

* every rank's shard is a real DeviceLayer(rank, world); their blocks gathered
  in rank order and permuted by the product's mq_permute_gathered are
  BIT-identical to the unsharded layer in exact mode (f32 / bf16 outputs) —
  sharding never changes the reference op order per element — and within the
  north_star tolerance in fast mode (a shard's own tiles split K differently);
* the engine's own NCCL path (mq_mixed_linear_allgather through the run-time
  NCCL binding) on a one-rank communicator equals mq_mixed_linear;
* the fused gather epilogue (mq_mixed_linear_peers) writes every shard's
  outputs into all ranks' full Y at the original columns: each Y equals the
  unsharded output; mq_peer_barrier completes across ranks on two streams;
* two processes sharing the GPU (gloo all_gather of CUDA tensors) run the
  sharded product path end to end and match the unsharded output bit for bit.
(NCCL refuses two ranks on one device, so NCCL with world > 1 needs the 8-GPU
box; bench.py --gpus N runs it.)
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as tmp

import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi

pytestmark = pytest.mark.gpu


def _same(y, ref, mode):
    """EXACT mode: bit-identical (the reference op order per element does not
    depend on the sharding). FAST mode: a shard has its own tiles, so its K
    splits and per-unit chunk rotation differ — within the north_star tolerance."""
    import torch
    if mode == capi.MQ_EXACT:
        assert torch.equal(y, ref)
    else:
        a, b = y.float(), ref.float()
        assert bool(torch.isfinite(a).all())
        assert float((a - b).abs().max() / b.abs().max()) <= 1e-3


def _layer(m, n, k, p=0.1, seed=3):
    W, A, prom = mq.bench_inputs(m, n, k, p, seed)
    return mq.partition_and_quantize(W, prom), A


@pytest.mark.parametrize("world,m,n,k,mode,dt", [(2, 16, 1024, 1024, capi.MQ_EXACT, "float32"),
                                                 (3, 16, 1000, 640, capi.MQ_FAST, "float16"),
                                                 (8, 5, 4096, 1024, capi.MQ_FAST, "float32"),
                                                 (4, 200, 2048, 512, capi.MQ_EXACT, "bfloat16")])
def test_sharded_layers_gather_bit_identical(cuda, world, m, n, k, mode, dt):
    import torch
    L, A = _layer(m, n, k)
    dA = torch.from_numpy(A).to(cuda)
    o = mq.exec_opts(mode, 128)
    dtype = getattr(torch, dt)
    ref = mq.DeviceLayer(L).forward(dA, out_dtype=dtype, opts=o)
    shards = [mq.DeviceLayer(L, rank=r, world=world) for r in range(world)]
    sc = shards[0].out_cols
    gathered = torch.stack([s.forward(dA, out_dtype=dtype, opts=o) for s in shards])  # [world, M, sc]
    cm = torch.from_numpy(shards[0].shard_colmap()).to(cuda)
    Y = mq.permute_gathered(gathered, cm, world, sc, m, n)
    _same(Y, ref, mode)


def test_allgather_nccl_one_rank(cuda):
    """The engine's NCCL path (dlopen'd NCCL, ncclAllGather on the caller's
    communicator) on a one-rank communicator equals the plain forward."""
    import torch
    L, A = _layer(16, 2048, 1024)
    dA = torch.from_numpy(A).to(cuda)
    dl = mq.DeviceLayer(L)
    comm = mq.NcclComm.create(mq.NcclComm.unique_id(), 1, 0, 0)
    o = mq.exec_opts(capi.MQ_EXACT, 128)
    Y = dl.forward_allgather(dA, comm, opts=o)
    assert torch.equal(Y, dl.forward(dA, opts=o))
    # a communicator whose size does not match the shard is a usage error
    with pytest.raises(capi.UsageError):
        mq.DeviceLayer(L, rank=0, world=2).forward_allgather(dA, comm, opts=o)


@pytest.mark.parametrize("world,m,mode", [(2, 16, capi.MQ_EXACT), (4, 64, capi.MQ_FAST), (3, 1, capi.MQ_FAST),
                                          (8, 130, capi.MQ_EXACT)])
def test_fused_peer_gather(cuda, world, m, mode):
    import torch
    L, A = _layer(m, 3000, 1024, seed=5)
    dA = torch.from_numpy(A).to(cuda)
    o = mq.exec_opts(mode, 128)
    ref = mq.DeviceLayer(L).forward(dA, opts=o)
    ys = [torch.full((m, L.out_features), float("nan"), device=cuda) for _ in range(world)]
    for r in range(world):  # each rank lists the outputs starting with its own
        mq.DeviceLayer(L, rank=r, world=world).forward_peers(dA, ys[r:] + ys[:r], opts=o)
    for y in ys:
        _same(y, ref, mode)


def test_peer_barrier_two_streams(cuda):
    """Two ranks (one stream each) meet at mq_peer_barrier; epochs advance."""
    import torch
    flags = [torch.zeros(2, dtype=torch.int32, device=cuda) for _ in range(2)]
    s = [torch.cuda.Stream(), torch.cuda.Stream()]
    for epoch in (1, 2, 3):
        for r in range(2):
            with torch.cuda.stream(s[r]):
                mq.peer_barrier(flags, 2, r, epoch, stream=s[r])
        torch.cuda.synchronize()
        assert all(int(f.min()) == epoch for f in flags)


def _free_port() -> int:
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    p = so.getsockname()[1]
    so.close()
    return p


def _gloo_worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist

    import paper_2412_14590_b200 as mqw
    from paper_2412_14590_b200 import capi as cw

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W, A, prom = mqw.bench_inputs(16, 2048, 1024, 0.1, 7)
        L = mqw.partition_and_quantize(W, prom)
        dA = torch.from_numpy(A).cuda()
        o = mqw.exec_opts(cw.MQ_EXACT, 128)
        sh = mqw.DeviceLayer(L, rank=rank, world=world)
        local = sh.forward(dA, opts=o)
        gathered = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(gathered, local)
        cm = torch.from_numpy(sh.shard_colmap()).cuda()
        Y = mqw.permute_gathered(torch.stack(gathered), cm, world, sh.out_cols, 16, 2048)
        ref = mqw.DeviceLayer(L).forward(dA, opts=o)
        q.put((rank, bool(torch.equal(Y, ref))))
    except Exception as e:  # report, do not hang the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_processes_gloo_product_path(cuda):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res
