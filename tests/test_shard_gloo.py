"""Multi-process (world_size 2, gloo on CPU) check of the output-feature
column-sharding path's host logic: every rank builds the same
layer, takes its slice of both the 8-bit and the 4-bit partitions from
mq_shard_plan, produces its local output block in gather order, the blocks
are all-gathered, and the colmap permutation restores the original column
order. The result must be BIT-identical to the unsharded output — sharding
never changes per-element arithmetic. (On the GPU the local block comes from
the sharded device layer and the gather is NCCL; here the oracle computes
each rank's block, standing in for the kernel as the checker.)
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as tmp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slice(q, a, b):
    import oracle_py as O
    return O.QTensor(q.bits, q.sym, q.group, b - a, q.cols, q.payload[a:b], q.scales[a:b],
                     None if q.zps is None else q.zps[a:b])


def _worker(rank, world, port, m, n, k, p, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    import torch
    import torch.distributed as dist

    import oracle_py as O
    import paper_2412_14590_b200 as mq

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W, A, prom = mq.bench_inputs(m, n, k, p, 3)
        L = mq.partition_and_quantize(W, prom)
        sc, colmap = mq.shard_plan(L, world)
        OL = O.partition_and_quantize(W, prom)
        codes, scales = O.quantize_acts(A, 128)  # activations replicated: every rank quantizes the same input
        n8, n4 = OL.sub8.rows, OL.sub4.rows
        a8, b8 = n8 * rank // world, n8 * (rank + 1) // world
        a4, b4 = n4 * rank // world, n4 * (rank + 1) // world
        y8 = O.gemm_sub(codes, scales, _slice(OL.sub8, a8, b8)) if b8 > a8 else np.zeros((m, 0), np.float32)
        y4 = O.gemm_sub(codes, scales, _slice(OL.sub4, a4, b4)) if b4 > a4 else np.zeros((m, 0), np.float32)
        local = np.zeros((m, sc), np.float32)  # rank block in gather order, padded to shard_cols
        local[:, : (b8 - a8) + (b4 - a4)] = np.concatenate([y8, y4], axis=1)
        gathered = [torch.zeros((m, sc)) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(local))
        g = torch.stack(gathered).numpy()  # [world, M, shard_cols]
        Y = np.zeros((m, n), np.float32)
        for r in range(world):  # mq_permute_gathered semantics
            valid = colmap[r] >= 0
            Y[:, colmap[r][valid]] = g[r][:, valid]
        ref, _, _ = O.mixed_linear(OL, A)
        q.put((rank, bool(np.array_equal(Y, ref)), O.fnv1a_hex(Y)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n,k,p", [(5, 300, 256, 0.1), (3, 129, 384, 0.5), (2, 64, 128, 0.0)])
def test_column_sharded_gather_is_bit_identical(m, n, k, p):
    world = 2
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, k, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert all(ok for _, ok, _ in res), res
    assert len({h for _, _, h in res}) == 1
