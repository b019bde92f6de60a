"""GPU tests of the engine's execution options and workspace contract
(include/mixllm/capi.h): one workspace reused across batch sizes and across
layers, the non-spinning (concurrent) joins, the L2 prefetch hint, the
activation scheme's f16 scale storage, and the USAGE errors for what the
sm_100a engine does not take.
"""
import numpy as np
import pytest

import oracle_py as O
import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi

pytestmark = pytest.mark.gpu
TOL = 1e-3


def _layer(n, k, p=0.1, seed=1):
    W, _, prom = mq.bench_inputs(1, n, k, p, seed)
    return mq.partition_and_quantize(W, prom)


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def _ws(dl, ms, opts):
    import torch
    n = max(capi.lib().mq_mixed_linear_workspace_bytes(dl.h, m, capi.C.byref(opts)) for m in ms)
    return torch.zeros(n, dtype=torch.uint8, device="cuda:0")


def test_one_workspace_across_batch_sizes(cuda):
    """FAST launches with different plans (decode split-K, wide-tile barrier
    join, stream-K, unit rounds) share ONE workspace in any order: each leaves
    its arrival counters at zero, so the next never reads stale words."""
    import torch
    L = _layer(4096, 14336)
    dl = mq.DeviceLayer(L)
    o = mq.exec_opts(capi.MQ_FAST, 128)
    seq = [256, 64, 256, 1024, 16, 64, 1, 1024, 96]
    ws = _ws(dl, seq, o)
    rng = np.random.default_rng(3)
    xs = {m: torch.from_numpy(rng.standard_normal((m, 14336)).astype(np.float32)).to(cuda) for m in set(seq)}
    ref = {m: dl.forward(xs[m], opts=o, workspace=_ws(dl, [m], o)).cpu().numpy() for m in set(seq)}
    for m in seq:
        y = dl.forward(xs[m], opts=o, workspace=ws).cpu().numpy()
        assert np.array_equal(y, ref[m]), m
    assert not ws[:32768].any()  # the counter region is zero again


def _rel_err(y, ref):
    return float(np.max(np.abs(y - ref)) / max(np.max(np.abs(ref)), 1e-30))


@pytest.mark.parametrize("tt", [0, 16, 64, 128])
def test_one_quantized_activation_feeds_qkv(cuda, tt):
    """mq_quantize_act_ws once, mq_mixed_linear_ws on q, k and v (different
    tile counts and split plans) from the same workspace. With an explicit
    token tile the split API is bit-identical to the fused forward; with the
    automatic one the fused forward may pick a per-layer tile for a narrow
    layer (auto_token_tile), so FAST results then agree within tolerance."""
    import torch
    layers = [mq.DeviceLayer(_layer(n, 4096, seed=s)) for n, s in ((4096, 2), (1024, 3), (1024, 4))]
    for m in (1, 16, 48, 200):
        o = mq.exec_opts(capi.MQ_FAST, 128, token_tile=tt)
        A = torch.from_numpy(np.random.default_rng(m).standard_normal((m, 4096)).astype(np.float32)).to(cuda)
        n = max(capi.lib().mq_mixed_linear_workspace_bytes(dl.h, m, capi.C.byref(o)) for dl in layers)
        ws = torch.zeros(n, dtype=torch.uint8, device=cuda)
        layers[0].quantize_ws(A, o, workspace=ws)
        for dl in layers:
            y = dl.forward_ws(m, ws, opts=o).cpu().numpy()
            ref = dl.forward(A, opts=o).cpu().numpy()
            if tt:
                assert np.array_equal(y, ref)
            else:
                assert _rel_err(y, ref) <= 1e-5


@pytest.mark.parametrize("m,n,k", [(64, 512, 2048), (96, 640, 2048), (1100, 4096, 1024)])
def test_concurrent_option_same_result(cuda, m, n, k):
    """concurrent=1 avoids every cross-CTA wait (the one-round barrier join
    becomes last-arrival); the slice-order sums are the same bits."""
    import torch
    L = _layer(n, k, seed=7)
    dl = mq.DeviceLayer(L)
    A = torch.from_numpy(np.random.default_rng(5).standard_normal((m, k)).astype(np.float32)).to(cuda)
    y0 = dl.forward(A, opts=mq.exec_opts(capi.MQ_FAST, 128)).cpu().numpy()
    y1 = dl.forward(A, opts=mq.exec_opts(capi.MQ_FAST, 128, concurrent=True)).cpu().numpy()
    assert np.array_equal(y0, y1)


def test_concurrent_launches_on_two_streams(cuda):
    """Two FAST launches with concurrent=1 on two streams at once (each a
    persistent grid of one CTA per SM) complete and match the serial result."""
    import torch
    a, b = mq.DeviceLayer(_layer(640, 2048, seed=8)), mq.DeviceLayer(_layer(4096, 1024, seed=9))
    xa = torch.from_numpy(np.random.default_rng(1).standard_normal((96, 2048)).astype(np.float32)).to(cuda)
    xb = torch.from_numpy(np.random.default_rng(2).standard_normal((1100, 1024)).astype(np.float32)).to(cuda)
    o = mq.exec_opts(capi.MQ_FAST, 128, concurrent=True)
    ra, rb = a.forward(xa, opts=o).cpu().numpy(), b.forward(xb, opts=o).cpu().numpy()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    wa, wb = a.workspace(96, o), b.workspace(1100, o)
    ya = torch.empty((96, 640), device=cuda)
    yb = torch.empty((1100, 4096), device=cuda)
    torch.cuda.synchronize()
    for _ in range(20):
        a.forward(xa, out=ya, opts=o, stream=s1, workspace=wa)
        b.forward(xb, out=yb, opts=o, stream=s2, workspace=wb)
    torch.cuda.synchronize()
    assert np.array_equal(ya.cpu().numpy(), ra) and np.array_equal(yb.cpu().numpy(), rb)


@pytest.mark.parametrize("m", [1, 16, 512])
def test_prefetch_next_layer_same_result(cuda, m):
    """The L2 prefetch hint changes no result (it only warms L2)."""
    import torch
    cur, nxt = mq.DeviceLayer(_layer(4096, 4096, seed=10)), mq.DeviceLayer(_layer(6144, 4096, seed=11))
    A = torch.from_numpy(np.random.default_rng(m).standard_normal((m, 4096)).astype(np.float32)).to(cuda)
    y0 = cur.forward(A, opts=mq.exec_opts(capi.MQ_FAST, 128)).cpu().numpy()
    for pb in (0, 1 << 20):
        y1 = cur.forward(A, opts=mq.exec_opts(capi.MQ_FAST, 128, prefetch_next=nxt, prefetch_bytes=pb)).cpu().numpy()
        assert np.array_equal(y0, y1)
    y2 = cur.forward(A, opts=mq.exec_opts(capi.MQ_EXACT, 128, prefetch_next=nxt)).cpu().numpy()
    assert np.array_equal(y2, cur.forward(A, opts=mq.exec_opts(capi.MQ_EXACT, 128)).cpu().numpy())


def test_act_scale_f16_matches_reference(cuda, golden):
    """scale_f16_storage on the activation scheme (quant.hpp:70-76,
    quant.cpp:81-86): codes, scales and the exact output equal the reference's
    own (golden act_f16, generated by oracle/_ref)."""
    import torch
    c = golden["act_f16"]
    W, A, prom = mq.bench_inputs(c["m"], c["n"], c["k"], c["percent"], 1)
    L = mq.partition_and_quantize(W, prom)
    dA = torch.from_numpy(A).to(cuda)
    codes, scales = mq.quantize_act(dA, 128, scale_f16=True)
    assert mq.fnv1a_hex(codes.cpu().numpy()[:, :c["k"]]) == c["act_codes"]
    assert mq.fnv1a_hex(np.ascontiguousarray(scales.cpu().numpy()[:, :c["m"]].T)) == c["act_scales"]
    dl = mq.DeviceLayer(L)
    Y = dl.forward(dA, opts=mq.exec_opts(capi.MQ_EXACT, 128, act_scale_f16=True)).cpu().numpy()
    assert mq.fnv1a_hex(Y) == c["out_f32"]
    Yd = mq.execute_mixed_linear(A, L, act_scheme=mq.QuantScheme(8, True, 128, True))
    assert mq.fnv1a_hex(Yd) == c["out_f32"]
    # fast mode and the per-token variant through the same flag, vs the oracle
    Yf = dl.forward(dA, opts=mq.exec_opts(capi.MQ_FAST, 128, act_scale_f16=True)).cpu().numpy()
    assert _rel(Yf, Y) <= TOL


def test_per_token_k_limit_is_a_usage_error(cuda):
    L = _layer(256, 40960)
    dl = mq.DeviceLayer(L)
    import torch
    A = torch.zeros((2, 40960), device=cuda)
    with pytest.raises(mq.UsageError, match="per-token"):
        dl.forward(A, opts=mq.exec_opts(capi.MQ_FAST, 40960))
    dl.forward(A, opts=mq.exec_opts(capi.MQ_FAST, 128))  # group-wise still runs


@pytest.mark.parametrize("g", [32, 64])
def test_group_below_128_is_a_usage_error(cuda, g):
    """The reference accepts groups in [1, 128] (gemm.cpp:21-23); the sm_100a
    engine's tiles use group 128 (a kind::i8 MMA is K = 32 and a K-group is
    four of them): smaller groups are rejected before any device work."""
    W, _, prom = mq.bench_inputs(1, 256, 512, 0.1, 1)
    L = mq.partition_and_quantize(W, prom, mq.QuantScheme(8, True, g), mq.QuantScheme(4, False, g))
    with pytest.raises(mq.UsageError, match="group size"):
        mq.DeviceLayer(L)
