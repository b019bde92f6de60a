"""GPU parity: the sm_100a engine (through the C ABI) against the oracle and
the reference's golden checksums (tests/golden/golden.json, generated from the
reference's own code by tests/golden/make_golden.py).

Bars (north_star): bit-exact for activation codes/scales and int32 group
partial sums; bit-exact f32 output in MQ_EXACT mode (reference op order);
MQ_FAST / per-token within max|gpu - ref| <= 1e-3 * max|ref|.
"""
import numpy as np
import pytest

import oracle_py as O
import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi

pytestmark = pytest.mark.gpu
TOL = 1e-3  # north_star: fp32-relative tolerance for rescaled outputs


def _layer(m, n, k, p, seed=1):
    W, A, prom = mq.bench_inputs(m, n, k, p, seed)
    return mq.partition_and_quantize(W, prom), A


def _oracle_layer(L):
    """The same quantized layer in the oracle's structures."""
    sub8 = O.QTensor(8, True, 128, L.sub8.rows, L.sub8.cols, L.sub8.payload, L.sub8.scales, None)
    sub4 = O.QTensor(4, False, 128, L.sub4.rows, L.sub4.cols, L.sub4.payload, L.sub4.scales, L.sub4.zero_points)
    return O.Layer(L.out_features, L.in_features, 128, L.index_map8, L.index_map4, sub8, sub4)


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


# ------------------------------------------------------------------ K1
@pytest.mark.parametrize("m,k", [(1, 4096), (16, 4096), (17, 384), (5, 200), (64, 512)])
def test_act_quant_groupwise_bit_exact(cuda, m, k):
    import torch
    _, A, _ = mq.bench_inputs(m, 8, k, 0.0, 7)
    codes, scales = mq.quantize_act(torch.from_numpy(A).to(cuda), 128)
    rc, rs = O.quantize_acts(A, 128)
    assert np.array_equal(codes.cpu().numpy()[:, :k], rc)
    assert np.array_equal(scales.cpu().numpy()[:, :m].T, rs)  # group-major on device
    assert not codes.cpu().numpy()[:, k:].any()  # padded columns zeroed


@pytest.mark.parametrize("m,k", [(1, 4096), (16, 4096), (3, 300)])
def test_act_quant_per_token_bit_exact(cuda, m, k):
    import torch
    _, A, _ = mq.bench_inputs(m, 8, k, 0.0, 11)
    codes, scales = mq.quantize_act(torch.from_numpy(A).to(cuda), k)
    rc, rs = O.quantize_acts(A, k)
    assert np.array_equal(codes.cpu().numpy()[:, :k], rc)
    assert np.array_equal(scales.cpu().numpy()[0, :m], rs.reshape(-1))


def test_act_quant_edge_values(cuda):
    import torch
    A = np.zeros((4, 256), np.float32)
    A[1, :128] = 5.0                     # constant group
    A[2, 3] = 1e-30                      # tiny amax: scale falls back to 1e-8
    A[3] = np.linspace(-2.5, 2.5, 256)   # exact .5 ties after division
    codes, scales = mq.quantize_act(torch.from_numpy(A).to(cuda), 128)
    rc, rs = O.quantize_acts(A, 128)
    assert np.array_equal(codes.cpu().numpy()[:, :256], rc)
    assert np.array_equal(scales.cpu().numpy()[:, :4].T, rs)


def test_act_quant_nonfinite_flag(cuda):
    import torch
    A = np.ones((3, 256), np.float32)
    A[2, 200] = np.nan
    err = torch.full((1,), 2**31 - 1, dtype=torch.int32, device=cuda)
    mq.quantize_act(torch.from_numpy(A).to(cuda), 128, err=err)
    assert int(err.item()) == 2 * 2 + 1  # row 2, group 1 (quant.hpp:56-64 DataError location)


# ------------------------------------------------------ K2 exact mode
@pytest.mark.parametrize("idx", range(9))
def test_exact_mode_matches_reference_checksum(cuda, golden, idx):
    import torch
    c = golden["cases"][idx]
    L, A = _layer(c["m"], c["n"], c["k"], c["percent"])
    dl = mq.DeviceLayer(L)
    Y = dl.forward(torch.from_numpy(A).to(cuda), opts=mq.exec_opts(capi.MQ_EXACT, 128))
    torch.cuda.synchronize()
    y = Y.cpu().numpy()
    if mq.fnv1a_hex(y) != c["out_f32"]:
        ref, _, _ = O.mixed_linear(_oracle_layer(L), A)
        bad = np.argwhere(y != ref)
        pytest.fail(f"checksum mismatch: {len(bad)} elements differ, first {bad[:4].tolist()}, rel {_rel(y, ref):.3g}")


def test_exact_mode_simt_debug_kernel_agrees(cuda, golden):
    import torch
    c = golden["cases"][6]
    L, A = _layer(c["m"], c["n"], c["k"], c["percent"])
    dl = mq.DeviceLayer(L)
    Y = dl.forward(torch.from_numpy(A).to(cuda), opts=mq.exec_opts(capi.MQ_EXACT, 128, gemm_impl=1))
    assert mq.fnv1a_hex(Y.cpu().numpy()) == c["out_f32"]


@pytest.mark.parametrize("m,n,k,p", [(16, 4096, 4096, 0.1), (7, 300, 384, 0.3), (40, 1024, 1024, 1.0)])
def test_w8_signed_mode_matches_spec_oracle(cuda, m, n, k, p):
    import torch
    L, A = _layer(m, n, k, p, seed=3)
    dl = mq.DeviceLayer(L, w8_mode=capi.MQ_W8_SIGNED)
    Y = dl.forward(torch.from_numpy(A).to(cuda), opts=mq.exec_opts(capi.MQ_EXACT, 128)).cpu().numpy()
    ref, _, _ = O.mixed_linear(_oracle_layer(L), A, w8_unsigned=False)
    assert np.array_equal(Y, ref)


# --------------------------------------------------- int32 partial sums
@pytest.mark.parametrize("which", [0, 1])
@pytest.mark.parametrize("m,n,k,p", [(16, 1024, 1024, 0.2), (3, 300, 200, 0.5)])
def test_group_partials_bit_exact(cuda, which, m, n, k, p):
    import torch
    L, A = _layer(m, n, k, p, seed=5)
    dl = mq.DeviceLayer(L)
    codes, _ = mq.quantize_act(torch.from_numpy(A).to(cuda), 128)
    part = dl.partials(codes, which).cpu().numpy()
    rc, _ = O.quantize_acts(A, 128)
    ol = _oracle_layer(L)
    ref = O.group_partials(rc, ol.sub8 if which == 0 else ol.sub4)
    assert np.array_equal(part, ref)


# ----------------------------------------------------------- fast mode
@pytest.mark.parametrize("m", [1, 16, 33, 64, 130, 512])
def test_fast_mode_within_tolerance(cuda, m):
    import torch
    L, A = _layer(m, 4096, 4096, 0.1, seed=9)
    dl = mq.DeviceLayer(L)
    Y = dl.forward(torch.from_numpy(A).to(cuda), opts=mq.exec_opts(capi.MQ_FAST, 128)).cpu().numpy()
    ref, _, _ = O.mixed_linear(_oracle_layer(L), A)
    assert _rel(Y, ref) <= TOL


@pytest.mark.parametrize("m,n,k", [(64, 512, 2048), (96, 640, 2048), (128, 1024, 1536)])
def test_fast_mode_wide_tile_k_split(cuda, m, n, k):
    """One wide token tile (BN 64/128) on a narrow layer: the K-split join of
    the 64/128-token partials (split_join_wide), within tolerance and
    bit-reproducible run to run."""
    import torch
    L, A = _layer(m, n, k, 0.1, seed=31)
    dl = mq.DeviceLayer(L)
    o = mq.exec_opts(capi.MQ_FAST, 128)
    dA = torch.from_numpy(A).to(cuda)
    Y = dl.forward(dA, opts=o).cpu().numpy()
    ref, _, _ = O.mixed_linear(_oracle_layer(L), A)
    assert _rel(Y, ref) <= TOL
    for ks in (2, 4):  # explicit splits through the same join
        assert _rel(dl.forward(dA, opts=mq.exec_opts(capi.MQ_FAST, 128, ksplit=ks)).cpu().numpy(), ref) <= TOL
    for _ in range(2):
        assert np.array_equal(dl.forward(dA, opts=o).cpu().numpy(), Y)


@pytest.mark.parametrize("m,tt,sched", [(576, 64, 2), (1100, 128, 2), (1100, 128, 1), (1100, 128, 0)])
def test_fast_mode_stream_k(cuda, m, tt, sched):
    """Stream-K schedule (cut items summed head + tail) vs unit rounds: both
    within tolerance of the oracle, and bit-reproducible run to run."""
    import torch
    L, A = _layer(m, 4096, 1024, 0.1, seed=21)
    dl = mq.DeviceLayer(L)
    o = mq.exec_opts(capi.MQ_FAST, 128, token_tile=tt, schedule=sched)
    dA = torch.from_numpy(A).to(cuda)
    Y = dl.forward(dA, opts=o).cpu().numpy()
    ref, _, _ = O.mixed_linear(_oracle_layer(L), A)
    assert _rel(Y, ref) <= TOL
    for _ in range(2):
        assert np.array_equal(dl.forward(dA, opts=o).cpu().numpy(), Y)


@pytest.mark.parametrize("m", [1, 16, 100])
def test_per_token_fast_mode_within_tolerance(cuda, m):
    import torch
    L, A = _layer(m, 2048, 4096, 0.1, seed=13)
    dl = mq.DeviceLayer(L)
    Y = dl.forward(torch.from_numpy(A).to(cuda), opts=mq.exec_opts(capi.MQ_FAST, 4096)).cpu().numpy()
    ref, _, _ = O.mixed_linear(_oracle_layer(L), A, act_group=4096)
    assert _rel(Y, ref) <= TOL


def test_per_token_exact_mode_bit_exact(cuda):
    import torch
    L, A = _layer(16, 1024, 2048, 0.1, seed=17)
    dl = mq.DeviceLayer(L)
    Y = dl.forward(torch.from_numpy(A).to(cuda), opts=mq.exec_opts(capi.MQ_EXACT, 2048)).cpu().numpy()
    ref, _, _ = O.mixed_linear(_oracle_layer(L), A, act_group=2048)
    assert np.array_equal(Y, ref)


@pytest.mark.parametrize("dt", ["float16", "bfloat16"])
def test_half_outputs(cuda, dt):
    import torch
    L, A = _layer(16, 1024, 1024, 0.1, seed=21)
    dl = mq.DeviceLayer(L)
    Y = dl.forward(torch.from_numpy(A).to(cuda), out_dtype=getattr(torch, dt),
                   opts=mq.exec_opts(capi.MQ_EXACT, 128)).float().cpu().numpy()
    ref, _, _ = O.mixed_linear(_oracle_layer(L), A)
    expect = torch.from_numpy(ref).to(getattr(torch, dt)).float().numpy()
    assert np.array_equal(Y, expect)  # exact f32 result rounded once to the output type


def test_fast_mode_deterministic(cuda):
    import torch
    L, A = _layer(16, 4096, 4096, 0.1, seed=23)
    dl = mq.DeviceLayer(L)
    dA = torch.from_numpy(A).to(cuda)
    o = mq.exec_opts(capi.MQ_FAST, 128)
    y1 = dl.forward(dA, opts=o).cpu().numpy()
    for _ in range(3):
        assert np.array_equal(dl.forward(dA, opts=o).cpu().numpy(), y1)


def test_half_inputs(cuda):
    import torch
    L, A = _layer(16, 512, 1024, 0.1, seed=29)
    A16 = torch.from_numpy(A).half()
    dl = mq.DeviceLayer(L)
    Y = dl.forward(A16.to(cuda), opts=mq.exec_opts(capi.MQ_EXACT, 128)).cpu().numpy()
    ref, _, _ = O.mixed_linear(_oracle_layer(L), A16.float().numpy())
    assert np.array_equal(Y, ref)


def test_drop_in_execute_mixed_linear_c1(cuda, golden):
    c = golden["cases"][0]
    W, A, prom = mq.bench_inputs(c["m"], c["n"], c["k"], c["percent"])
    L = mq.partition_and_quantize(W, prom)
    Y = mq.execute_mixed_linear(A, L)
    assert mq.fnv1a_hex(Y) == c["out_f32"] == "5bb508ecbf3b895f"


def test_drop_in_nonfinite_raises_data_error(cuda):
    W, A, prom = mq.bench_inputs(2, 256, 256, 0.1)
    A[1, 130] = np.inf
    L = mq.partition_and_quantize(W, prom)
    with pytest.raises(mq.DataError, match="row 1, group 1"):
        mq.execute_mixed_linear(A, L)


def test_run_bench_checksum(cuda, golden):
    c = golden["cases"][0]
    r = mq.run_bench(c["m"], c["n"], c["k"], c["percent"], repeats=2)
    assert r["checksum"] == c["out_f32"]


def test_cpp_dropin_binary(cuda):
    """The reference's C++ call shapes (run_bench, execute_mixed_linear,
    execute_mixed_on_codes, a quantized_forward-style chain) compiled against
    include/mixllm/mixquant.hpp: golden checksums, errors before compute."""
    import os
    import subprocess
    from paper_2412_14590_b200 import _build
    assert os.path.exists(_build.TEST_BIN), "tests/cpp/_bin/test_dropin not built (run __graft_entry__.build())"
    r = subprocess.run([_build.TEST_BIN, "--gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_quantized_model_device_layers(cuda):
    """quantized.json written by the reference -> DeviceLayers -> MQ_EXACT forward
    bit-identical to the oracle on the loaded layers."""
    import os
    import torch
    fx = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "quantized_v1")
    layers = mq.load_device_layers(fx)
    assert sorted(layers) == ["blk0.proj", "blk0.pure4"]
    for name, dl in layers.items():
        L = dl.layer
        A = np.random.default_rng(7).standard_normal((9, L.in_features)).astype(np.float32)
        Y = dl.forward(torch.from_numpy(A).to(cuda), opts=mq.exec_opts(capi.MQ_EXACT, 128)).cpu().numpy()
        ref, _, _ = O.mixed_linear(_oracle_layer(L), A)
        assert np.array_equal(Y, ref), name


def test_bench_json_contract(cuda):
    """bench.py prints one JSON line with the keys the driver and the judge read."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--steps", "3", "--warmup", "3",
                          "--no-sweep", "--no-cpu"], capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] <= 1.5 and r["peak"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] == 3 * 8
    assert "workload" in d["config"]


@pytest.mark.parametrize("m,n,k,tt,sched,ag", [(1100, 4096, 1024, 128, 2, 1024), (96, 640, 2048, 0, 0, 2048),
                                               (300, 1024, 1000, 128, 2, 128)])
def test_fast_mode_split_paths_per_token_and_ragged(cuda, m, n, k, tt, sched, ag):
    """Per-token activations (s_a applied after the K join) through stream-K and
    the wide-tile K-split, and a ragged last K-group through stream-K."""
    import torch
    L, A = _layer(m, n, k, 0.1, seed=41)
    dl = mq.DeviceLayer(L)
    o = mq.exec_opts(capi.MQ_FAST, ag, token_tile=tt, schedule=sched)
    Y = dl.forward(torch.from_numpy(A).to(cuda), opts=o).cpu().numpy()
    ref, _, _ = O.mixed_linear(_oracle_layer(L), A, act_group=None if ag == 128 else ag)
    assert _rel(Y, ref) <= TOL


def test_bf16_output_wide_split(cuda):
    """bf16 output through the wide-tile K-split join equals the f32 result rounded once."""
    import torch
    L, A = _layer(96, 640, 2048, 0.1, seed=43)
    dl = mq.DeviceLayer(L)
    dA = torch.from_numpy(A).to(cuda)
    o = mq.exec_opts(capi.MQ_FAST, 128)
    y32 = dl.forward(dA, opts=o).cpu()
    y16 = dl.forward(dA, opts=o, out_dtype=torch.bfloat16).cpu()
    assert torch.equal(y16.float(), y32.to(torch.bfloat16).float())


@pytest.mark.parametrize("m,n,k,sched,ag", [(16, 4096, 4096, 2, 128), (1, 4096, 4096, 2, 128), (16, 28672, 4096, 0, 128),
                                            (32, 6144, 4096, 2, 128), (16, 4096, 14336, 2, 128),
                                            (16, 4096, 4096, 2, 4096), (7, 640, 1000, 2, 128)])
def test_fast_mode_decode_stream_k(cuda, m, n, k, sched, ag):
    """Decode stream-K (token tiles <= 32): equal bytes per CTA, items cut into
    any number of pieces on consecutive CTAs and joined by the last piece in
    CTA order — within tolerance, bit-reproducible, and equal to the unit
    schedule within tolerance. Covers per-token scales and a ragged K-group."""
    import torch
    L, A = _layer(m, n, k, 0.1, seed=47)
    dl = mq.DeviceLayer(L)
    dA = torch.from_numpy(A).to(cuda)
    o = mq.exec_opts(capi.MQ_FAST, ag, schedule=sched)
    Y = dl.forward(dA, opts=o).cpu().numpy()
    ref, _, _ = O.mixed_linear(_oracle_layer(L), A, act_group=None if ag == 128 else ag)
    assert _rel(Y, ref) <= TOL
    for _ in range(2):
        assert np.array_equal(dl.forward(dA, opts=o).cpu().numpy(), Y)
    Yu = dl.forward(dA, opts=mq.exec_opts(capi.MQ_FAST, ag, schedule=1)).cpu().numpy()
    assert _rel(Yu, ref) <= TOL
