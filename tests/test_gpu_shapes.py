"""GPU parity on the shapes bench.py measures (BASELINE configs[1]: the fused
Llama-3.1-8B projections) and on the Llama-3.1-70B linear shapes (configs[2]).

- MQ_EXACT reproduces the REFERENCE's own output checksum (golden.json
  "cases_large", generated from oracle/_ref = the reference sources compiled
  unmodified, tests/golden/make_golden.py) at qkv 6144x4096, gate_up
  28672x4096, down 4096x14336 (M 16 and 512), 70B 8192x8192 (M 16 and 256),
  1024x8192, 28672x8192 (M 1) and 8192x28672 (G = 224).
- MQ_FAST (the mode bench.py times) at M in {1, 16, 64, 256, 512} on every
  shape: the full output within max|fast - exact| <= 1e-3 * max|exact|, and a
  sample of output features (both sub-problems) against the C oracle
  (oracle/mqo.c, gemm_block restated) within the same bound.
- fp16 output (the bench's output type) equals the f32 result rounded once.
"""
import numpy as np
import pytest

import oracle_py as O
import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi

pytestmark = pytest.mark.gpu
TOL = 1e-3  # north_star: fp32-relative tolerance of rescaled outputs

SHAPES = {
    "8b_qkv": (6144, 4096), "8b_o": (4096, 4096), "8b_gate_up": (28672, 4096), "8b_down": (4096, 14336),
    "70b_qo": (8192, 8192), "70b_kv": (1024, 8192), "70b_gate": (28672, 8192), "70b_down": (8192, 28672),
}
BATCHES = (1, 16, 64, 256, 512)
_CACHE = {}


def _layer(n, k, p=0.10, seed=1):
    key = (n, k, p, seed)
    if key not in _CACHE:
        if len(_CACHE) >= 3:  # bound host + device memory across the module
            _CACHE.pop(next(iter(_CACHE)))
        W, _, prom = mq.bench_inputs(1, n, k, p, seed)
        L = mq.partition_and_quantize(W, prom)
        del W
        _CACHE[key] = (L, mq.DeviceLayer(L))
    return _CACHE[key]


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def _rows(q, idx, bits):
    """Oracle QTensor of the selected rows of one sub-problem."""
    return O.QTensor(bits, bits == 8, 128, len(idx), q.cols, np.ascontiguousarray(q.payload[idx]),
                     np.ascontiguousarray(q.scales[idx]),
                     None if bits == 8 else np.ascontiguousarray(q.zero_points[idx]))


def _oracle_sample(L, A, act_group, rng, n8s=32, n4s=64):
    """Oracle outputs of a random sample of sub8 and sub4 output features:
    (original columns, f32 [M, cols])."""
    codes, scales = O.quantize_acts(A, act_group)
    cols, outs = [], []
    for q, bits, mp, ns in ((L.sub8, 8, L.index_map8, n8s), (L.sub4, 4, L.index_map4, n4s)):
        if q.rows == 0:
            continue
        idx = np.sort(rng.choice(q.rows, size=min(ns, q.rows), replace=False))
        outs.append(O.gemm_sub(codes, scales, _rows(q, idx, bits)))
        cols.append(mp[idx])
    return np.concatenate(cols), np.concatenate(outs, axis=1)


@pytest.mark.parametrize("idx", range(9))
def test_exact_large_shapes_match_reference_checksum(cuda, golden, idx):
    import torch
    c = golden["cases_large"][idx]
    W, A, prom = mq.bench_inputs(c["m"], c["n"], c["k"], c["percent"], 1)
    L = mq.partition_and_quantize(W, prom)
    del W
    assert (L.sub8.rows, L.sub4.rows) == (c["n8"], c["n4"])
    dl = mq.DeviceLayer(L)
    dA = torch.from_numpy(A).to(cuda)
    codes, _ = mq.quantize_act(dA, 128)
    assert mq.fnv1a_hex(codes.cpu().numpy()[:, :c["k"]]) == c["act_codes"]
    Y = dl.forward(dA, opts=mq.exec_opts(capi.MQ_EXACT, 128)).cpu().numpy()
    assert mq.fnv1a_hex(Y) == c["out_f32"], f"exact checksum differs from the reference at {c['m']}x{c['n']}x{c['k']}"


@pytest.mark.parametrize("m", BATCHES)
@pytest.mark.parametrize("shape", list(SHAPES))
def test_fast_mode_bench_shapes(cuda, shape, m):
    import torch
    n, k = SHAPES[shape]
    L, dl = _layer(n, k)
    rng = np.random.default_rng(1000 + m)
    A = rng.standard_normal((m, k)).astype(np.float32)
    dA = torch.from_numpy(A).to(cuda)
    fast = mq.exec_opts(capi.MQ_FAST, 128)
    yf = dl.forward(dA, opts=fast).cpu().numpy()
    ye = dl.forward(dA, opts=mq.exec_opts(capi.MQ_EXACT, 128)).cpu().numpy()
    assert _rel(yf, ye) <= TOL
    cols, ref = _oracle_sample(L, A, 128, rng)
    assert _rel(yf[:, cols], ref) <= TOL
    assert np.array_equal(ye[:, cols], ref)  # exact mode: bit-identical on the sample too
    if m == 16:  # the bench's output type
        y16 = dl.forward(dA, opts=fast, out_dtype=torch.float16).cpu()
        assert torch.equal(y16, torch.from_numpy(yf).half())


@pytest.mark.parametrize("m", (16, 512))
@pytest.mark.parametrize("shape", ["8b_qkv", "8b_down", "70b_qo"])
def test_fast_mode_per_token_bench_shapes(cuda, shape, m):
    import torch
    n, k = SHAPES[shape]
    L, dl = _layer(n, k)
    rng = np.random.default_rng(2000 + m)
    A = rng.standard_normal((m, k)).astype(np.float32)
    yf = dl.forward(torch.from_numpy(A).to(cuda), opts=mq.exec_opts(capi.MQ_FAST, k)).cpu().numpy()
    cols, ref = _oracle_sample(L, A, k, rng)
    assert _rel(yf[:, cols], ref) <= TOL
