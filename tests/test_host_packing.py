"""Host side of the product (libmixllm_b200.so, C++), no GPU: the packing API
must be bit-exact with the oracle / the reference layouts, and raise the
reference's error types before any compute.

Reference: quantize_tensor (quant.hpp:183-243), pack/unpack_nibbles
(tensor.cpp:63-94), partition_and_quantize (mixed.cpp:46-81),
prepack_weights (gemm.cpp:89-108), reassemble_output (mixed.cpp:83-120),
run_bench's generator (gemm.cpp:211-227), fnv1a (gemm.cpp:194-204).
"""
import ctypes as C

import numpy as np
import pytest

import oracle_py as O
import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi


@pytest.mark.parametrize("m,n,k,p,seed", [(4, 64, 256, 0.1, 1), (1, 300, 200, 0.25, 2), (7, 129, 384, 1.0, 3),
                                          (2, 50, 130, 0.0, 4)])
def test_bench_inputs_identical(m, n, k, p, seed):
    a = mq.bench_inputs(m, n, k, p, seed)
    b = O.bench_inputs(m, n, k, p, seed)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("bits,sym,group,f16", [(4, False, 128, False), (8, True, 128, False), (8, True, 64, True),
                                                (4, False, 32, True), (8, False, 128, False), (8, True, 200, False)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_quantize_tensor_bit_exact(bits, sym, group, f16, dtype):
    m = (O.normal_matrix(9, 333, 7) * 3.0).astype(dtype)
    m[2, 5:70] = 0.0       # zero run (all-zero group when group <= 64)
    m[3, :] = -1.25        # constant rows
    q = mq.quantize_tensor(m, mq.QuantScheme(bits, sym, group, f16))
    r = O.quantize_tensor(m, bits, sym, group, f16)
    assert np.array_equal(q.payload, r.payload)
    assert np.array_equal(q.scales, r.scales)
    if not sym:
        assert np.array_equal(q.zero_points, r.zps)


def test_quantize_tensor_errors():
    m = np.ones((3, 8))
    m[2, 6] = np.nan
    with pytest.raises(mq.DataError, match="row 2, group 1"):
        mq.quantize_tensor(m, mq.QuantScheme(4, False, 4))
    with pytest.raises(mq.UsageError):
        mq.quantize_tensor(np.ones((1, 8)), mq.QuantScheme(4, True, 128))  # 4-bit symmetric
    with pytest.raises(mq.UsageError):
        mq.quantize_tensor(np.ones((1, 8)), mq.QuantScheme(5, False, 128))
    with pytest.raises(mq.UsageError):
        mq.quantize_tensor(np.ones((1, 8)), mq.QuantScheme(4, False, 0))


def test_kats_through_product():  # test_quant_core.cpp:33-80 via the product's tensor quantizer
    q = mq.quantize_tensor(np.array([[0.0, 1.0, 2.0, 3.0]]), mq.QuantScheme(4, False, 128))
    assert q.scales[0, 0] == np.float32(0.2) and q.zero_points[0, 0] == 0
    assert [q.code(0, i) for i in range(4)] == [0, 5, 10, 15]
    q = mq.quantize_tensor(np.array([[-1.0, 0.5]]), mq.QuantScheme(8, True, 128))
    assert [q.code(0, i) for i in range(2)] == [-127, 64]
    q = mq.quantize_tensor(np.array([[-2.0, -2.0]]), mq.QuantScheme(4, False, 128))
    assert q.scales[0, 0] == 2.0 and q.zero_points[0, 0] == 1
    assert mq.fast_i2f(5) == 5.0 and mq.fast_i2f(-(1 << 22)) == -(1 << 22)
    assert mq.round_scale_f16(1.0) == 1.0 and mq.round_scale_f16(1e-12) > 0


def test_nibbles():  # test_tensor_store.cpp:10-41
    assert mq.pack_nibbles([3, 5]).tolist() == [0x53]
    assert mq.pack_nibbles([15, 15, 1]).tolist() == [0xFF, 0x01]
    with pytest.raises(mq.DataError):
        mq.pack_nibbles([16])
    with pytest.raises(mq.DataError):
        mq.unpack_nibbles([0x12], 3)
    rng = np.random.default_rng(5)
    for _ in range(200):
        v = rng.integers(0, 16, int(rng.integers(0, 70))).astype(np.uint8)
        assert np.array_equal(mq.unpack_nibbles(mq.pack_nibbles(v), v.size), v)


@pytest.mark.parametrize("n,k,p,seed", [(256, 512, 0.1, 1), (300, 200, 0.3, 2), (77, 130, 0.0, 3),
                                        (64, 256, 1.0, 4), (1, 128, 1.0, 5)])
def test_partition_prepack_bit_exact(n, k, p, seed):
    W, _, prom = mq.bench_inputs(1, n, k, p, seed)
    L = mq.partition_and_quantize(W, prom)
    R = O.partition_and_quantize(W, prom)
    assert np.array_equal(L.index_map8, R.map8) and np.array_equal(L.index_map4, R.map4)
    assert np.array_equal(L.sub8.payload, R.sub8.payload) and np.array_equal(L.sub8.scales, R.sub8.scales)
    assert np.array_equal(L.sub4.payload, R.sub4.payload) and np.array_equal(L.sub4.scales, R.sub4.scales)
    assert np.array_equal(L.sub4.zero_points, R.sub4.zps)
    assert np.array_equal(mq.prepack_weights(L, 0), O.prepack(R.sub8))
    assert np.array_equal(mq.prepack_weights(L, 1), O.prepack(R.sub4))
    mq.validate_mixed_layer(L)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_partition_matches_reference_build():
    W, _, prom = mq.bench_inputs(1, 200, 384, 0.2, 9)
    L = mq.partition_and_quantize(W, prom)
    ex = O.RefLayer(W, prom, 128).export()
    assert np.array_equal(L.sub8.payload, ex["p8"]) and np.array_equal(L.sub4.payload, ex["p4"])
    assert np.array_equal(L.sub4.zero_points, ex["z4"]) and np.array_equal(L.sub4.scales, ex["s4"])


def test_partition_errors():
    W = np.ones((6, 8))
    with pytest.raises(mq.UsageError):
        mq.partition_and_quantize(W, [6])      # out of range
    with pytest.raises(mq.UsageError):
        mq.partition_and_quantize(W, [1, 1])   # duplicate
    with pytest.raises(mq.DataError, match="share group boundaries"):  # validate_mixed_layer, mixed.cpp:39-42
        mq.partition_and_quantize(W, [1], mq.QuantScheme(8, True, 128), mq.QuantScheme(4, False, 64))


def test_validate_layer_rejects_broken_maps():
    W, _, prom = mq.bench_inputs(1, 64, 256, 0.25, 3)
    L = mq.partition_and_quantize(W, prom)
    L.index_map4 = L.index_map4.copy()
    L.index_map4[0] = L.index_map8[0]  # a column covered twice
    with pytest.raises(mq.DataError):
        mq.validate_mixed_layer(L)
    L2 = mq.partition_and_quantize(W, prom)
    L2.sub4.scales = L2.sub4.scales.copy()
    L2.sub4.scales[1, 0] = 0.0         # non-positive scale (quant.cpp:98)
    with pytest.raises(mq.DataError):
        mq.validate_mixed_layer(L2)


def test_reassemble_output():
    y8 = np.array([[10.0, 40.0]], np.float32)
    y4 = np.array([[0.0, 2.0, 3.0, 5.0]], np.float32)
    out = mq.reassemble_output(y8, y4, np.array([1, 4]), np.array([0, 2, 3, 5]), 6)
    assert out.tolist() == [[0.0, 10.0, 2.0, 3.0, 40.0, 5.0]]
    assert np.array_equal(out, O.reassemble(y8, y4, np.array([1, 4]), np.array([0, 2, 3, 5]), 6))
    with pytest.raises(mq.DataError):
        mq.reassemble_output(y8, y4, np.array([1, 1]), np.array([0, 2, 3, 5]), 6)
    with pytest.raises(mq.UsageError):
        mq.reassemble_output(y8, y4, np.array([1]), np.array([0, 2, 3, 5]), 6)


def test_fnv1a_matches_oracle():
    a = np.arange(1000, dtype=np.float32) * 0.37
    assert mq.fnv1a_hex(a) == O.fnv1a_hex(a)
    assert mq.fnv1a_hex(np.zeros(0, np.uint8)) == "cbf29ce484222325"  # FNV-1a-64 offset basis


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_plan_covers_every_column_once(world):
    W, _, prom = mq.bench_inputs(1, 1000, 128, 0.1, 11)
    L = mq.partition_and_quantize(W, prom)
    sc, cm = mq.shard_plan(L, world)
    valid = cm[cm >= 0]
    assert np.array_equal(np.sort(valid), np.arange(1000))
    n8, n4 = L.sub8.rows, L.sub4.rows
    for r in range(world):  # balanced per precision: rank r holds both partitions' slices
        row = cm[r][cm[r] >= 0]
        a8, b8 = n8 * r // world, n8 * (r + 1) // world
        a4, b4 = n4 * r // world, n4 * (r + 1) // world
        assert np.array_equal(row, np.concatenate([L.index_map8[a8:b8], L.index_map4[a4:b4]]))
    assert sc == max((n8 * (r + 1) // world - n8 * r // world) + (n4 * (r + 1) // world - n4 * r // world)
                     for r in range(world))


def test_no_device_fails_loudly():
    """Device entry points have no CPU fallback: without a GPU they return MQ_CUDA."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    W, _, prom = mq.bench_inputs(1, 64, 256, 0.1, 1)
    L = mq.partition_and_quantize(W, prom)
    with pytest.raises(capi.CudaError):
        mq.DeviceLayer(L)


def test_capi_exports_every_declared_symbol():
    """Every function declared in include/*.h is exported by the library."""
    import os
    import re
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    names = set()
    for d, _, fs in os.walk(os.path.join(root, "include")):
        for f in fs:
            if f.endswith(".h"):
                src = open(os.path.join(d, f)).read()
                src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
                names |= set(re.findall(r"\b(mq_[a-z0-9_]+)\s*\(", src))
    assert len(names) >= 25
    lib = C.CDLL(capi.LIB_PATH)
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(capi.PROTOTYPES) <= names  # the binding declares nothing the header lacks
