"""GPU offline weight quantization and prepack against the
host packer, which is itself pinned byte for byte to the reference
(test_host_packing.py, test_oracle_golden.py):

* mq_partition_and_quantize_device produces the reference layouts (payload,
  scales, zero points, index maps) bit for bit, for the engine schemes and for
  the reference's other legal schemes (odd group sizes, ragged K, f16 scale
  storage, 8-bit asymmetric), on degenerate groups (constant, zero) too;
* mq_layer_create_device packs the same engine-layout bytes and column map as
  mq_layer_create (also for a shard of a column-sharded layer);
* non-finite weights and bad metadata raise DataError before any packing.
"""
import numpy as np
import pytest

import oracle_py as O
import paper_2412_14590_b200 as mq
from paper_2412_14590_b200 import capi

pytestmark = pytest.mark.gpu


def _both(W, prom, large=mq.LARGEBIT, small=mq.SMALLBIT):
    import torch
    Lh = mq.partition_and_quantize(W, prom, large, small)
    dq = mq.partition_and_quantize_device(torch.from_numpy(W).cuda(), prom, large, small)
    return Lh, dq


def _same_ref_layouts(Lh, Ld):
    assert np.array_equal(Lh.index_map8, Ld.index_map8) and np.array_equal(Lh.index_map4, Ld.index_map4)
    for a, b in ((Lh.sub8, Ld.sub8), (Lh.sub4, Ld.sub4)):
        assert np.array_equal(a.payload, b.payload)
        assert np.array_equal(a.scales.view(np.uint32), b.scales.view(np.uint32))
        if a.zero_points is not None:
            assert np.array_equal(a.zero_points, b.zero_points)


@pytest.mark.parametrize("n,k,p", [(640, 2048, 0.1), (1024, 1000, 0.1), (300, 4096, 0.0), (257, 384, 1.0)])
def test_device_quantize_bit_exact(cuda, n, k, p):
    W, _, prom = mq.bench_inputs(1, n, k, p, 5)
    Lh, dq = _both(W, prom)
    _same_ref_layouts(Lh, dq.to_host())


@pytest.mark.parametrize("g", [100, 127, 64])
def test_device_quantize_other_schemes(cuda, g):
    """The reference accepts any group size (groups may straddle nibble pairs)
    and scale_f16_storage."""
    W, _, prom = mq.bench_inputs(1, 200, 1000, 0.2, 6)
    W[3, :] = 0.25          # constant groups (mx == mn)
    W[4, :g] = 0.0          # an all-zero group
    W[5, 10] = 1e-30        # tiny values
    large = mq.QuantScheme(8, True, g, g != 127)
    small = mq.QuantScheme(4, False, g, g == 127)
    Lh, dq = _both(W, prom, large, small)
    _same_ref_layouts(Lh, dq.to_host())


def test_device_quantize_matches_oracle_kats(cuda):
    """The restated reference quantizers (oracle) agree on the device path."""
    import torch
    W, _, prom = mq.bench_inputs(1, 128, 512, 0.1, 8)
    dq = mq.partition_and_quantize_device(torch.from_numpy(W).cuda(), prom).to_host()
    o4 = O.quantize_tensor(np.ascontiguousarray(W[dq.index_map4]), 4, False, 128)
    assert np.array_equal(dq.sub4.payload, o4.payload) and np.array_equal(dq.sub4.scales, o4.scales)


@pytest.mark.parametrize("n,k,rank,world", [(4096, 4096, 0, 1), (1000, 1000, 0, 1), (3000, 2048, 1, 3)])
def test_device_pack_same_bytes(cuda, n, k, rank, world):
    import torch
    W, _, prom = mq.bench_inputs(1, n, k, 0.1, 9)
    Lh = mq.partition_and_quantize(W, prom)
    dq = mq.partition_and_quantize_device(torch.from_numpy(W).cuda(), prom)
    a = mq.DeviceLayer(Lh, rank=rank, world=world)
    b = mq.DeviceLayer.from_device(dq, rank=rank, world=world)
    wa, ca = a.export_packed()
    wb, cb = b.export_packed()
    assert wa.size == wb.size and np.array_equal(wa, wb)
    assert np.array_equal(ca, cb)


def test_device_layer_forward_exact(cuda):
    """A layer quantized and packed entirely on the GPU reproduces the
    reference's golden C1-shape output in exact mode (same bytes => same bits)."""
    import torch
    W, A, prom = mq.bench_inputs(16, 1024, 2048, 0.1, 3)
    Lh = mq.partition_and_quantize(W, prom)
    dl = mq.DeviceLayer.from_device(mq.partition_and_quantize_device(torch.from_numpy(W).cuda(), prom))
    dA = torch.from_numpy(A).cuda()
    o = mq.exec_opts(capi.MQ_EXACT, 128)
    assert torch.equal(dl.forward(dA, opts=o), mq.DeviceLayer(Lh).forward(dA, opts=o))


def test_device_quantize_nonfinite_is_data_error(cuda):
    import torch
    W, _, prom = mq.bench_inputs(1, 64, 256, 0.1, 2)
    W[7, 200] = np.nan
    with pytest.raises(capi.DataError) as eh:
        mq.partition_and_quantize(W, prom)
    with pytest.raises(capi.DataError) as ed:
        mq.partition_and_quantize_device(torch.from_numpy(W).cuda(), prom)
    assert str(eh.value) == str(ed.value)


def test_device_create_checks_metadata(cuda):
    """validate_quantized on device metadata: a non-positive scale is a DataError."""
    import torch
    W, _, prom = mq.bench_inputs(1, 256, 256, 0.1, 4)
    dq = mq.partition_and_quantize_device(torch.from_numpy(W).cuda(), prom)
    Lh = dq.to_host()
    Lh.sub4.scales[3, 1] = 0.0
    bad = torch.from_numpy(Lh.sub4.scales).cuda()
    d = capi.mq_layer_desc.from_buffer_copy(dq.d)
    d.scales4 = bad.data_ptr()
    import ctypes as C
    h = C.c_void_p()
    st = capi.lib().mq_layer_create_device(C.byref(d), None, 0, None, C.byref(h))
    assert st == capi.MQ_DATA and b"non-positive scale" in capi.lib().mq_last_error()
