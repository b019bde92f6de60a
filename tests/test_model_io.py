"""quantized.json ("mixquant-quantized-v1", mixed.cpp:208-370) I/O of the host
mirror, pinned to the REFERENCE's own writer and reader:
tests/golden/quantized_v1/ was written by the reference's save_quantized_model
(tests/golden/make_quantized_fixture.py, oracle/_ref); the loader must read it
back bit-identical to partition_and_quantize of the same seeded weights, and
the reference's load_quantized_model must read what our saver writes."""
import json
import os
import shutil

import numpy as np
import pytest

import paper_2412_14590_b200 as mq

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURE = os.path.join(HERE, "golden", "quantized_v1")
LAYERS = [("blk0.proj", 256, 384, 0.10, 1), ("blk0.pure4", 128, 256, 0.0, 2)]


def _expected():
    out = {}
    for name, n, k, p, seed in LAYERS:
        W, _, prom = mq.bench_inputs(1, n, k, p, seed)
        out[name] = mq.partition_and_quantize(W, prom, name=name)
    return out


def _same(a: mq.MixedLinearLayer, b: mq.MixedLinearLayer):
    assert (a.name, a.out_features, a.in_features) == (b.name, b.out_features, b.in_features)
    assert np.array_equal(a.index_map8, b.index_map8) and np.array_equal(a.index_map4, b.index_map4)
    for sa, sb in ((a.sub8, b.sub8), (a.sub4, b.sub4)):
        assert (sa.rows, sa.cols, sa.scheme) == (sb.rows, sb.cols, sb.scheme)
        assert np.array_equal(sa.payload.reshape(-1), sb.payload.reshape(-1))
        assert np.array_equal(sa.scales.view(np.uint32), sb.scales.view(np.uint32))
        if sa.zero_points is not None or sb.zero_points is not None:
            assert np.array_equal(sa.zero_points, sb.zero_points)


def test_load_reference_written_fixture():
    qm = mq.load_quantized_model(FIXTURE)
    assert qm.source_model == "run_bench-seeded" and qm.percent == pytest.approx(0.10)
    assert qm.largebit == mq.LARGEBIT and qm.smallbit == mq.SMALLBIT and qm.act_scheme == mq.ACT_SCHEME
    exp = _expected()
    assert [l.name for l in qm.linears] == [n for n, *_ in LAYERS]
    for layer in qm.linears:
        _same(layer, exp[layer.name])
    assert qm.linears[1].sub8.rows == 0  # empty sub-problem: no files, rebuilt from the scheme


def test_save_round_trip_and_reference_reads_it(tmp_path):
    exp = _expected()
    qm = mq.QuantizedModel("run_bench-seeded", 0.10, linears=[exp[n] for n, *_ in LAYERS])
    out = str(tmp_path / "q")
    mq.save_quantized_model(qm, out)
    assert sorted(os.listdir(out)) == sorted(os.listdir(FIXTURE))
    for f in os.listdir(FIXTURE):  # tensor files byte-identical to the reference writer's
        if f.endswith(".bin"):
            assert open(os.path.join(out, f), "rb").read() == open(os.path.join(FIXTURE, f), "rb").read(), f
    assert json.load(open(os.path.join(out, "quantized.json"))) == json.load(open(os.path.join(FIXTURE, "quantized.json")))
    back = mq.load_quantized_model(out)
    for a, b in zip(back.linears, qm.linears):
        _same(a, b)
    O = pytest.importorskip("oracle_py")
    if not os.path.exists(O.REF_SO):
        pytest.skip("oracle/_ref not built")
    refs = O.RefLayer.load_quantized(out)
    for r, layer in zip(refs, qm.linears):
        e = r.export()
        assert np.array_equal(e["map8"], layer.index_map8) and np.array_equal(e["map4"], layer.index_map4)
        assert np.array_equal(e["p4"], layer.sub4.payload) and np.array_equal(e["z4"], layer.sub4.zero_points)
        assert np.array_equal(e["s4"].view(np.uint32), layer.sub4.scales.view(np.uint32))
        if layer.sub8.rows:
            assert np.array_equal(e["p8"], layer.sub8.payload)


def _copy(tmp_path):
    d = str(tmp_path / "fx")
    shutil.copytree(FIXTURE, d)
    return d


def test_errors_match_reference_classes(tmp_path):
    with pytest.raises(mq.DataError, match="cannot open"):
        mq.load_quantized_model(str(tmp_path / "missing"))
    d = _copy(tmp_path)
    with open(os.path.join(d, "blk0.proj.sub4.scales.bin"), "r+b") as f:  # truncated tensor
        f.truncate(100)
    with pytest.raises(mq.DataError, match="bytes, expected"):
        mq.load_quantized_model(d)
    d = _copy(tmp_path / "b")
    j = json.load(open(os.path.join(d, "quantized.json")))
    del j["layers"][0]["in_features"]  # malformed manifest
    json.dump(j, open(os.path.join(d, "quantized.json"), "w"))
    with pytest.raises(mq.DataError, match="malformed"):
        mq.load_quantized_model(d)
    d = _copy(tmp_path / "c")
    j = json.load(open(os.path.join(d, "quantized.json")))
    j["smallbit"]["bit_width"] = 3  # validate_scheme -> UsageError (mixed.cpp:226)
    json.dump(j, open(os.path.join(d, "quantized.json"), "w"))
    with pytest.raises(mq.UsageError, match="bit_width"):
        mq.load_quantized_model(d)
    d = _copy(tmp_path / "e")
    j = json.load(open(os.path.join(d, "quantized.json")))
    j["layers"][0]["index_map4"][0] = 6  # maps no longer a permutation -> validate_mixed_layer
    json.dump(j, open(os.path.join(d, "quantized.json"), "w"))
    with pytest.raises(mq.DataError):
        mq.load_quantized_model(d)
