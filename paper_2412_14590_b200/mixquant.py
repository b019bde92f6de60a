"""Python mirror of the reference's `mixquant` hot-path API over the C ABI.

Same names, argument meaning and error behaviour as the reference C++ API
(proj/include/mixquant/{quant,mixed,gemm}.hpp): UsageError / DataError are
raised before any compute. Host packing runs in the C++ library (bit-exact);
every GEMM runs on the B200 through libmixllm_b200.so — there is no CPU path.
Device buffers are torch CUDA tensors (plumbing only).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import capi
from .capi import DataError, UsageError, check, lib  # noqa: F401

P = C.c_void_p


def _p(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(P)
    return C.c_void_p(a.data_ptr())  # torch tensor


# ------------------------------------------------------------------ schemes
@dataclass(frozen=True)
class QuantScheme:
    """QuantScheme (quant.hpp:25-36)."""
    bit_width: int = 4
    symmetric: bool = False
    group_size: int = 128
    scale_f16_storage: bool = False

    def c(self) -> capi.mq_scheme:
        return capi.mq_scheme(self.bit_width, int(self.symmetric), self.group_size, int(self.scale_f16_storage))


LARGEBIT = QuantScheme(8, True, 128)   # gemm.cpp:229
SMALLBIT = QuantScheme(4, False, 128)  # gemm.cpp:230
ACT_SCHEME = QuantScheme(8, True, 128)  # gemm.cpp:231


@dataclass
class QuantizedTensor:
    """QuantizedTensor (quant.hpp:146-176), reference layouts, host numpy."""
    scheme: QuantScheme
    rows: int
    cols: int
    payload: np.ndarray
    scales: np.ndarray
    zero_points: np.ndarray | None

    def num_groups(self) -> int:
        return 0 if self.cols == 0 else (self.cols + self.scheme.group_size - 1) // self.scheme.group_size

    def row_stride_bytes(self) -> int:
        return (self.cols + 1) // 2 if self.scheme.bit_width == 4 else self.cols

    def code(self, r: int, c: int) -> int:
        if self.scheme.bit_width == 4:
            b = int(self.payload[r, c // 2])
            return (b >> 4) if c % 2 else (b & 0x0F)
        b = int(self.payload[r, c])
        return b - 256 if (self.scheme.symmetric and b > 127) else b


def quantize_tensor(m: np.ndarray, scheme: QuantScheme) -> QuantizedTensor:
    """quantize_tensor<float|double> (quant.hpp:183-243)."""
    m = np.ascontiguousarray(m)
    if m.ndim != 2:
        raise UsageError("quantize_tensor expects a matrix")
    rows, cols = m.shape
    g = scheme.group_size
    if g < 1:
        raise UsageError(f"group_size must be >= 1, got {g}")
    G = 0 if cols == 0 else (cols + g - 1) // g
    stride = (cols + 1) // 2 if scheme.bit_width == 4 else cols
    payload = np.zeros((rows, stride), np.uint8)
    scales = np.zeros((rows, G), np.float32)
    zps = None if scheme.symmetric else np.zeros((rows, G), np.uint8)
    sc = scheme.c()
    if m.dtype == np.float64:
        st = lib().mq_quantize_tensor_f64(_p(m), rows, cols, C.byref(sc), _p(payload), _p(scales), _p(zps), None, None)
    elif m.dtype == np.float32:
        st = lib().mq_quantize_tensor_f32(_p(m), rows, cols, C.byref(sc), _p(payload), _p(scales), _p(zps), None, None)
    else:
        raise UsageError(f"unsupported dtype {m.dtype}")
    check(st)
    return QuantizedTensor(scheme, rows, cols, payload, scales, zps)


def pack_nibbles(values) -> np.ndarray:
    v = np.ascontiguousarray(np.asarray(values, np.uint8))
    out = np.zeros((v.size + 1) // 2, np.uint8)
    check(lib().mq_pack_nibbles(_p(v), v.size, _p(out)))
    return out


def unpack_nibbles(data, count: int) -> np.ndarray:
    b = np.ascontiguousarray(np.asarray(data, np.uint8))
    out = np.zeros(max(count, 0), np.uint8)
    check(lib().mq_unpack_nibbles(_p(b), b.size, count, _p(out)))
    return out


def fast_i2f(x: int) -> float:
    return lib().mq_fast_i2f(x)


def round_scale_f16(s: float) -> float:
    return lib().mq_round_scale_f16(s)


def fnv1a_hex(a) -> str:
    a = np.ascontiguousarray(a)
    return "%016x" % lib().mq_fnv1a(_p(a), a.nbytes)


# ----------------------------------------------------------------- layers
@dataclass
class MixedLinearLayer:
    """MixedLinearLayer (mixed.hpp:16-24): reference layouts on the host."""
    name: str
    out_features: int
    in_features: int
    sub8: QuantizedTensor
    sub4: QuantizedTensor
    index_map8: np.ndarray
    index_map4: np.ndarray
    _keep: list = field(default_factory=list, repr=False)

    def desc(self) -> capi.mq_layer_desc:
        d = capi.mq_layer_desc()
        d.out_features = self.out_features
        d.in_features = self.in_features
        d.group_size = (self.sub4 if self.sub4.rows else self.sub8).scheme.group_size
        d.n8, d.n4 = self.sub8.rows, self.sub4.rows
        arrs = [np.ascontiguousarray(x) for x in (self.index_map8.astype(np.int32), self.index_map4.astype(np.int32),
                                                  self.sub8.payload, self.sub8.scales, self.sub4.payload,
                                                  self.sub4.scales,
                                                  self.sub4.zero_points if self.sub4.zero_points is not None
                                                  else np.zeros((0,), np.uint8))]
        self._keep = arrs
        (d.index_map8, d.index_map4, d.payload8, d.scales8, d.payload4, d.scales4, d.zero_points4) = \
            [a.ctypes.data for a in arrs]
        return d


def partition_and_quantize(weight: np.ndarray, promoted, largebit: QuantScheme = LARGEBIT,
                           smallbit: QuantScheme = SMALLBIT, name: str = "") -> MixedLinearLayer:
    """partition_and_quantize (mixed.cpp:46-81) — host C++, bit-exact."""
    W = np.ascontiguousarray(weight, np.float64)
    N, K = W.shape
    prom = np.ascontiguousarray(np.asarray(promoted, np.int32).reshape(-1))
    h = C.c_void_p()
    check(lib().mq_partition_and_quantize(_p(W), N, K, _p(prom), prom.size, C.byref(largebit.c()),
                                          C.byref(smallbit.c()), C.byref(h)))
    try:
        d = capi.mq_layer_desc()
        check(lib().mq_host_layer_desc(h, C.byref(d)))
        G = 0 if K == 0 else (K + largebit.group_size - 1) // largebit.group_size

        def arr(ptr, n, dt):
            if n == 0:
                return np.zeros((0,), dt)
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(np.ctypeslib.as_ctypes_type(dt))), (n,)).copy()

        n8, n4 = d.n8, d.n4
        sub8 = QuantizedTensor(largebit, n8, K, arr(d.payload8, n8 * K, np.uint8).reshape(n8, K),
                               arr(d.scales8, n8 * G, np.float32).reshape(n8, G), None)
        s4 = (K + 1) // 2
        sub4 = QuantizedTensor(smallbit, n4, K, arr(d.payload4, n4 * s4, np.uint8).reshape(n4, s4),
                               arr(d.scales4, n4 * G, np.float32).reshape(n4, G),
                               arr(d.zero_points4, n4 * G, np.uint8).reshape(n4, G))
        return MixedLinearLayer(name, N, K, sub8, sub4, arr(d.index_map8, n8, np.int32), arr(d.index_map4, n4, np.int32))
    finally:
        lib().mq_host_layer_destroy(h)


class DeviceQuantizedLayer:
    """partition_and_quantize on the GPU (mq_partition_and_quantize_device):
    the reference layouts stay in device memory (owned here); index maps on
    the host. `to_host()` copies them into a MixedLinearLayer (e.g. for
    save_quantized_model); `DeviceLayer.from_device(...)` packs the engine
    layout on the GPU."""

    def __init__(self, handle, device: int, largebit: QuantScheme, smallbit: QuantScheme, name: str = ""):
        self.h = handle
        self.device = device
        self.largebit, self.smallbit, self.name = largebit, smallbit, name
        self.d = capi.mq_layer_desc()
        check(lib().mq_device_qlayer_desc(handle, C.byref(self.d)))

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            try:
                lib().mq_device_qlayer_destroy(h)
            except Exception:
                pass
            self.h = None

    def to_host(self) -> MixedLinearLayer:
        d = self.d
        K = d.in_features
        G = 0 if K == 0 else (K + d.group_size - 1) // d.group_size

        def dev(ptr, n, dt):
            if n == 0:
                return np.zeros((0,), dt)
            nbytes = n * np.dtype(dt).itemsize
            return _device_view(ptr, nbytes, self.device).cpu().numpy().view(dt).copy()

        def host(ptr, n, dt):
            if n == 0:
                return np.zeros((0,), dt)
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(np.ctypeslib.as_ctypes_type(dt))), (n,)).copy()

        n8, n4, s4 = d.n8, d.n4, (K + 1) // 2
        sub8 = QuantizedTensor(self.largebit, n8, K, dev(d.payload8, n8 * K, np.uint8).reshape(n8, K),
                               dev(d.scales8, n8 * G, np.float32).reshape(n8, G), None)
        sub4 = QuantizedTensor(self.smallbit, n4, K, dev(d.payload4, n4 * s4, np.uint8).reshape(n4, s4),
                               dev(d.scales4, n4 * G, np.float32).reshape(n4, G),
                               dev(d.zero_points4, n4 * G, np.uint8).reshape(n4, G))
        return MixedLinearLayer(self.name, d.out_features, K, sub8, sub4, host(d.index_map8, n8, np.int32),
                                host(d.index_map4, n4, np.int32))


def _device_view(ptr, nbytes: int, device: int):
    """A uint8 CUDA tensor view of `nbytes` at a raw device pointer owned by the
    library (torch as plumbing: __cuda_array_interface__, no copy, no ownership)."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (int(ptr), False), "version": 3,
                                    "strides": None}
    with torch.cuda.device(device):
        return torch.as_tensor(_Arr(), device=f"cuda:{device}")


def pinned_view(t):
    """A CUDA tensor aliasing a pinned host tensor (UVA): the engine's kernels read
    or write it over PCIe directly — e.g. K1 quantizing activations straight from
    pinned host memory, with no copy-engine transfer in between."""
    import torch
    if t.is_cuda or not t.is_pinned():
        raise UsageError("pinned_view expects a pinned host tensor")
    typestr = {torch.float32: "<f4", torch.float16: "<f2", torch.bfloat16: "<V2", torch.uint8: "|u1"}[t.dtype]

    class _A:
        __cuda_array_interface__ = {"shape": tuple(t.shape), "typestr": typestr, "data": (t.data_ptr(), False),
                                    "version": 3, "strides": None}
    v = torch.as_tensor(_A(), device=f"cuda:{torch.cuda.current_device()}")
    return v.view(t.dtype) if t.dtype == torch.bfloat16 else v


def partition_and_quantize_device(weight, promoted, largebit: QuantScheme = LARGEBIT,
                                  smallbit: QuantScheme = SMALLBIT, name: str = "",
                                  stream=None) -> DeviceQuantizedLayer:
    """partition_and_quantize (mixed.cpp:46-81) on the GPU, bit-exact with the
    host version: weight is a CUDA float64 [N, K] tensor."""
    import torch
    if not (isinstance(weight, torch.Tensor) and weight.is_cuda and weight.dtype == torch.float64):
        raise UsageError("partition_and_quantize_device expects a CUDA float64 weight tensor")
    W = weight.contiguous()
    N, K = W.shape
    prom = np.ascontiguousarray(np.asarray(promoted, np.int32).reshape(-1))
    h = C.c_void_p()
    check(lib().mq_partition_and_quantize_device(_p(W), N, K, _p(prom), prom.size, C.byref(largebit.c()),
                                                 C.byref(smallbit.c()), W.device.index, _stream(stream), C.byref(h)))
    return DeviceQuantizedLayer(h, W.device.index, largebit, smallbit, name)


# ------------------------------------------------------- quantized model I/O
# "mixquant-quantized-v1" directories (mixed.cpp:208-370): quantized.json plus
# raw little-endian tensors per sub-problem — <layer>.sub{8,4}.codes.bin u8
# [rows, row_stride], .scales.bin f32 [rows, G], .zero_points.bin u8 [rows, G]
# (asymmetric only). Empty sub-problems write no files.
QUANTIZED_FORMAT = "mixquant-quantized-v1"


@dataclass
class QuantizedModel:
    """QuantizedModel (mixed.hpp:81-88)."""
    source_model: str = ""
    percent: float = 0.0
    act_scheme: QuantScheme = ACT_SCHEME
    largebit: QuantScheme = LARGEBIT
    smallbit: QuantScheme = SMALLBIT
    linears: list = field(default_factory=list)


def _scheme_json(s: QuantScheme) -> dict:  # scheme_to_json (mixed.cpp:213-218)
    return {"bit_width": s.bit_width, "symmetric": bool(s.symmetric), "group_size": s.group_size,
            "scale_f16_storage": bool(s.scale_f16_storage)}


def _scheme_from_json(j) -> QuantScheme:  # scheme_from_json (mixed.cpp:220-228)
    s = QuantScheme(int(j["bit_width"]), bool(j["symmetric"]), int(j["group_size"]), bool(j["scale_f16_storage"]))
    if s.bit_width not in (4, 8):  # validate_scheme (quant.cpp:7-16)
        raise UsageError(f"bit_width must be 4 or 8, got {s.bit_width}")
    if s.group_size < 1:
        raise UsageError(f"group_size must be >= 1, got {s.group_size}")
    return s


_DTYPES = {"f64": (np.float64, 8), "f32": (np.float32, 4), "i32": (np.int32, 4), "i8": (np.int8, 1),
           "u8": (np.uint8, 1)}  # dtype_from_name / dtype_payload_bytes (tensor.cpp:19-39)


def save_quantized_model(qm: QuantizedModel, path) -> None:
    """save_quantized_model (mixed.cpp:308-334) + write_sub (:251-274)."""
    import json
    import os
    os.makedirs(path, exist_ok=True)
    layers = []
    for layer in qm.linears:
        validate_mixed_layer(layer)
        tensors = {}
        for tag, sub in (("sub8", layer.sub8), ("sub4", layer.sub4)):
            if sub.rows == 0:
                continue
            prefix = f"{layer.name}.{tag}"
            roles = [("codes", "u8", np.ascontiguousarray(sub.payload, np.uint8).reshape(sub.rows, -1)),
                     ("scales", "f32", np.ascontiguousarray(sub.scales, np.float32))]
            if not sub.scheme.symmetric:
                roles.append(("zero_points", "u8", np.ascontiguousarray(sub.zero_points, np.uint8)))
            for role, dt, arr in roles:
                fname = f"{prefix}.{role}.bin"
                arr.tofile(os.path.join(path, fname))
                tensors[f"{prefix}_{role}"] = {"file": fname, "dtype": dt, "shape": [int(d) for d in arr.shape]}
        layers.append({"name": layer.name, "out_features": int(layer.out_features),
                       "in_features": int(layer.in_features),
                       "index_map8": [int(v) for v in layer.index_map8],
                       "index_map4": [int(v) for v in layer.index_map4], "tensors": tensors})
    j = {"format": QUANTIZED_FORMAT, "source_model": qm.source_model, "percent": float(qm.percent),
         "act_scheme": _scheme_json(qm.act_scheme), "largebit": _scheme_json(qm.largebit),
         "smallbit": _scheme_json(qm.smallbit), "layers": layers}
    try:
        with open(os.path.join(path, "quantized.json"), "w") as f:
            f.write(json.dumps(j, indent=2) + "\n")
    except OSError as e:
        raise DataError(f"cannot write quantized manifest in '{path}': {e}") from None


def load_quantized_model(path) -> QuantizedModel:
    """load_quantized_model (mixed.cpp:336-370) + read_sub (:276-306): DataError
    on a missing or malformed manifest, a tensor whose bytes do not match its
    declared shape (make_tensor, tensor.cpp:47-61), or a layer that fails
    validate_mixed_layer."""
    import json
    import os
    manifest = os.path.join(path, "quantized.json")
    try:
        with open(manifest) as f:
            text = f.read()
    except OSError:
        raise DataError(f"cannot open '{manifest}'") from None
    try:
        j = json.loads(text)
        qm = QuantizedModel(str(j["source_model"]), float(j["percent"]), _scheme_from_json(j["act_scheme"]),
                            _scheme_from_json(j["largebit"]), _scheme_from_json(j["smallbit"]))

        def read_tensor(jt, role):
            ref = jt[role]
            fname = os.path.join(path, str(ref["file"]))
            if str(ref["dtype"]) not in _DTYPES:
                raise DataError(f"unknown dtype '{ref['dtype']}'")
            dt, width = _DTYPES[str(ref["dtype"])]
            shape = [int(d) for d in ref["shape"]]
            if not shape or any(d < 1 for d in shape):
                raise DataError("tensor dimensions must be >= 1")
            try:
                raw = np.fromfile(fname, np.uint8)
            except OSError:
                raise DataError(f"cannot open '{fname}'") from None
            expected = int(np.prod(shape)) * width
            if raw.size != expected:
                raise DataError(f"tensor payload is {raw.size} bytes, expected {expected}")
            return raw.view(dt).reshape(shape)

        def read_sub(jt, prefix, scheme, rows, cols):
            G = 0 if cols == 0 else (cols + scheme.group_size - 1) // scheme.group_size
            if rows == 0:
                stride = cols if scheme.bit_width == 8 else (cols + 1) // 2
                return QuantizedTensor(scheme, 0, cols, np.zeros((0, stride), np.uint8), np.zeros((0, G), np.float32),
                                       None if scheme.symmetric else np.zeros((0, G), np.uint8))
            codes = read_tensor(jt, prefix + "_codes")
            scales = read_tensor(jt, prefix + "_scales").astype(np.float32, copy=False)
            zp = None if scheme.symmetric else read_tensor(jt, prefix + "_zero_points").astype(np.uint8, copy=False)
            return QuantizedTensor(scheme, rows, cols, np.ascontiguousarray(codes.reshape(rows, -1)),
                                   np.ascontiguousarray(scales), None if zp is None else np.ascontiguousarray(zp))

        for jl in j["layers"]:
            name = str(jl["name"])
            N, K = int(jl["out_features"]), int(jl["in_features"])
            m8 = np.asarray(jl["index_map8"], np.int32)
            m4 = np.asarray(jl["index_map4"], np.int32)
            jt = jl["tensors"]
            layer = MixedLinearLayer(name, N, K, read_sub(jt, name + ".sub8", qm.largebit, m8.size, K),
                                     read_sub(jt, name + ".sub4", qm.smallbit, m4.size, K), m8, m4)
            validate_mixed_layer(layer)
            qm.linears.append(layer)
        return qm
    except (DataError, UsageError):
        raise
    except (KeyError, TypeError, ValueError, json.JSONDecodeError) as e:
        raise DataError(f"malformed quantized manifest '{manifest}': {e}") from None


def load_device_layers(path, device: int = 0, w8_mode: int = capi.MQ_W8_REFERENCE) -> dict:
    """quantized.json -> {layer name: DeviceLayer} (each packed once into HBM)."""
    return {layer.name: DeviceLayer(layer, device, w8_mode=w8_mode) for layer in load_quantized_model(path).linears}


def validate_mixed_layer(layer: MixedLinearLayer) -> None:
    check(lib().mq_validate_layer(C.byref(layer.desc())))


def prepack_weights(layer: MixedLinearLayer, which: int) -> np.ndarray:
    """prepack_weights (gemm.cpp:89-108) of sub8 (which=0) / sub4 (which=1)."""
    rows = layer.sub8.rows if which == 0 else layer.sub4.rows
    out = np.zeros(rows * layer.in_features, np.uint8)
    check(lib().mq_prepack_reference(C.byref(layer.desc()), which, _p(out)))
    return out


def reassemble_output(y8, y4, map8, map4, out_features: int) -> np.ndarray:
    """reassemble_output (mixed.cpp:83-120) on host arrays."""
    y8 = np.ascontiguousarray(y8, np.float32)
    y4 = np.ascontiguousarray(y4, np.float32)
    map8 = np.ascontiguousarray(map8, np.int32)
    map4 = np.ascontiguousarray(map4, np.int32)
    if y8.shape[1] != map8.size or y4.shape[1] != map4.size:
        raise UsageError("reassemble_output: column counts do not match index maps")
    M = max(y8.shape[0], y4.shape[0])
    out = np.zeros((M, out_features), np.float32)
    check(lib().mq_reassemble_output(_p(y8), map8.size, _p(y4), map4.size, _p(map8), _p(map4), M, out_features,
                                     _p(out)))
    return out


def shard_plan(layer: MixedLinearLayer, world: int):
    """Output-feature column-sharding plan, host only: returns
    (shard_cols, colmap [world, shard_cols]) — rank r's local column j is
    original column colmap[r, j] (-1 = padding)."""
    d = layer.desc()
    sc = C.c_int64()
    check(lib().mq_shard_plan(C.byref(d), world, C.byref(sc), None))
    out = np.zeros(world * sc.value, np.int32)
    check(lib().mq_shard_plan(C.byref(d), world, C.byref(sc), _p(out)))
    return sc.value, out.reshape(world, sc.value)


def bench_inputs(m: int, n: int, k: int, percent: float, seed: int = 1):
    """run_bench's synthetic inputs (gemm.cpp:211-227), byte-for-byte."""
    W = np.empty((n, k), np.float64)
    A = np.empty((m, k), np.float32)
    prom = np.empty(max(n, 1), np.int32)
    cnt = lib().mq_bench_inputs(m, n, k, percent, seed, _p(W), _p(A), _p(prom))
    return W, A, prom[:cnt].copy()


# ------------------------------------------------------------ device engine
_DT = {"float32": capi.MQ_F32, "float16": capi.MQ_F16, "bfloat16": capi.MQ_BF16}


def _dt(t) -> int:
    return _DT[str(t.dtype).replace("torch.", "")]


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def exec_opts(mode: int = capi.MQ_EXACT, act_group: int = 0, ksplit: int = 0, token_tile: int = 0,
              gemm_impl: int = 0, pdl: bool = True, schedule: int = 0, concurrent: bool = False,
              act_scale_f16: bool = False, prefetch_next: "DeviceLayer | None" = None,
              prefetch_bytes: int = 0) -> capi.mq_exec_opts:
    """mq_exec_opts (capi.h). prefetch_next: the DeviceLayer this stream runs next
    (its weights are prefetched into L2 at the end of this launch's reads)."""
    return capi.mq_exec_opts(mode, act_group, ksplit, token_tile, gemm_impl, 0 if pdl else 1, schedule,
                             int(concurrent), int(act_scale_f16),
                             prefetch_next.h.value if prefetch_next is not None else None, prefetch_bytes)


class DeviceLayer:
    """A mixed layer packed once into the engine's HBM layout (mq_layer_create)."""

    def __init__(self, layer: MixedLinearLayer, device: int = 0, w8_mode: int = capi.MQ_W8_REFERENCE,
                 rank: int = 0, world: int = 1):
        self.layer = layer
        opts = capi.mq_layer_opts(w8_mode, rank, world)
        h = C.c_void_p()
        check(lib().mq_layer_create(C.byref(layer.desc()), C.byref(opts), device, C.byref(h)))
        self.h = h
        self.device = device
        self.info = capi.mq_layer_info()
        check(lib().mq_layer_get_info(h, C.byref(self.info)))
        self._ws = {}

    @classmethod
    def from_device(cls, dq: "DeviceQuantizedLayer", device: int | None = None, w8_mode: int = capi.MQ_W8_REFERENCE,
                    rank: int = 0, world: int = 1, stream=None) -> "DeviceLayer":
        """mq_layer_create_device: pack the engine layout on the GPU from a
        device-quantized layer (no host round trip)."""
        self = cls.__new__(cls)
        self.layer = None
        self.device = dq.device if device is None else device
        opts = capi.mq_layer_opts(w8_mode, rank, world)
        h = C.c_void_p()
        check(lib().mq_layer_create_device(C.byref(dq.d), C.byref(opts), self.device, _stream(stream), C.byref(h)))
        self.h = h
        self.info = capi.mq_layer_info()
        check(lib().mq_layer_get_info(h, C.byref(self.info)))
        self._ws = {}
        return self

    @classmethod
    def replicas(cls, layer: MixedLinearLayer, n: int, device: int = 0, w8_mode: int = capi.MQ_W8_REFERENCE,
                 rank: int = 0, world: int = 1) -> list:
        """n independent device copies of one layer: the reference layouts are
        uploaded once and each copy is packed on the GPU (mq_layer_create_device)
        — benchmarks rotate copies so the weights stream from HBM, not L2."""
        import torch
        dv = f"cuda:{device}"
        keep = [torch.from_numpy(np.ascontiguousarray(a)).to(dv) for a in
                (layer.sub8.payload, layer.sub8.scales, layer.sub4.payload, layer.sub4.scales,
                 layer.sub4.zero_points if layer.sub4.zero_points is not None else np.zeros((1,), np.uint8))]
        d = layer.desc()  # host maps (kept alive by `layer`)
        (d.payload8, d.scales8, d.payload4, d.scales4, d.zero_points4) = [t.data_ptr() for t in keep]
        out = []
        for _ in range(n):
            self = cls.__new__(cls)
            self.layer, self.device, self._ws = layer, device, {}
            h = C.c_void_p()
            check(lib().mq_layer_create_device(C.byref(d), C.byref(capi.mq_layer_opts(w8_mode, rank, world)), device,
                                               None, C.byref(h)))
            self.h = h
            self.info = capi.mq_layer_info()
            check(lib().mq_layer_get_info(h, C.byref(self.info)))
            out.append(self)
        return out

    def export_packed(self):
        """(packed engine layout bytes, tile-row column map) copied to host."""
        wq = np.zeros(self.info.device_bytes, np.uint8)
        cm = np.zeros((self.info.tiles8 + self.info.tiles4) * 128, np.int32)
        check(lib().mq_layer_export_packed(self.h, _p(wq), wq.nbytes, _p(cm)))
        return wq, cm

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            try:
                lib().mq_layer_destroy(h)
            except Exception:  # interpreter shutdown: module globals already gone
                pass
            self.h = None

    @property
    def out_cols(self) -> int:
        return self.info.shard_cols if self.info.world > 1 else self.info.out_features

    def shard_colmap(self) -> np.ndarray:
        out = np.zeros(self.info.world * self.info.shard_cols, np.int32)
        check(lib().mq_layer_shard_colmap(self.h, _p(out)))
        return out

    def workspace(self, M: int, opts: capi.mq_exec_opts, full: bool = True):
        import torch
        n = (lib().mq_mixed_linear_workspace_bytes if full else lib().mq_forward_workspace_bytes)(
            self.h, M, C.byref(opts))
        key = (full, n)
        if key not in self._ws:
            self._ws[key] = torch.zeros(max(int(n), 16), dtype=torch.uint8, device=f"cuda:{self.device}")
        return self._ws[key]

    def forward(self, A, out=None, out_dtype=None, opts: capi.mq_exec_opts | None = None, err=None,
                stream=None, workspace=None):
        """execute_mixed_linear on device: A [M, K] f32/f16/bf16 (torch cuda)."""
        import torch
        opts = opts or exec_opts()
        M = A.shape[0]
        if out is None:
            out = torch.empty((M, self.out_cols), dtype=out_dtype or torch.float32, device=A.device)
        if opts.gemm_impl == 1:  # SIMT debug kernel: takes reference-layout codes
            ag = opts.act_group or self.info.group_size
            codes, scales = quantize_act(A, ag, err=err, stream=stream)
            return self.forward_codes(codes, scales, out=out, opts=opts, stream=stream)
        ws = workspace if workspace is not None else self.workspace(M, opts, True)
        check(lib().mq_mixed_linear(self.h, _p(A), _dt(A), M, _p(out), _dt(out), C.byref(opts), _p(ws),
                                    _p(err), _stream(stream)))
        return out

    def forward_codes(self, codes, scales, out=None, out_dtype=None, opts: capi.mq_exec_opts | None = None,
                      stream=None, workspace=None):
        """execute_mixed_on_codes on device: codes int8 [M, ldc], scales f32
        group-major [G, lds] (as quantize_act returns them)."""
        import torch
        opts = opts or exec_opts()
        M = codes.shape[0]
        if out is None:
            out = torch.empty((M, self.out_cols), dtype=out_dtype or torch.float32, device=codes.device)
        ws = workspace if workspace is not None else self.workspace(M, opts, False)
        lds = scales.stride(0) if scales.dim() == 2 else scales.numel()
        check(lib().mq_mixed_linear_codes(self.h, _p(codes), codes.stride(0), _p(scales), lds, M, _p(out),
                                          _dt(out), C.byref(opts), _p(ws), _stream(stream)))
        return out

    def quantize_ws(self, A, opts: capi.mq_exec_opts | None = None, err=None, stream=None, workspace=None):
        """K1 into the engine activation layout inside a workspace (mq_quantize_act_ws);
        returns the workspace, to be consumed by forward_ws (one or many layers)."""
        opts = opts or exec_opts()
        ws = workspace if workspace is not None else self.workspace(A.shape[0], opts, True)
        check(lib().mq_quantize_act_ws(self.h, _p(A), _dt(A), A.shape[0], C.byref(opts), _p(ws), _p(err),
                                       _stream(stream)))
        return ws

    def forward_ws(self, M: int, ws, out=None, out_dtype=None, opts: capi.mq_exec_opts | None = None, stream=None):
        """K2 alone on activations quantize_ws left in `ws` (mq_mixed_linear_ws)."""
        import torch
        opts = opts or exec_opts()
        if out is None:
            out = torch.empty((M, self.out_cols), dtype=out_dtype or torch.float32, device=ws.device)
        check(lib().mq_mixed_linear_ws(self.h, M, _p(ws), _p(out), _dt(out), C.byref(opts), _stream(stream)))
        return out

    def forward_allgather(self, A, comm: "NcclComm", out=None, out_dtype=None, opts: capi.mq_exec_opts | None = None,
                          err=None, stream=None):
        """Column-sharded forward (mq_mixed_linear_allgather): this rank's shard,
        NCCL all-gather of every rank's block on `comm`, permute to the original
        column order. Returns the full Y [M, out_features]."""
        import torch
        opts = opts or exec_opts()
        M = A.shape[0]
        dt = out_dtype or (out.dtype if out is not None else torch.float32)
        if out is None:
            out = torch.empty((M, self.info.out_features), dtype=dt, device=A.device)
        n = lib().mq_mixed_linear_allgather_workspace_bytes(self.h, M, C.byref(opts), _dt(out))
        key = ("ag", int(n))
        if key not in self._ws:
            self._ws[key] = torch.zeros(max(int(n), 16), dtype=torch.uint8, device=A.device)
        check(lib().mq_mixed_linear_allgather(self.h, _p(A), _dt(A), M, _p(out), _dt(out), C.byref(opts),
                                              _p(self._ws[key]), _p(err), comm.ptr, _stream(stream)))
        return out

    def forward_peers(self, A, y_peers, opts: capi.mq_exec_opts | None = None, err=None, stream=None,
                      workspace=None):
        """Fused gather (mq_mixed_linear_peers): the epilogue writes this shard's
        outputs into every tensor of y_peers ([M, out_features] each, one per rank,
        peer-accessible) at the original columns."""
        opts = opts or exec_opts()
        M = A.shape[0]
        ptrs = (P * len(y_peers))(*[t.data_ptr() for t in y_peers])
        ws = workspace if workspace is not None else self.workspace(M, opts, True)
        check(lib().mq_mixed_linear_peers(self.h, _p(A), _dt(A), M, ptrs, len(y_peers), _dt(y_peers[0]),
                                          C.byref(opts), _p(ws), _p(err), _stream(stream)))
        return y_peers

    def partials(self, codes, which: int, stream=None):
        import torch
        M = codes.shape[0]
        rows = self.info.n8 if which == 0 else self.info.n4
        G = (self.info.in_features + self.info.group_size - 1) // self.info.group_size
        out = torch.zeros((G, M, rows), dtype=torch.int32, device=codes.device)
        check(lib().mq_gemm_partials(self.h, _p(codes), codes.stride(0), M, which, _p(out), _stream(stream)))
        return out


class NcclComm:
    """An NCCL communicator for the sharded forwards, bound through the engine's
    run-time NCCL binding (capi.h: mq_nccl_*). `create` makes a new one from a
    shared unique id; `from_torch` borrows a torch ProcessGroupNCCL's (the same
    NCCL library is used, so the handle is valid for the engine)."""

    def __init__(self, ptr, owned: bool):
        self.ptr = C.c_void_p(ptr) if not isinstance(ptr, C.c_void_p) else ptr
        self.owned = owned

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().mq_nccl_unique_id(buf))
        return bytes(buf)

    @classmethod
    def create(cls, uid: bytes, world: int, rank: int, device: int) -> "NcclComm":
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        check(lib().mq_nccl_comm_init(buf, world, rank, device, C.byref(h)))
        return cls(h, True)

    @classmethod
    def from_torch(cls, group=None, device=None) -> "NcclComm":
        import torch
        import torch.distributed as dist
        pg = group or dist.group.WORLD
        be = pg._get_backend(torch.device("cuda", torch.cuda.current_device() if device is None else device))
        return cls(be._comm_ptr(), False)

    def __del__(self):
        if getattr(self, "owned", False) and self.ptr:
            try:
                lib().mq_nccl_comm_destroy(self.ptr)
            except Exception:
                pass
            self.owned = False


def peer_barrier(flags, world: int, rank: int, epoch: int, stream=None) -> None:
    """mq_peer_barrier: flags = per-rank uint32 [world] tensors (peer-mapped)."""
    ptrs = (P * len(flags))(*[t.data_ptr() for t in flags])
    check(lib().mq_peer_barrier(ptrs, world, rank, epoch, _stream(stream)))


def quantize_act(A, group_size: int, ldc: int | None = None, err=None, stream=None, scale_f16: bool = False):
    """Activation quantization on device: returns (codes int8 [M, ldc],
    scales f32 group-major [G, lds]; G = 1 for per-token). scales[:, :M].T is
    the reference's [M, G] array. scale_f16: the scheme's scale_f16_storage."""
    import torch
    M, K = A.shape
    if scale_f16:
        ldc = ldc or (K + 127) // 128 * 128
        codes = torch.empty((M, ldc), dtype=torch.int8, device=A.device)
        G = 1 if group_size >= K else (K + group_size - 1) // group_size
        lds = (M + 3) // 4 * 4
        scales = torch.empty((G, lds), dtype=torch.float32, device=A.device)
        sc = capi.mq_scheme(8, 1, group_size, 1)
        check(lib().mq_quantize_act_scheme(_p(A), _dt(A), M, K, A.stride(0), C.byref(sc), _p(codes), ldc,
                                           _p(scales), lds, _p(err), _stream(stream)))
        return codes, scales
    ldc = ldc or (K + 127) // 128 * 128
    codes = torch.empty((M, ldc), dtype=torch.int8, device=A.device)
    G = 1 if group_size >= K else (K + group_size - 1) // group_size
    lds = (M + 3) // 4 * 4
    scales = torch.empty((G, lds), dtype=torch.float32, device=A.device)
    check(lib().mq_quantize_act(_p(A), _dt(A), M, K, A.stride(0), group_size, _p(codes), ldc, _p(scales), lds,
                                _p(err), _stream(stream)))
    return codes, scales


def permute_gathered(gathered, colmap_dev, world: int, shard_cols: int, M: int, N: int, out=None, stream=None):
    import torch
    if out is None:
        out = torch.empty((M, N), dtype=gathered.dtype, device=gathered.device)
    check(lib().mq_permute_gathered(_p(gathered), _p(colmap_dev), world, shard_cols, M, N, _p(out), _dt(out),
                                    _stream(stream)))
    return out


# ----------------------------------------------- reference-shaped drop-ins
def execute_mixed_linear(activations: np.ndarray, layer: MixedLinearLayer, act_scheme: QuantScheme = ACT_SCHEME,
                         mode: int = capi.MQ_EXACT, w8_mode: int = capi.MQ_W8_REFERENCE,
                         device: int = 0) -> np.ndarray:
    """execute_mixed_linear (gemm.cpp:183-192): host f32 in, host f32 out,
    computed on the B200 (synchronous, like the reference)."""
    import torch
    if act_scheme.bit_width != 8 or not act_scheme.symmetric:
        raise UsageError("activation scheme must be 8-bit symmetric")
    A = np.ascontiguousarray(activations, np.float32)
    if A.shape[1] != layer.in_features:
        raise UsageError("activation K does not match the layer's in_features")
    dl = DeviceLayer(layer, device, w8_mode)
    err = torch.full((1,), 2**31 - 1, dtype=torch.int32, device=f"cuda:{device}")
    Y = dl.forward(torch.from_numpy(A).to(f"cuda:{device}"),
                   opts=exec_opts(mode, act_scheme.group_size, act_scale_f16=act_scheme.scale_f16_storage), err=err)
    torch.cuda.synchronize(device)
    e = int(err.item())
    if e != 2**31 - 1:
        G = (layer.in_features + act_scheme.group_size - 1) // act_scheme.group_size
        raise DataError(f"row {e // G}, group {e % G}: quantize: non-finite input value")
    return Y.cpu().numpy()


def run_bench(m: int, n: int, k: int, percent: float = 0.1, group_size: int = 128, repeats: int = 3,
              seed: int = 1, mode: int = capi.MQ_EXACT, device: int = 0) -> dict:
    """run_bench (gemm.cpp:206-259) on the B200: same generator, same
    checksum definition (FNV-1a over the f32 output), CUDA-event timing of
    the device forward (activation quantization + GEMM + scatter)."""
    import torch
    W, A, prom = bench_inputs(m, n, k, percent, seed)
    layer = partition_and_quantize(W, prom, QuantScheme(8, True, group_size), QuantScheme(4, False, group_size), "bench")
    dl = DeviceLayer(layer, device)
    dA = torch.from_numpy(A).to(f"cuda:{device}")
    opts = exec_opts(mode, group_size)
    Y = dl.forward(dA, opts=opts)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(repeats):
        dl.forward(dA, out=Y, opts=opts)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / repeats
    out = Y.cpu().numpy()
    return dict(m=m, n=n, k=k, percent=percent, group_size=group_size, repeats=repeats, wall_ms=ms,
                gops=2.0 * m * n * k / (ms * 1e6), checksum=fnv1a_hex(out))
