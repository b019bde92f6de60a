"""ctypes bindings for the CPU oracle (oracle/_build/libmqo.so) and the
reference build (oracle/_ref/libmqref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, always as the checker or the
CPU baseline, never as the measured GPU product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
MQO_SO = os.path.join(HERE, "_build", "libmqo.so")
REF_SO = os.path.join(HERE, "_ref", "libmqref.so")

_P = C.c_void_p
_I64 = C.c_int64


def build(ref: bool | None = None) -> None:
    """Compile the oracle (and the reference, when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref is None:
        ref = os.path.isdir("/root/reference/proj")
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(_P)


_mqo = None
_ref = None


def mqo():
    global _mqo
    if _mqo is None:
        if not os.path.exists(MQO_SO):
            build(ref=False)
        lib = C.CDLL(MQO_SO)
        lib.mqo_fast_i2f.restype = C.c_float
        lib.mqo_fast_i2f.argtypes = [C.c_int32]
        lib.mqo_round_scale_f16.restype = C.c_float
        lib.mqo_round_scale_f16.argtypes = [C.c_float]
        lib.mqo_fnv1a.restype = C.c_uint64
        lib.mqo_fnv1a.argtypes = [_P, C.c_uint64]
        lib.mqo_bench_inputs.restype = _I64
        lib.mqo_bench_inputs.argtypes = [_I64, _I64, _I64, C.c_double, C.c_uint64, _P, _P, _P]
        for fn in ("mqo_quantize_tensor_f32", "mqo_quantize_tensor_f64"):
            getattr(lib, fn).argtypes = [_P, _I64, _I64, C.c_int, C.c_int, C.c_int, C.c_int,
                                         _P, _P, _P, _P, _P]
        lib.mqo_partition_maps.argtypes = [_I64, _P, _I64, _P, _P, _P, _P]
        lib.mqo_prepack.argtypes = [_P, C.c_int, C.c_int, _I64, _I64, C.c_int, _P]
        lib.mqo_gemm_sub.argtypes = [_P, _P, _I64, _I64, _I64, C.c_int, _P, C.c_int, C.c_int,
                                     _P, _P, _I64, C.c_int, C.c_int, _P]
        lib.mqo_group_partials.argtypes = [_P, _I64, _I64, C.c_int, _P, C.c_int, C.c_int, _P,
                                           _I64, C.c_int, _P]
        lib.mqo_reassemble.argtypes = [_P, _I64, _P, _I64, _P, _P, _I64, _I64, _P]
        lib.mqo_pack_nibbles.argtypes = [_P, _I64, _P]
        lib.mqo_unpack_nibbles.argtypes = [_P, _I64, _I64, _P]
        for fn in ("mqo_quant_group_sym_f64", "mqo_quant_group_sym_f32"):
            getattr(lib, fn).argtypes = [_P, _I64, C.c_int, C.c_int, _P, _P]
        for fn in ("mqo_quant_group_asym_f64", "mqo_quant_group_asym_f32"):
            getattr(lib, fn).argtypes = [_P, _I64, C.c_int, C.c_int, _P, _P, _P]
        lib.mqo_rng_uniform_int.restype = _I64
        lib.mqo_rng_uniform_int.argtypes = [_P, _I64, _I64]
        lib.mqo_rng_seed.argtypes = [_P, C.c_uint64]
        lib.mqo_rng_next.restype = C.c_uint64
        lib.mqo_rng_next.argtypes = [_P]
        lib.mqo_rng_normal.restype = C.c_double
        lib.mqo_rng_normal.argtypes = [_P]
        _mqo = lib
    return _mqo


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        lib.mqref_last_error.restype = C.c_char_p
        lib.mqref_run_bench.argtypes = [_I64, _I64, _I64, C.c_double, C.c_int, C.c_int, C.c_int,
                                        C.c_int, C.c_uint64, _P, _P, C.c_char_p]
        lib.mqref_layer_create.argtypes = [_P, _I64, _I64, _P, _I64, C.c_int, _P]
        lib.mqref_layer_destroy.argtypes = [_P]
        lib.mqref_layer_dims.argtypes = [_P, _P, _P]
        lib.mqref_layer_export.argtypes = [_P, _P, _P, _P, _P, _P, _P, _P]
        lib.mqref_layer_prepack.argtypes = [_P, C.c_int, _P]
        lib.mqref_layer_forward.argtypes = [_P, _P, _I64, C.c_int, C.c_int, _P, _P]
        lib.mqref_layer_forward_f16.argtypes = [_P, _P, _I64, C.c_int, C.c_int, C.c_int, _P, _P]
        lib.mqref_quantize_tensor.argtypes = [_P, C.c_int, _I64, _I64, C.c_int, C.c_int, C.c_int,
                                              C.c_int, _P, _P, _P]
        lib.mqref_fast_i2f.restype = C.c_float
        lib.mqref_fast_i2f.argtypes = [C.c_int32]
        _ref = lib
    return _ref


def fnv1a_hex(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return "%016x" % mqo().mqo_fnv1a(_ptr(a), a.nbytes)


# ------------------------------------------------------------------ inputs
def bench_inputs(m: int, n: int, k: int, percent: float, seed: int = 1):
    """run_bench's generator (proj/src/gemm.cpp:211-227): W f64, A f32, promoted."""
    W = np.empty((n, k), np.float64)
    A = np.empty((m, k), np.float32)
    prom = np.empty(max(n, 1), np.int32)
    cnt = mqo().mqo_bench_inputs(m, n, k, percent, seed, _ptr(W), _ptr(A), _ptr(prom))
    return W, A, prom[:cnt].copy()


def normal_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """random_matrix of proj/tests/test_util.hpp:70-77 (Xoshiro normals, row-major)."""
    st = (C.c_uint64 * 6)()
    lib = mqo()
    lib.mqo_rng_seed(C.cast(st, _P), seed)
    out = np.empty((rows, cols), np.float64)
    flat = out.reshape(-1)
    for i in range(flat.size):
        flat[i] = lib.mqo_rng_normal(C.cast(st, _P))
    return out


# ------------------------------------------------------------- quantizers
def quant_group_sym(x, bits: int, f16: bool = False):
    """quantize_group_sym<double|float> (quant.hpp:117-140): (codes int8, scale f32)."""
    x = np.ascontiguousarray(x)
    codes = np.zeros(max(x.size, 1), np.int8)
    sc = np.zeros(1, np.float32)
    fn = mqo().mqo_quant_group_sym_f64 if x.dtype == np.float64 else mqo().mqo_quant_group_sym_f32
    st = fn(_ptr(x), x.size, bits, int(f16), _ptr(codes), _ptr(sc))
    if st:
        raise OracleError(st, "group quantization")
    return codes[: x.size], sc[0]


def quant_group_asym(x, bits: int, f16: bool = False):
    """quantize_group_asym<double|float> (quant.hpp:84-112): (codes u8, scale f32, zero point)."""
    x = np.ascontiguousarray(x)
    codes = np.zeros(max(x.size, 1), np.uint8)
    sc = np.zeros(1, np.float32)
    zp = np.zeros(1, np.uint8)
    fn = mqo().mqo_quant_group_asym_f64 if x.dtype == np.float64 else mqo().mqo_quant_group_asym_f32
    st = fn(_ptr(x), x.size, bits, int(f16), _ptr(codes), _ptr(sc), _ptr(zp))
    if st:
        raise OracleError(st, "group quantization")
    return codes[: x.size], sc[0], int(zp[0])


class Rng:
    """Xoshiro256pp (rng.hpp:29-82) — the reference tests' generator."""

    def __init__(self, seed: int):
        self.st = (C.c_uint64 * 6)()
        mqo().mqo_rng_seed(C.cast(self.st, _P), seed)

    def normal(self) -> float:
        return mqo().mqo_rng_normal(C.cast(self.st, _P))

    def uniform_int(self, lo: int, hi: int) -> int:
        return mqo().mqo_rng_uniform_int(C.cast(self.st, _P), lo, hi)


@dataclass
class QTensor:
    bits: int
    sym: bool
    group: int
    rows: int
    cols: int
    payload: np.ndarray  # u8 [rows, stride]
    scales: np.ndarray   # f32 [rows, G]
    zps: np.ndarray | None  # u8 [rows, G]

    @property
    def G(self) -> int:
        return 0 if self.cols == 0 else (self.cols + self.group - 1) // self.group

    def codes(self) -> np.ndarray:
        """Raw codes [rows, cols] (int32): unsigned for asym, signed for sym."""
        if self.bits == 4:
            lo = (self.payload & 0x0F).astype(np.int32)
            hi = (self.payload >> 4).astype(np.int32)
            c = np.stack([lo, hi], axis=-1).reshape(self.rows, -1)[:, : self.cols]
            return c
        if self.sym:
            return self.payload.view(np.int8).astype(np.int32)
        return self.payload.astype(np.int32)


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"status {status}: {msg}")
        self.status = status


def quantize_tensor(m: np.ndarray, bits: int, sym: bool, group: int, f16: bool = False) -> QTensor:
    """quantize_tensor<Scalar> (quant.hpp:183-243) in the oracle; Scalar from dtype."""
    m = np.ascontiguousarray(m)
    rows, cols = m.shape
    G = 0 if cols == 0 else (cols + group - 1) // group
    stride = (cols + 1) // 2 if bits == 4 else cols
    payload = np.zeros((rows, stride), np.uint8)
    scales = np.zeros((rows, G), np.float32)
    zps = None if sym else np.zeros((rows, G), np.uint8)
    er = np.zeros(2, np.int64)
    fn = mqo().mqo_quantize_tensor_f64 if m.dtype == np.float64 else mqo().mqo_quantize_tensor_f32
    if m.dtype not in (np.float64, np.float32):
        raise TypeError(m.dtype)
    st = fn(_ptr(m), rows, cols, bits, int(sym), group, int(f16), _ptr(payload), _ptr(scales),
            _ptr(zps), _ptr(er[:1]), _ptr(er[1:]))
    if st:
        raise OracleError(st, f"row {er[0]}, group {er[1]}")
    return QTensor(bits, sym, group, rows, cols, payload, scales, zps)


@dataclass
class Layer:
    N: int
    K: int
    group: int
    map8: np.ndarray
    map4: np.ndarray
    sub8: QTensor
    sub4: QTensor


def partition_and_quantize(W: np.ndarray, promoted, group: int = 128) -> Layer:
    """partition_and_quantize (mixed.cpp:46-81) with {8,sym,g} / {4,asym,g}."""
    N, K = W.shape
    promoted = np.ascontiguousarray(np.asarray(promoted, np.int32))
    map8 = np.zeros(max(N, 1), np.int32)
    map4 = np.zeros(max(N, 1), np.int32)
    n8 = np.zeros(1, np.int64)
    n4 = np.zeros(1, np.int64)
    st = mqo().mqo_partition_maps(N, _ptr(promoted), promoted.size, _ptr(map8), _ptr(n8),
                                  _ptr(map4), _ptr(n4))
    if st:
        raise OracleError(st, "bad promoted list")
    map8 = map8[: n8[0]].copy()
    map4 = map4[: n4[0]].copy()
    W = np.ascontiguousarray(W, np.float64)
    sub8 = quantize_tensor(W[map8], 8, True, group)
    sub4 = quantize_tensor(W[map4], 4, False, group)
    return Layer(N, K, group, map8, map4, sub8, sub4)


def prepack(q: QTensor) -> np.ndarray:
    out = np.zeros(q.rows * q.cols, np.uint8)
    mqo().mqo_prepack(_ptr(q.payload), q.bits, int(q.sym), q.rows, q.cols, q.group, _ptr(out))
    return out


def quantize_acts(A: np.ndarray, group: int, f16: bool = False):
    """Activation quantization {8, sym, group, f16} (gemm.cpp:190); group=K is per-token."""
    q = quantize_tensor(np.ascontiguousarray(A, np.float32), 8, True, group, f16)
    return q.payload.view(np.int8).copy(), q.scales


def gemm_sub(a_codes, a_scales, q: QTensor, fast: bool = True, w8_unsigned: bool = True) -> np.ndarray:
    """gemm_block over one sub-problem; returns f32 [M, rows]. w8_unsigned
    reproduces the reference's uint8 read-back of 8-bit codes (see mqo.h)."""
    a_codes = np.ascontiguousarray(a_codes, np.int8)
    a_scales = np.ascontiguousarray(a_scales, np.float32)
    M, K = a_codes.shape
    out = np.zeros((M, q.rows), np.float32)
    sc = a_scales.shape[1] if a_scales.ndim == 2 else 1
    mqo().mqo_gemm_sub(_ptr(a_codes), _ptr(a_scales), sc, M, K, q.group, _ptr(q.payload), q.bits,
                       int(q.sym), _ptr(q.scales), _ptr(q.zps), q.rows, int(fast), int(w8_unsigned), _ptr(out))
    return out


def group_partials(a_codes, q: QTensor, w8_unsigned: bool = True) -> np.ndarray:
    """int32 S[g, m, r] (step-1 integer group sums)."""
    a_codes = np.ascontiguousarray(a_codes, np.int8)
    M, K = a_codes.shape
    out = np.zeros((q.G, M, q.rows), np.int32)
    mqo().mqo_group_partials(_ptr(a_codes), M, K, q.group, _ptr(q.payload), q.bits, int(q.sym),
                             _ptr(q.zps), q.rows, int(w8_unsigned), _ptr(out))
    return out


def reassemble(y8, y4, map8, map4, N: int) -> np.ndarray:
    y8 = np.ascontiguousarray(y8, np.float32)
    y4 = np.ascontiguousarray(y4, np.float32)
    M = max(y8.shape[0], y4.shape[0])
    out = np.zeros((M, N), np.float32)
    st = mqo().mqo_reassemble(_ptr(y8), y8.shape[1], _ptr(y4), y4.shape[1],
                              _ptr(np.ascontiguousarray(map8, np.int32)),
                              _ptr(np.ascontiguousarray(map4, np.int32)), M, N, _ptr(out))
    if st:
        raise OracleError(st, "bad maps")
    return out


def mixed_linear(layer: Layer, A: np.ndarray, act_group: int | None = None, fast: bool = True,
                 w8_unsigned: bool = True, act_f16: bool = False):
    """execute_mixed_linear (gemm.cpp:183-192). act_group = K selects the
    per-token extension (s_a broadcast across groups); act_f16 the activation
    scheme's scale_f16_storage. Returns (Y, codes, scales)."""
    act_group = layer.group if act_group is None else act_group
    codes, scales = quantize_acts(A, act_group, act_f16)
    y8 = gemm_sub(codes, scales, layer.sub8, fast, w8_unsigned) if layer.sub8.rows else np.zeros((A.shape[0], 0), np.float32)
    y4 = gemm_sub(codes, scales, layer.sub4, fast) if layer.sub4.rows else np.zeros((A.shape[0], 0), np.float32)
    return reassemble(y8, y4, layer.map8, layer.map4, layer.N), codes, scales


# --------------------------------------------------------------- reference
class RefLayer:
    """The reference's own MixedLinearLayer (oracle/_ref/libmqref.so)."""

    def __init__(self, W: np.ndarray, promoted, group: int = 128):
        W = np.ascontiguousarray(W, np.float64)
        promoted = np.ascontiguousarray(np.asarray(promoted, np.int32))
        self.N, self.K = W.shape
        h = C.c_void_p()
        st = ref().mqref_layer_create(_ptr(W), self.N, self.K, _ptr(promoted), promoted.size,
                                      group, C.byref(h))
        if st:
            raise OracleError(st, ref().mqref_last_error().decode())
        self.h = h
        n8 = np.zeros(1, np.int64)
        n4 = np.zeros(1, np.int64)
        ref().mqref_layer_dims(h, _ptr(n8), _ptr(n4))
        self.n8, self.n4 = int(n8[0]), int(n4[0])
        self.group = group

    @classmethod
    def load_quantized(cls, path: str) -> list:
        """The reference's load_quantized_model (mixed.cpp:336-370): one layer per linear."""
        hs = (C.c_void_p * 64)()
        n = C.c_int(0)
        dims = np.zeros(128, np.int64)
        lib = ref()
        lib.mqref_load_quantized.argtypes = [C.c_char_p, _P, C.c_int, _P, _P]
        st = lib.mqref_load_quantized(path.encode(), C.cast(hs, _P), 64, C.byref(n), _ptr(dims))
        if st:
            raise OracleError(st, lib.mqref_last_error().decode())
        out = []
        for i in range(n.value):
            o = cls.__new__(cls)
            o.h = C.c_void_p(hs[i])
            o.N, o.K = int(dims[2 * i]), int(dims[2 * i + 1])
            n8 = np.zeros(1, np.int64)
            n4 = np.zeros(1, np.int64)
            lib.mqref_layer_dims(o.h, _ptr(n8), _ptr(n4))
            o.n8, o.n4 = int(n8[0]), int(n4[0])
            o.group = 128
            out.append(o)
        return out

    def export(self):
        G = (self.K + self.group - 1) // self.group
        map8 = np.zeros(self.n8, np.int32)
        map4 = np.zeros(self.n4, np.int32)
        p8 = np.zeros((self.n8, self.K), np.uint8)
        s8 = np.zeros((self.n8, G), np.float32)
        p4 = np.zeros((self.n4, (self.K + 1) // 2), np.uint8)
        s4 = np.zeros((self.n4, G), np.float32)
        z4 = np.zeros((self.n4, G), np.uint8)
        ref().mqref_layer_export(self.h, _ptr(map8), _ptr(map4), _ptr(p8), _ptr(s8), _ptr(p4),
                                 _ptr(s4), _ptr(z4))
        return dict(map8=map8, map4=map4, p8=p8, s8=s8, p4=p4, s4=s4, z4=z4)

    def prepack(self, which: int) -> np.ndarray:
        rows = self.n8 if which == 0 else self.n4
        out = np.zeros(rows * self.K, np.uint8)
        st = ref().mqref_layer_prepack(self.h, which, _ptr(out))
        if st:
            raise OracleError(st, ref().mqref_last_error().decode())
        return out

    def forward(self, A: np.ndarray, fast: bool = True, workers: int = 1, act_f16: bool = False):
        A = np.ascontiguousarray(A, np.float32)
        out = np.zeros((A.shape[0], self.N), np.float32)
        ms = np.zeros(1, np.float64)
        st = ref().mqref_layer_forward_f16(self.h, _ptr(A), A.shape[0], int(act_f16), int(fast), workers,
                                           _ptr(out), _ptr(ms))
        if st:
            raise OracleError(st, ref().mqref_last_error().decode())
        return out, float(ms[0])

    def __del__(self):
        try:
            ref().mqref_layer_destroy(self.h)
        except Exception:
            pass


def ref_run_bench(m, n, k, percent, group=128, fast=True, workers=1, repeats=1, seed=1):
    wall = np.zeros(1, np.float64)
    gops = np.zeros(1, np.float64)
    cs = C.create_string_buffer(17)
    st = ref().mqref_run_bench(m, n, k, percent, group, int(fast), workers, repeats, seed,
                               _ptr(wall), _ptr(gops), cs)
    if st:
        raise OracleError(st, ref().mqref_last_error().decode())
    return dict(wall_ms=float(wall[0]), gops=float(gops[0]), checksum=cs.value.decode())
