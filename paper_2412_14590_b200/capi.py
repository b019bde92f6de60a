"""ctypes binding of the C ABI declared in include/mixllm/capi.h.

Loads the in-tree libmixllm_b200.so. There is no fallback: if the library is
missing the import fails loudly (build it with __graft_entry__.build() or
`python paper_2412_14590_b200/_build.py`).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MQ_LIB") or os.path.join(_HERE, "libmixllm_b200.so")  # MQ_LIB: development variants

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32

MQ_OK, MQ_USAGE, MQ_DATA, MQ_INTERNAL, MQ_CUDA = range(5)
MQ_F32, MQ_F16, MQ_BF16 = range(3)
MQ_EXACT, MQ_FAST = 0, 1
MQ_W8_REFERENCE, MQ_W8_SIGNED = 0, 1


class mq_scheme(C.Structure):
    _fields_ = [("bit_width", I32), ("symmetric", I32), ("group_size", I32), ("scale_f16_storage", I32)]


class mq_layer_desc(C.Structure):
    _fields_ = [
        ("out_features", I64), ("in_features", I64), ("group_size", I32),
        ("n8", I64), ("n4", I64),
        ("index_map8", P), ("index_map4", P),
        ("payload8", P), ("scales8", P),
        ("payload4", P), ("scales4", P), ("zero_points4", P),
    ]


class mq_layer_opts(C.Structure):
    _fields_ = [("w8_mode", I32), ("rank", I32), ("world", I32)]


class mq_layer_info(C.Structure):
    _fields_ = [
        ("out_features", I64), ("in_features", I64), ("group_size", I32),
        ("n8", I64), ("n4", I64), ("tiles8", I64), ("tiles4", I64),
        ("device_bytes", I64), ("weight_stream_bytes", I64),
        ("rank", I32), ("world", I32), ("shard_cols", I64),
    ]


class mq_exec_opts(C.Structure):
    _fields_ = [("mode", I32), ("act_group", I32), ("ksplit", I32), ("token_tile", I32), ("gemm_impl", I32),
                ("no_pdl", I32), ("schedule", I32), ("concurrent", I32), ("act_scale_f16", I32),
                ("prefetch_next", P), ("prefetch_bytes", I64)]


# name -> (restype, argtypes); mirrors capi.h one to one.
PROTOTYPES = {
    "mq_last_error": (C.c_char_p, []),
    "mq_version": (C.c_char_p, []),
    "mq_quantize_tensor_f32": (C.c_int, [P, I64, I64, C.POINTER(mq_scheme), P, P, P, P, P]),
    "mq_quantize_tensor_f64": (C.c_int, [P, I64, I64, C.POINTER(mq_scheme), P, P, P, P, P]),
    "mq_pack_nibbles": (C.c_int, [P, I64, P]),
    "mq_unpack_nibbles": (C.c_int, [P, I64, I64, P]),
    "mq_round_scale_f16": (C.c_float, [C.c_float]),
    "mq_fast_i2f": (C.c_float, [C.c_int32]),
    "mq_partition_and_quantize": (C.c_int, [P, I64, I64, P, I64, C.POINTER(mq_scheme), C.POINTER(mq_scheme), C.POINTER(P)]),
    "mq_host_layer_desc": (C.c_int, [P, C.POINTER(mq_layer_desc)]),
    "mq_host_layer_destroy": (None, [P]),
    "mq_validate_layer": (C.c_int, [C.POINTER(mq_layer_desc)]),
    "mq_prepack_reference": (C.c_int, [C.POINTER(mq_layer_desc), I32, P]),
    "mq_reassemble_output": (C.c_int, [P, I64, P, I64, P, P, I64, I64, P]),
    "mq_bench_inputs": (I64, [I64, I64, I64, C.c_double, C.c_uint64, P, P, P]),
    "mq_fnv1a": (C.c_uint64, [P, C.c_uint64]),
    "mq_shard_plan": (C.c_int, [C.POINTER(mq_layer_desc), I32, C.POINTER(I64), P]),
    "mq_layer_create": (C.c_int, [C.POINTER(mq_layer_desc), C.POINTER(mq_layer_opts), C.c_int, C.POINTER(P)]),
    "mq_layer_destroy": (None, [P]),
    "mq_layer_get_info": (C.c_int, [P, C.POINTER(mq_layer_info)]),
    "mq_layer_shard_colmap": (C.c_int, [P, P]),
    "mq_quantize_act": (C.c_int, [P, C.c_int, I64, I64, I64, I32, P, I64, P, I64, P, P]),
    "mq_quantize_act_scheme": (C.c_int, [P, C.c_int, I64, I64, I64, C.POINTER(mq_scheme), P, I64, P, I64, P, P]),
    "mq_forward_workspace_bytes": (C.c_size_t, [P, I64, C.POINTER(mq_exec_opts)]),
    "mq_mixed_linear_codes": (C.c_int, [P, P, I64, P, I64, I64, P, C.c_int, C.POINTER(mq_exec_opts), P, P]),
    "mq_mixed_linear": (C.c_int, [P, P, C.c_int, I64, P, C.c_int, C.POINTER(mq_exec_opts), P, P, P]),
    "mq_mixed_linear_workspace_bytes": (C.c_size_t, [P, I64, C.POINTER(mq_exec_opts)]),
    "mq_gemm_partials": (C.c_int, [P, P, I64, I64, I32, P, P]),
    "mq_quantize_act_ws": (C.c_int, [P, P, C.c_int, I64, C.POINTER(mq_exec_opts), P, P, P]),
    "mq_mixed_linear_ws": (C.c_int, [P, I64, P, P, C.c_int, C.POINTER(mq_exec_opts), P]),
    "mq_permute_gathered": (C.c_int, [P, P, I32, I64, I64, I64, P, C.c_int, P]),
    "mq_partition_and_quantize_device": (C.c_int, [P, I64, I64, P, I64, C.POINTER(mq_scheme), C.POINTER(mq_scheme),
                                                   C.c_int, P, C.POINTER(P)]),
    "mq_device_qlayer_desc": (C.c_int, [P, C.POINTER(mq_layer_desc)]),
    "mq_device_qlayer_destroy": (None, [P]),
    "mq_layer_create_device": (C.c_int, [C.POINTER(mq_layer_desc), C.POINTER(mq_layer_opts), C.c_int, P,
                                         C.POINTER(P)]),
    "mq_layer_export_packed": (C.c_int, [P, P, C.c_size_t, P]),
    "mq_nccl_unique_id": (C.c_int, [P]),
    "mq_nccl_comm_init": (C.c_int, [P, I32, I32, C.c_int, C.POINTER(P)]),
    "mq_nccl_comm_destroy": (C.c_int, [P]),
    "mq_mixed_linear_allgather_workspace_bytes": (C.c_size_t, [P, I64, C.POINTER(mq_exec_opts), C.c_int]),
    "mq_mixed_linear_allgather": (C.c_int, [P, P, C.c_int, I64, P, C.c_int, C.POINTER(mq_exec_opts), P, P, P, P]),
    "mq_mixed_linear_peers": (C.c_int, [P, P, C.c_int, I64, C.POINTER(P), I32, C.c_int, C.POINTER(mq_exec_opts), P,
                                        P, P]),
    "mq_peer_barrier": (C.c_int, [C.POINTER(P), I32, I32, C.c_uint32, P]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class MQError(RuntimeError):
    status = MQ_INTERNAL


class UsageError(MQError):
    """mixquant::UsageError (proj/include/mixquant/errors.hpp:9-12), CLI exit 1."""
    status = MQ_USAGE


class DataError(MQError):
    """mixquant::DataError (errors.hpp:14-19), CLI exit 2."""
    status = MQ_DATA


class CudaError(MQError):
    status = MQ_CUDA


def check(st: int) -> None:
    if st == MQ_OK:
        return
    msg = lib().mq_last_error().decode()
    cls = {MQ_USAGE: UsageError, MQ_DATA: DataError, MQ_CUDA: CudaError}.get(st, MQError)
    raise cls(msg)
