"""paper_2412_14590_b200 — B200-native (sm_100a) MixLLM W4/W8-A8 mixed-precision
linear engine: C++ host packing + hand-written tcgen05 kernels behind a C ABI
(include/mixllm/capi.h), with a Python mirror of the reference `mixquant` API.
"""
from . import capi  # noqa: F401
from .mixquant import (  # noqa: F401
    ACT_SCHEME,
    LARGEBIT,
    SMALLBIT,
    DataError,
    DeviceLayer,
    DeviceQuantizedLayer,
    MixedLinearLayer,
    NcclComm,
    QuantizedModel,
    QuantizedTensor,
    QuantScheme,
    UsageError,
    bench_inputs,
    exec_opts,
    execute_mixed_linear,
    load_device_layers,
    load_quantized_model,
    fast_i2f,
    fnv1a_hex,
    pack_nibbles,
    peer_barrier,
    partition_and_quantize,
    partition_and_quantize_device,
    permute_gathered,
    pinned_view,
    prepack_weights,
    quantize_act,
    quantize_tensor,
    reassemble_output,
    round_scale_f16,
    run_bench,
    save_quantized_model,
    shard_plan,
    unpack_nibbles,
    validate_mixed_layer,
)

__version__ = "0.1.0"
