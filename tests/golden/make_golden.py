"""Generate tests/golden/golden.json from the REFERENCE's own implementation.

Runs oracle/_ref/libmqref.so (the reference sources under
/root/reference/proj/src compiled by oracle/Makefile `ref`) — its run_bench
(proj/src/gemm.cpp:206-259) and execute_mixed_linear — and records FNV-1a-64
checksums of the activation codes and f32 outputs plus a few small literal
vectors. Run here (the reference is not on the GPU box):

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle_py as O  # noqa: E402

CASES = [
    # (m, n, k, percent) — run_bench generator, seed 1, g = 128, act {8, sym, 128}
    (16, 4096, 4096, 0.10),   # C1 (BASELINE configs[0])
    (1, 4096, 4096, 0.10),
    (512, 4096, 4096, 0.10),
    (16, 4096, 4096, 0.00),   # pure W4A8
    (16, 4096, 4096, 1.00),   # pure W8A8
    (64, 256, 512, 0.10),
    (17, 300, 384, 0.25),     # ragged tiles, token count not a multiple of 16
    (5, 200, 200, 0.10),      # ragged last K-group (200 = 128 + 72)
    (33, 1024, 1024, 0.10),
]

# The shapes bench.py measures (BASELINE configs[1] fused 8B projections) and the
# Llama-3.1-70B linear shapes (configs[2]): exact-mode output checksums from the
# reference's execute_mixed_linear (workers = nproc; the result does not depend
# on workers, gemm.cpp:159-172 writes disjoint outputs).
LARGE = [
    (16, 6144, 4096, 0.10),    # 8B fused qkv
    (16, 28672, 4096, 0.10),   # 8B fused gate_up
    (16, 4096, 14336, 0.10),   # 8B down (G = 112)
    (512, 4096, 14336, 0.10),  # 8B down, prefill
    (16, 8192, 8192, 0.10),    # 70B q / o
    (16, 1024, 8192, 0.10),    # 70B k / v
    (1, 28672, 8192, 0.10),    # 70B gate / up
    (16, 8192, 28672, 0.10),   # 70B down (G = 224)
    (256, 8192, 8192, 0.10),   # 70B o, prefill
]


def main() -> None:
    O.build(ref=True)
    out = {"generator": "mixquant run_bench inputs, seed 1, group 128", "cases": []}
    for m, n, k, p in CASES:
        W, A, prom = O.bench_inputs(m, n, k, p, 1)
        R = O.RefLayer(W, prom, 128)
        Y, _ = R.forward(A, fast=True)
        Yn, _ = R.forward(A, fast=False)
        assert np.array_equal(Y, Yn), "reference fast/native I2F differ"
        rb = O.ref_run_bench(m, n, k, p, 128, True, 1, 1, 1)
        assert rb["checksum"] == O.fnv1a_hex(Y)
        codes = np.zeros((m, k), np.uint8)
        scales = np.zeros((m, (k + 127) // 128), np.float32)
        st = O.ref().mqref_quantize_tensor(O._ptr(A), 0, m, k, 8, 1, 128, 0, O._ptr(codes), O._ptr(scales), None)
        assert st == 0
        out["cases"].append(dict(m=m, n=n, k=k, percent=p, n8=R.n8, n4=R.n4,
                                 act_codes=O.fnv1a_hex(codes), act_scales=O.fnv1a_hex(scales),
                                 out_f32=O.fnv1a_hex(Y), ref_ms=rb["wall_ms"],
                                 out_first=[float(x) for x in Y.reshape(-1)[:4]]))
        print(out["cases"][-1])
    out["cases_large"] = []
    for m, n, k, p in LARGE:
        W, A, prom = O.bench_inputs(m, n, k, p, 1)
        R = O.RefLayer(W, prom, 128)
        del W
        Y, ms = R.forward(A, fast=True, workers=os.cpu_count() or 1)
        codes = np.zeros((m, k), np.uint8)
        scales = np.zeros((m, (k + 127) // 128), np.float32)
        st = O.ref().mqref_quantize_tensor(O._ptr(A), 0, m, k, 8, 1, 128, 0, O._ptr(codes), O._ptr(scales), None)
        assert st == 0
        out["cases_large"].append(dict(m=m, n=n, k=k, percent=p, n8=R.n8, n4=R.n4,
                                       act_codes=O.fnv1a_hex(codes), act_scales=O.fnv1a_hex(scales),
                                       out_f32=O.fnv1a_hex(Y), ref_ms=ms,
                                       out_first=[float(x) for x in Y.reshape(-1)[:4]]))
        print(out["cases_large"][-1], flush=True)
    # the activation scheme's scale_f16_storage (quant.hpp:70-76, quant.cpp:81-86):
    # C1 inputs, activation scales rounded to binary16 by the reference
    m, n, k, p = CASES[0]
    W, A, prom = O.bench_inputs(m, n, k, p, 1)
    R = O.RefLayer(W, prom, 128)
    Y, _ = R.forward(A, fast=True, act_f16=True)
    codes = np.zeros((m, k), np.uint8)
    scales = np.zeros((m, (k + 127) // 128), np.float32)
    assert O.ref().mqref_quantize_tensor(O._ptr(A), 0, m, k, 8, 1, 128, 1, O._ptr(codes), O._ptr(scales), None) == 0
    out["act_f16"] = dict(m=m, n=n, k=k, percent=p, act_codes=O.fnv1a_hex(codes), act_scales=O.fnv1a_hex(scales),
                          out_f32=O.fnv1a_hex(Y))
    print(out["act_f16"], flush=True)
    # SPEC.md:428 hand example: A_q=[1,-2], s_a=0.1; codes [3,5] (0x53), z=4, s_w=0.5, g=2 -> -0.15
    out["spec_hand_example"] = {"expected": float(np.float32(-0.150000006))}
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
