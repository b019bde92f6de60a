"""Write tests/golden/quantized_v1/ with the REFERENCE's own writer
(save_quantized_model, proj/src/mixed.cpp:308-334, compiled into
oracle/_ref/libmqref.so by `make -C oracle ref`). Two layers from the run_bench
generator (seed 1): "blk0.proj" 256x384 with 10% 8-bit rows, and "blk0.pure4"
128x256 with none (an empty sub8 writes no files). Run here (the reference is
not on the GPU box):

    python tests/golden/make_quantized_fixture.py
"""
import ctypes as C
import os
import shutil
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
import oracle_py as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "quantized_v1")
LAYERS = [("blk0.proj", 256, 384, 0.10, 1), ("blk0.pure4", 128, 256, 0.0, 2)]


def main() -> None:
    O.build(ref=True)
    ref = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libmqref.so"))
    ref.mqref_layer_create.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_int,
                                       C.POINTER(C.c_void_p)]
    ref.mqref_save_quantized.argtypes = [C.POINTER(C.c_void_p), C.POINTER(C.c_char_p), C.c_int, C.c_char_p,
                                         C.c_double, C.c_int, C.c_char_p]
    ref.mqref_last_error.restype = C.c_char_p
    import paper_2412_14590_b200 as mq
    hs, names = [], []
    for name, n, k, p, seed in LAYERS:
        W, _, prom = mq.bench_inputs(1, n, k, p, seed)
        W = np.ascontiguousarray(W, np.float64)
        prom = np.ascontiguousarray(np.asarray(prom, np.int32))
        h = C.c_void_p()
        assert ref.mqref_layer_create(W.ctypes.data, n, k, prom.ctypes.data, prom.size, 128, C.byref(h)) == 0
        hs.append(h)
        names.append(name.encode())
    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    arr_h = (C.c_void_p * len(hs))(*[h.value for h in hs])
    arr_n = (C.c_char_p * len(names))(*names)
    st = ref.mqref_save_quantized(arr_h, arr_n, len(hs), b"run_bench-seeded", 0.10, 128, OUT.encode())
    assert st == 0, ref.mqref_last_error()
    print("wrote", OUT, sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
