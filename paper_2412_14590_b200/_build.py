"""In-tree build of libmixllm_b200.so (sm_100a only).

Kernels: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo (no fast
math; the activation quantizer and the exact-mode epilogue rely on IEEE
division/rounding intrinsics). Host: g++ -O2 -ffp-contract=off (bit-exact host
quantizers). Output: paper_2412_14590_b200/libmixllm_b200.so.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_obj")
LIB = os.path.join(PKG, "libmixllm_b200.so")
TEST_BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "test_dropin")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INC = ["-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "-I" + os.path.join(CUDA, "include")]

CU_SRCS = ["kernels/act_quant.cu", "kernels/mixed_gemm_sm100.cu", "kernels/mixed_gemm_peers.cu",
           "kernels/mixed_gemm_simt.cu", "kernels/weight_quant.cu"]
CPP_SRCS = ["host/mq_host.cpp", "host/mq_layer.cpp", "host/mq_nccl.cpp"]


def _deps() -> list[str]:
    out = []
    for d, _, fs in os.walk(CSRC):
        out += [os.path.join(d, f) for f in fs if f.endswith((".cuh", ".hpp", ".h"))]
    out.append(os.path.join(ROOT, "include", "mixllm", "capi.h"))
    return out


def _stale(target: str, srcs: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in srcs)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {cmd[0]} {cmd[-1]}")


def build(verbose: bool = False, force: bool = False, defines: tuple = (), lib: str | None = None,
          obj: str | None = None) -> str:
    """defines/lib/obj: development variants (e.g. -DMQ_NS_MAX=12) built beside the product library."""
    lib_path = lib or LIB
    obj_dir = obj or OBJ
    os.makedirs(obj_dir, exist_ok=True)
    deps = _deps()
    objs, jobs = [], []
    for src in CU_SRCS:
        s = os.path.join(CSRC, src)
        o = os.path.join(obj_dir, os.path.basename(src) + ".o")
        objs.append(o)
        if force or _stale(o, [s] + deps):
            jobs.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *defines,
                         "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3",
                         *INC, "-c", s, "-o", o])
    if jobs:  # the kernel translation units compile in parallel
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(len(jobs)) as ex:
            list(ex.map(_run, jobs))
    for src in CPP_SRCS:
        s = os.path.join(CSRC, src)
        o = os.path.join(obj_dir, os.path.basename(src) + ".o")
        objs.append(o)
        if force or _stale(o, [s] + deps):
            _run(["g++", *defines, "-std=gnu++20", "-O2", "-ffp-contract=off", "-fPIC", "-Wall", "-Wno-unused-function",
                  *INC, "-c", s, "-o", o])
    if force or _stale(lib_path, objs):
        _run([NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", lib_path, *objs,
              "-L" + os.path.join(CUDA, "lib64"), "-lcudart_static", "-ldl", "-lrt", "-lpthread"])
    # the C++ drop-in test driver (reference call shapes over include/mixllm/mixquant.hpp)
    tsrc = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
    if lib is not None:
        return lib_path
    if os.path.exists(tsrc):
        os.makedirs(os.path.dirname(TEST_BIN), exist_ok=True)
        if force or _stale(TEST_BIN, [tsrc, LIB, os.path.join(ROOT, "include", "mixllm", "mixquant.hpp")]):
            _run(["g++", "-std=gnu++20", "-O2", "-Wall", *INC, tsrc, "-o", TEST_BIN, "-L" + PKG, "-lmixllm_b200",
                  "-Wl,-rpath," + PKG, "-L" + os.path.join(CUDA, "lib64"), "-lcudart_static", "-ldl", "-lrt",
                  "-lpthread"])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
