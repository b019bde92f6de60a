"""The C++ drop-in header (include/mixllm/mixquant.hpp) host checks, no GPU:
reference KATs and partition/scatter through the reference's C++ names."""
import os
import subprocess

from paper_2412_14590_b200 import _build


def test_cpp_dropin_host_checks():
    if not os.path.exists(_build.TEST_BIN):
        _build.build()
    r = subprocess.run([_build.TEST_BIN], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
