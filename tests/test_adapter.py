"""The C++ drop-in (include/ttrec_gpu.hpp): the reference's own types and test
helpers drive the GPU through ttrec::gpu::forward_bags / backward_bags /
sgd_step / lookup_row, checked by the reference's CPU operators
(oracle/adapter_test.cpp, built by `make -C oracle` into oracle/_ref/)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_test")


@pytest.mark.skipif(not os.path.exists(BIN), reason="adapter_test not built (needs the reference)")
def test_adapter_binary_links_against_libttgpu():
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    line = next(l for l in out.splitlines() if "libttgpu" in l)
    assert "not found" not in line and "paper_2101_11714_b200/lib/libttgpu.so" in line


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="adapter_test not built (needs the reference)")
def test_cpp_adapter_against_reference_operators():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASSED" in r.stdout
