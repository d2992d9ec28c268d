"""GPU: the reference-side C++ binding (include/evcm_cuda_backend.hpp), compiled
against the reference headers into oracle/_ref/adapter_test, agrees with the
reference Engine on the reference's own fixtures (tests/cpp/adapter_test.cpp)."""
import os
import subprocess

import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
EXE = os.path.join(os.path.dirname(O.REF_SO), "adapter_test")


@pytest.mark.skipif(not os.path.exists(EXE), reason="adapter_test not built (needs /root/reference)")
def test_cpp_adapter_matches_reference_engine():
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("OK")
