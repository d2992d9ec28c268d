"""CPU: the C-ABI library (libevcm_cuda.so) loads, exports every entry point
declared in include/*.h, and fails loudly (no CPU fallback) without a GPU."""
import ctypes as C
import os
import re

import pytest

import paper_2412_06359_b200 as P
from paper_2412_06359_b200 import engine as E

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    inc = os.path.join(ROOT, "include")
    for f in os.listdir(inc):
        if f.endswith(".h"):
            syms |= set(re.findall(r"EVCM_API\s+[\w\s\*]+?\b(evcm_cuda_\w+)\s*\(",
                                   open(os.path.join(inc, f)).read()))
    return sorted(syms)


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("evcm_cuda_create", "evcm_cuda_forward", "evcm_cuda_backward",
              "evcm_cuda_depth_pose_to_flows", "evcm_cuda_depth_pose_to_flows_backward",
              "evcm_cuda_chain_batch", "evcm_cuda_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = P.load_library()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_no_undeclared_exports():
    out = os.popen(f"nm -D --defined-only {E.library_path()}").read()
    exported = set(re.findall(r" T (evcm_cuda_\w+)", out))
    assert exported == set(declared_symbols())


def test_error_names_and_abi_version():
    lib = P.load_library()
    names = {c: lib.evcm_cuda_error_name(c).decode() for c in (1, 2, 3, 4, 5, 6, 7, 20, 21)}
    assert names[1] == "ConfigError" and names[2] == "DimensionMismatchError"
    assert names[3] == "CoordinateRangeError" and names[5] == "UnsortedEventsError"
    assert lib.evcm_cuda_abi_version() == 2


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors in engine.py agree with the C structs of include/evcm_cuda.h."""
    assert P.EVENT_DTYPE.itemsize == 16  # evcm::Event (types.hpp:106-113)
    src = tmp_path / "sz.c"
    src.write_text('#include "evcm_cuda.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu %zu %zu %zu\\n",'
                   'sizeof(evcm_event), sizeof(evcm_cuda_options), sizeof(evcm_slice),'
                   'sizeof(evcm_flows), sizeof(evcm_loss), sizeof(evcm_chain_batch),'
                   'sizeof(evcm_chain_out), offsetof(evcm_chain_batch, events));return 0;}')
    exe = tmp_path / "sz"
    assert os.system(f"gcc -I{ROOT}/include -o {exe} {src}") == 0
    got = [int(x) for x in os.popen(str(exe)).read().split()]
    want = [16, C.sizeof(E._Options), C.sizeof(E._Slice), C.sizeof(E._Flows), C.sizeof(E._Loss),
            C.sizeof(E._ChainBatch), C.sizeof(E._ChainOut), E._ChainBatch.events.offset]
    assert got == want


def test_default_options():
    lib = P.load_library()
    o = E._Options()
    lib.evcm_cuda_default_options(C.byref(o))
    # deterministic by default, as the reference (engine.hpp:60)
    assert o.stack_f64 == 1 and o.grad_f64 == 0 and o.algo == 2 and o.deterministic == 1
    assert P.EngineOptions().deterministic is True


def test_abi_version():
    assert P.load_library().evcm_cuda_abi_version() == 2


def test_backend_names():
    """Backend is 'cuda'; 'gpu' stays rejected (test_optimize.cpp:102)."""
    assert P.backend_from_name("cuda") == "cuda"
    with pytest.raises(P.ConfigError):
        P.backend_from_name("gpu")
    with pytest.raises(P.ConfigError):
        P.Engine(P.EngineOptions(algo="magic"))


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="needs a GPU-less host")
def test_engine_fails_loudly_without_gpu():
    with pytest.raises(P.Error):
        P.Engine()
