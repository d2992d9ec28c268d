import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "ref: needs oracle/_ref/libevcm_ref.so (the compiled reference)")


@pytest.fixture(scope="session")
def engine():
    """The owner-computes pipeline (fast mode)."""
    import paper_2412_06359_b200 as P
    return P.Engine(P.EngineOptions(algo="owner"))


@pytest.fixture(scope="session")
def engine_f64():
    import paper_2412_06359_b200 as P
    return P.Engine(P.EngineOptions(stack_f64=True, grad_f64=True, algo="atomic", deterministic=False))


@pytest.fixture(scope="session")
def engine_fast():
    import paper_2412_06359_b200 as P
    return P.Engine(P.EngineOptions(stack_f64=False, algo="atomic", deterministic=False))


@pytest.fixture(scope="session")
def engine_atomic():
    import paper_2412_06359_b200 as P
    return P.Engine(P.EngineOptions(algo="atomic", deterministic=False))


@pytest.fixture(scope="session")
def engine_det():
    import paper_2412_06359_b200 as P
    return P.Engine(P.EngineOptions(deterministic=True))
