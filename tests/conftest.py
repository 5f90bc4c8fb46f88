import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device; parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running (large-size) test")


def _impl_module(name):
    if name == "oracle":
        from oracle import oracle as m
        return m
    import paper_2110_02820_b200 as m
    return m


@pytest.fixture(params=[pytest.param("oracle"), pytest.param("b200", marks=pytest.mark.gpu)])
def impl(request):
    """The implementation under test: the CPU oracle (CPU suite) or the B200
    product (GPU suite). Both expose the reference's API names."""
    return _impl_module(request.param)


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as m
    return m
