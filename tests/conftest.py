"""Test configuration.

Markers:
  gpu — needs a CUDA device (run on the B200 box: pytest -m gpu).
Everything else runs on CPU: the oracle (C restatement + the reference library
built from its sources) against the golden vectors, host logic, the C-ABI
library's exported symbols, and the multi-rank shard/merge logic over gloo.
"""
import os
import sys

import pytest

# a K12 code-generator error fails the test instead of falling back silently
os.environ.setdefault("RQ_JIT_STRICT", "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA device (B200)")


def _cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracle_built():
    from oracle import refpy
    if not os.path.exists(refpy.ORQ_SO) or (
            os.path.isdir(refpy.REFERENCE_SRC) and not os.path.exists(refpy.REF_SO)):
        refpy.build()
    return refpy


@pytest.fixture(scope="session")
def ref(oracle_built):
    if not os.path.exists(oracle_built.REF_SO):
        pytest.skip("reference library not built (no /root/reference here and no prebuilt _ref)")
    return oracle_built.Ref()


@pytest.fixture(scope="session")
def orq(oracle_built):
    return oracle_built.Orq()


@pytest.fixture(scope="session")
def rq():
    """The device API. Fails loudly if the CUDA library is missing."""
    from paper_2506_10092_b200 import runq
    return runq
