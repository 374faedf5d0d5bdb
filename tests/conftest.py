"""Shared pytest setup: markers, import paths and backend fixtures."""
from __future__ import annotations

import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
# side-by-side simulations (run_clusters) on more than 8 streams
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libfbgpu.so")


@pytest.fixture(scope="session")
def oracle():
    from backends import OracleLib
    return OracleLib()


@pytest.fixture(scope="session")
def ref():
    from backends import RefLib
    if not RefLib.available():
        pytest.skip("oracle/_ref/libfbsim_ref.so not built (needs /root/reference)")
    return RefLib()


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(HERE, "golden", "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def fb():
    """The product library on a GPU; fails loudly (no fallback) if unusable."""
    from paper_2510_14392_b200 import fbgpu
    fbgpu.lib()
    if fbgpu.device_count() < 1:
        pytest.fail("no CUDA device visible for a gpu-marked test")
    return fbgpu
