"""Shared fixtures. `-m "not gpu"` runs here (no GPU); `-m gpu` runs on a B200 via gpurun.

The oracle (oracle/, test infrastructure) is the checker; the product package is what is tested.
"""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running full-size check")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.pyoracle import REF_SO, RefOracle
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefOracle()


@pytest.fixture(scope="session")
def vx():
    """The product package on a real GPU (fails loudly if the CUDA library is missing)."""
    import paper_2009_09500_b200 as vx
    ctx = vx.default_context()  # raises CudaError without a device: there is no fallback
    # device buffers in the tests come from torch: run on its stream so a torch.zeros() that is
    # still in flight cannot race the kernels
    ctx.use_torch_stream()
    return vx
