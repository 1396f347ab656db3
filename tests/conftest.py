import os
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _ensure_oracle():
    from oracle import oracle as O
    if not O.available("port"):
        import subprocess
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "libxaoracle.so"], check=True,
                       capture_output=True)


@pytest.fixture(scope="session")
def port():
    _ensure_oracle()
    from oracle.oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Oracle, available
    if not available("reference"):
        pytest.skip("oracle/_ref not built (needs /root/reference; see oracle/Makefile)")
    return Oracle("reference")


@pytest.fixture(scope="session")
def golden():
    path = ROOT / "tests" / "golden" / "golden.npz"
    return dict(np.load(path, allow_pickle=False))


@pytest.fixture(scope="session")
def xa():
    """The product API on cuda:0 (GPU tests only)."""
    import paper_2503_03479_b200 as xa
    from paper_2503_03479_b200 import build
    build.build()
    return xa
