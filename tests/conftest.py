"""Test configuration: `gpu` marks tests that need a B200 (run on the GPU box
via gpurun); everything else runs on CPU here.  The oracle (oracle/) is the
parity checker and is only ever imported from tests."""
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long statistical test")


@pytest.fixture(scope="session")
def port():
    from oracle.build_oracle import build_port
    build_port()
    from oracle.oracle import Port
    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Ref, ref_available
    if not ref_available():
        from oracle.build_oracle import build_ref
        if build_ref() is None:
            pytest.skip("reference build (oracle/_ref) unavailable")
    return Ref()


@pytest.fixture(scope="session")
def smc():
    import paper_2604_03271_b200 as S
    return S
