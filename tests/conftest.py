import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import core

    core.build()
    return core


@pytest.fixture(scope="session")
def native_lib():
    from paper_2010_08454_b200 import build

    build.build()
    from paper_2010_08454_b200 import _native

    return _native.lib()


@pytest.fixture(scope="session")
def cuda(native_lib):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    return torch.device("cuda", 0)
