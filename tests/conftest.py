import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA extension")


@pytest.fixture(scope="session")
def oracle():
    import oracle as O
    O.build()  # C restatement; cheap, idempotent
    return O


@pytest.fixture(scope="session")
def ccq():
    import paper_2507_07145_b200 as P
    P.lib()  # fail loudly if the product library is missing
    return P


@pytest.fixture(scope="session")
def cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    major, minor = torch.cuda.get_device_capability(0)
    assert (major, minor) == (10, 0), f"expected sm_100 (B200), got sm_{major}{minor}"
    return torch
