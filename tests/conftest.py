import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def port():
    from oracle import oracle
    if not oracle.available("port"):
        oracle.build()
    return oracle.Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle
    if not oracle.available("reference"):
        pytest.skip("oracle/_ref/libqft_ref.so not built (needs /root/reference at build time)")
    return oracle.Oracle("reference")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    import paper_2310_07147_b200 as q
    return q
