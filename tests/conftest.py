import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device")
    config.addinivalue_line("markers", "slow: long-running case")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build(ref=os.path.isdir(oracle.REF_SRC))
    return oracle.Orc()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not os.path.exists(oracle.REF_SO):
        if os.path.isdir(oracle.REF_SRC):
            oracle.build(ref=True)
        else:
            pytest.skip("oracle/_ref/libuscg_ref.so not built and /root/reference absent")
    return oracle.Ref()


@pytest.fixture(scope="session")
def ub():
    import paper_2208_12964_b200 as ub
    ub.load()
    return ub
