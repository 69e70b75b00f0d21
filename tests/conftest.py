import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE step counts)")


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import load_oracle

    return load_oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import load_ref

    r = load_ref()
    if r is None:
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return r


@pytest.fixture(scope="session")
def pg():
    import paper_1507_06565_b200 as pg

    return pg


@pytest.fixture(scope="session")
def gpu(pg):
    if pg.device_count() < 1:
        pytest.fail("GPU test selected but no CUDA device is visible")
    return pg
