import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
for p in (str(ROOT), str(ROOT / "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")


@pytest.fixture(scope="session")
def oracle_lib():
    import cpu_checkers
    cpu_checkers.build_checkers()
    return cpu_checkers.oracle()


@pytest.fixture(scope="session")
def reference_lib():
    import cpu_checkers
    cpu_checkers.build_checkers()
    if not cpu_checkers.reference_available():
        pytest.skip("oracle/_ref/libks_ref.so not built (no /root/reference on this box)")
    return cpu_checkers.reference()
