import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")
    # Build the checker and the product library if a fresh checkout lacks them
    # (nvcc cross-compiles; no GPU needed).
    import __graft_entry__

    __graft_entry__._load_by_path("oracle_build", ROOT / "oracle" / "build.py").build()
    lib = ROOT / "paper_2208_04726_b200" / "libpvo_b200.so"
    if not lib.exists():
        __graft_entry__._load_by_path("pvo_build", ROOT / "paper_2208_04726_b200" / "build.py").build()


@pytest.fixture(scope="session")
def ctx():
    from paper_2208_04726_b200 import Context

    c = Context(int(os.environ.get("PVO_DEVICE", "0")))
    yield c
    c.close()


@pytest.fixture(scope="session")
def orc():
    import oracle.pyoracle as o

    return o
