import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100) device")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


def _cuda_available() -> bool:
    try:
        import paper_2301_02959_b200 as ts
        return ts.device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda():
    if not _cuda_available():
        pytest.fail("GPU test needs a CUDA device (no CPU fallback exists)")
    return True


@pytest.fixture(scope="session")
def tmp_spec_dir(tmp_path_factory):
    return tmp_path_factory.mktemp("specs")
