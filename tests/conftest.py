import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU and the built library")


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle():
    from checkers import Checker

    return Checker("oracle")


@pytest.fixture(scope="session")
def ref():
    from checkers import Checker, ref_available

    if not ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Checker("ref")
