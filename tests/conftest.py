import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and libdooly_b200.so")


def pytest_collection_modifyitems(config, items):
    import torch

    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def corpus():
    from paper_2605_07985_b200 import modelir

    return modelir.load_manifest(modelir.builtin_manifest_path("corpus12"))


@pytest.fixture(scope="session")
def fixtures_manifest():
    from paper_2605_07985_b200 import modelir

    return modelir.load_manifest(modelir.builtin_manifest_path("fixtures"))


@pytest.fixture(scope="session")
def dev():
    import torch

    return torch.device("cuda", 0)
