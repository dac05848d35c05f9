"""Test configuration.

Markers:
  gpu   needs a CUDA device (a B200); run with `pytest -m gpu` on the GPU box.
Everything unmarked runs on CPU in the build container.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load_golden(name: str) -> dict:
    return json.loads((GOLDEN / name).read_text())


@pytest.fixture(scope="session")
def devicert_golden() -> dict:
    return load_golden("devicert_vectors.json")


@pytest.fixture(scope="session")
def fallback_golden() -> dict:
    return load_golden("fallback_runs.json")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test needs a CUDA device")
    from paper_2106_03219_b200 import _lib

    _lib.load()  # the native library must load; there is no fallback
    return torch.device("cuda", 0)
