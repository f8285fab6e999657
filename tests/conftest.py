"""Shared test fixtures.  `-m gpu` tests need a B200; everything else runs on CPU."""
import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def golden_runs():
    return json.loads((GOLDEN / "runs.json").read_text())["cases"]


@pytest.fixture(scope="session")
def golden_runs_draft_model():
    """Compression / contention runs (scripts/make_golden_draft_model.py)."""
    return json.loads((GOLDEN / "runs_draft_model.json").read_text())["cases"]


@pytest.fixture(scope="session")
def golden_runs_conservative():
    """Conservative parallel rounds (scripts/make_golden_conservative.py)."""
    return json.loads((GOLDEN / "runs_conservative.json").read_text())["cases"]


@pytest.fixture(scope="session")
def golden_streams():
    return json.loads((GOLDEN / "streams.json").read_text())


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
