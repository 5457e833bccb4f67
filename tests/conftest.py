"""Shared pytest setup: repo root on sys.path, the `gpu` marker, fixtures loader."""
import json
import pathlib
import sys

import pytest

REPO = pathlib.Path(__file__).resolve().parents[1]
GOLDEN = REPO / "tests" / "golden"
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    path = GOLDEN / name
    if name.endswith(".json"):
        return json.loads(path.read_text())
    return path.read_bytes()


@pytest.fixture(scope="session")
def golden():
    return load_golden
