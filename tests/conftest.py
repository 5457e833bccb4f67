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


def pytest_sessionfinish(session, exitstatus):
    """Under BX_LIB=checked (the bounds-checked library build), fail the session
    if any kernel run in this process recorded an out-of-bounds index."""
    import os
    if os.environ.get("BX_LIB") != "checked":
        return
    from paper_2402_14607_b200 import _lib
    if _lib._handle is None:
        return
    try:
        import torch
        if not torch.cuda.is_available():
            return
    except ImportError:
        return
    n, first = _lib.checked_violations()
    print(f"\nchecked build: {n} bounds violations (first {first})")
    if n:
        session.exitstatus = 1
