"""Run every kernel family under the bounds-checked library build.

compute-sanitizer is closed on this pool, so libbx_b200_checked.so (built with
-DBX_CHECKED) compares every shared/global index with its bound and counts
violations on the device; this test drives all kernel families through it in
a subprocess (BX_LIB=checked) and requires zero violations and exact results."""
import os
import pathlib
import subprocess
import sys

import pytest

REPO = pathlib.Path(__file__).resolve().parents[1]
CHECKED = REPO / "paper_2402_14607_b200" / "_lib" / "libbx_b200_checked.so"

pytestmark = pytest.mark.gpu


def test_all_kernel_families_within_bounds():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not CHECKED.exists():
        pytest.skip("checked library not built (python -m paper_2402_14607_b200.build --checked)")
    r = subprocess.run([sys.executable, str(REPO / "tools" / "sanitize_smoke.py")],
                       env={**os.environ, "BX_LIB": "checked"}, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "checked_violations 0" in r.stdout


def test_checker_catches_a_planted_violation():
    """BX_CHECK_SELFTEST shrinks the output bound by one word: must be reported."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not CHECKED.exists():
        pytest.skip("checked library not built")
    code = (
        "import torch, sys; sys.path.insert(0, %r)\n"
        "from paper_2402_14607_b200 import device as D, _lib\n"
        "x, n = D.to_device_stream(bytes(range(256)) * 64, 'cuda')\n"
        "D.extract_eq(x, n, x, n, 4, 64, 512)\n"
        "print('violations', _lib.checked_violations()[0])\n" % str(REPO))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       env={**os.environ, "BX_LIB": "checked", "BX_CHECK_SELFTEST": "1"})
    assert r.returncode == 0, r.stderr[-2000:]
    count = int(r.stdout.split("violations")[-1].split()[0])
    assert count > 0
