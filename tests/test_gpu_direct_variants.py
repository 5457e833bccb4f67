"""The direct kernel's load-width knob (BX_WIDE: 256-bit loads for q = 16)
changes the code path, never the bits: parity for both settings, every
power-of-two q, odd and even unit counts, partial warps and output offsets."""
import os
import pathlib
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

CHILD = pathlib.Path(__file__).with_name("gpu_direct_variants_child.py")


@pytest.mark.parametrize("lib", ["default", "checked"])
@pytest.mark.parametrize("wide", [0, 1])
def test_direct_load_width(wide, lib):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = {**os.environ, "BX_WIDE": str(wide)}
    if lib == "checked":
        env["BX_LIB"] = "checked"   # bounds-checked build: every read/write checked
    r = subprocess.run([sys.executable, str(CHILD), str(wide + 1)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert r.stdout.startswith("ok"), r.stdout
