"""GPU parity of the dot-product (IDP.2A) holes kernels: randomized shapes for
every q in 9..64 (tile kernel thread splits, bit offsets), the aligned direct
and period kernels at multi-CTA sizes, with dense inputs (all ones, 90-95% ones)
that maximise the per-field product counts -- against the C oracle, bit-exact.
tests/test_dot_model.py pins the same arithmetic on the CPU."""
import pathlib
import runpy
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

REPO = pathlib.Path(__file__).resolve().parents[1]


def test_dot_kernels_randomized_and_dense(capsys, monkeypatch):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    monkeypatch.setattr(sys, "argv", ["r02_dot_stress.py", "1"])
    runpy.run_path(str(REPO / "tools" / "gpu" / "r02_dot_stress.py"), run_name="__main__")
    out = capsys.readouterr().out
    assert out.startswith("ok "), out
    assert int(out.split()[1]) >= 200


@pytest.mark.parametrize("stages", ["1", "2"])
def test_tma_stage_variants_agree_with_oracle(stages):
    """The TMA kernel picks one or two input stages per launch from occupancy;
    both forced settings (BX_TMA_STAGES is read once per process) must give the
    oracle's bits on the same randomized shapes."""
    import os
    import subprocess

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, str(REPO / "tools" / "gpu" / "r02_dot_stress.py"), "1"],
                       env={**os.environ, "BX_TMA_STAGES": stages}, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.startswith("ok "), r.stdout
