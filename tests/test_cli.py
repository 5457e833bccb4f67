"""CLI parity (reference pkg/tests/test_cli.py patterns): plan printing and exit
codes on CPU; file round trips through the GPU path under -m gpu."""

import numpy as np
import pytest

import paper_2402_14607_b200 as bx
from paper_2402_14607_b200.cli import main
from oracle import coracle



def test_params_prints_flagship_plan(capsys):
    assert main(["params", "--b", "16", "--delta", "10.74/16", "--N", "2^47",
                 "--epsilon", "2^-30"]) == 0
    plan = bx.plan_from_text(capsys.readouterr().out)
    assert plan.vec_len == 71 and plan.field_bits == 80


def test_params_n_bits(capsys):
    assert main(["params", "--b", "16", "--delta", "10.74/16", "--N-bits", "2^51",
                 "--epsilon", "2^-30"]) == 0
    assert bx.plan_from_text(capsys.readouterr().out).num_samples == 2**47
    assert main(["params", "--b", "16", "--delta", "10.74/16", "--N-bits", "1001",
                 "--epsilon", "2^-30"]) == 2


def test_params_exit_codes(capsys):
    assert main(["params", "--b", "16", "--delta", "1/2", "--N", "2^40", "--epsilon", "2^-30"]) == 4
    assert main(["params", "--b", "16", "--delta", "0.51", "--N", "2^500",
                 "--epsilon", "2^-300"]) == 3
    assert main(["params", "--b", "16", "--delta", "3/4", "--N", "2^40", "--epsilon", "2"]) == 2


def test_extract_two_stdin_is_usage_error(tmp_path, capsys):
    out = tmp_path / "o.bin"
    assert main(["extract-eq", "--x", "-", "--y", "-", "--out", str(out), "--b", "8",
                 "--delta", "3/4", "--epsilon", "2^-10", "--N", "100"]) == 2


def test_missing_file_is_io_error(tmp_path, capsys):
    assert main(["extract-eq", "--x", str(tmp_path / "nope"), "--y", str(tmp_path / "nope2"),
                 "--out", str(tmp_path / "o"), "--b", "8", "--delta", "3/4",
                 "--epsilon", "2^-10"]) == 5


@pytest.mark.gpu
def test_extract_eq_files_round_trip(tmp_path, capsys):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(5)
    xb, yb = rng.bytes(40_000), rng.bytes(40_000)
    (tmp_path / "x.bin").write_bytes(xb)
    (tmp_path / "y.bin").write_bytes(yb)
    args = ["extract-eq", "--x", str(tmp_path / "x.bin"), "--y", str(tmp_path / "y.bin"),
            "--b", "8", "--delta", "3/4", "--epsilon", "2^-10"]
    assert main(args + ["--out", str(tmp_path / "o1.bin"), "--report", str(tmp_path / "r1")]) == 0
    assert main(args + ["--out", str(tmp_path / "o2.bin"), "--report", str(tmp_path / "r2")]) == 0
    o1 = (tmp_path / "o1.bin").read_bytes()
    assert o1 == (tmp_path / "o2.bin").read_bytes()
    assert main(args + ["--out", str(tmp_path / "o4.bin"), "--devices", "0,0"]) == 0
    assert (tmp_path / "o4.bin").read_bytes() == o1
    rep = bx.ExtractionReport.from_text((tmp_path / "r1").read_text())
    plan = rep.plan
    want = coracle.extract_eq(xb, yb, plan.field_bits, plan.vec_len, rep.blocks_completed)
    assert o1 == want and rep.stop_reason == "completed"
    # neq with growth 0 reproduces eq through files
    nargs = ["extract-neq", "--x", str(tmp_path / "x.bin"), "--y", str(tmp_path / "y.bin"),
             "--b", "8", "--delta", "3/4", "--q1", str(plan.field_bits), "--growth", "0",
             "--max-blocks", str(plan.num_blocks), "--out", str(tmp_path / "o3.bin"),
             "--report", str(tmp_path / "r3")]
    assert main(nargs) == 0
    assert (tmp_path / "o3.bin").read_bytes() == o1
