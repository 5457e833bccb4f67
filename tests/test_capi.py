"""The C ABI from plain C: the header compiles as C99, and (on a GPU) a C
program using only include/blockext_b200.h + libbx_b200.so matches the oracle."""
import os
import pathlib
import subprocess

import pytest

REPO = pathlib.Path(__file__).resolve().parents[1]
LIBDIR = REPO / "paper_2402_14607_b200" / "_lib"
CUDA = pathlib.Path("/usr/local/cuda")


def _build(tmp_path) -> pathlib.Path:
    exe = tmp_path / "capi_smoke"
    cmd = ["gcc", "-std=c99", "-O1", "-I", str(REPO / "include"), "-I", str(CUDA / "include"),
           str(REPO / "tests" / "capi" / "capi_smoke.c"), "-o", str(exe),
           "-L", str(LIBDIR), "-lbx_b200", "-L", str(REPO / "oracle" / "_build"), "-lbx_oracle",
           "-L", str(CUDA / "lib64"), "-lcudart", "-Wl,-rpath," + str(LIBDIR),
           "-Wl,-rpath," + str(REPO / "oracle" / "_build"), "-Wl,-rpath," + str(CUDA / "lib64")]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_header_is_c99(tmp_path):
    src = tmp_path / "h.c"
    src.write_text('#include "blockext_b200.h"\nint (*volatile probe)(void) = bx_version;\nint main(void){return probe != 0 ? 0 : 1;}\n')
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-c", "-I", str(REPO / "include"),
                    str(src), "-o", str(tmp_path / "h.o")], check=True)


def test_capi_program_links(tmp_path):
    if not (LIBDIR / "libbx_b200.so").exists():
        pytest.skip("library not built")
    from oracle import coracle
    coracle.lib()   # builds oracle/_build if needed
    _build(tmp_path)


@pytest.mark.gpu
def test_capi_program_matches_oracle(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import coracle
    coracle.lib()
    exe = _build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120,
                       env={**os.environ})
    assert r.returncode == 0, r.stdout + r.stderr
    assert "fails=0" in r.stdout
