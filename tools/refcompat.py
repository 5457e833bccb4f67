"""Run the reference's own test modules against this package (drop-in check).

    python tools/refcompat.py prepare     # in the build container (reads /root/reference)
    python -m pytest refcompat -q         # anywhere (GPU box for the compute tests)

`prepare` copies selected reference test modules into ./refcompat/ (git-ignored,
never committed) with `blockext` imports pointed at paper_2402_14607_b200.
Nothing of the reference is stored in the repository; the results of a run are
summarised in profiles/.
"""
import pathlib
import re
import shutil
import sys

REPO = pathlib.Path(__file__).resolve().parents[1]
SRC = pathlib.Path("/root/reference/pkg/tests")
DST = REPO / "refcompat"
MODULES = ["test_extractor.py", "test_gf2q.py", "test_bitio.py", "test_params.py", "test_verify.py"]


def prepare() -> None:
    if DST.exists():
        shutil.rmtree(DST)
    DST.mkdir()
    (DST / "conftest.py").write_text(
        "import sys, pathlib\n"
        "sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))\n"
        "sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent))\n"
        "import torch\n"
        "if torch.cuda.is_available():  # warm the CUDA context before timed hypothesis cases\n"
        "    from paper_2402_14607_b200 import device as _D\n"
        "    _D.pack(torch.zeros(8, dtype=torch.uint8, device='cuda'), 1)\n"
        "    torch.cuda.synchronize()\n")
    for name in MODULES:
        text = (SRC / name).read_text()
        text = text.replace("from tests.test_bitio import DribbleIO", "from test_bitio import DribbleIO")
        text = re.sub(r"\bblockext\b", "paper_2402_14607_b200", text)
        (DST / name).write_text(text)
    print("prepared", len(MODULES), "modules in", DST)


if __name__ == "__main__":
    if sys.argv[1:] == ["prepare"]:
        prepare()
