"""Build an experimental variant of the library with extra -D flags.

    python tools/build_variant.py NAME -DFOO=1 ...   ->  _exp/NAME/libbx_b200.so

Load it with BX_LIB=/abs/path/libbx_b200.so (paper_2402_14607_b200/_lib.py).
For A/B measurements only; _exp/ is git-ignored but travels with gpurun."""
import concurrent.futures as cf
import os
import pathlib
import subprocess
import sys

REPO = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

from paper_2402_14607_b200 import build as B  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out = REPO / "_exp" / name
    out.mkdir(parents=True, exist_ok=True)
    srcs = sorted(B.CSRC.glob("*.cu"))

    def comp(src):
        obj = out / (src.stem + ".o")
        subprocess.run([B.nvcc(), *B.ARCH, *B.NVCC_FLAGS, *defs, "-c", str(src), "-o", str(obj)],
                       check=True)
        return obj

    with cf.ThreadPoolExecutor(os.cpu_count() or 4) as ex:
        objs = list(ex.map(comp, srcs))
    lib = out / "libbx_b200.so"
    subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", str(lib), *map(str, objs)], check=True)
    for o in objs:            # keep only the library (the snapshot travels to the GPU box)
        o.unlink()
    print(lib)


if __name__ == "__main__":
    main()
