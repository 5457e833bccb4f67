"""bench.py keeps the driver's JSON contract (one line, required keys and types)."""
import json
import os
import pathlib
import subprocess
import sys

import pytest

REPO = pathlib.Path(__file__).resolve().parents[1]


def _run(args, timeout=600):
    r = subprocess.run([sys.executable, str(REPO / "bench.py"), *args], capture_output=True,
                       text=True, timeout=timeout, cwd=str(REPO), env={**os.environ})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--ref-blocks", "4096"])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "cpu_baseline"):
        assert k in d, k
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"] == "c5" and d["value"] > 0
    assert d["config"]["legs"] == ["c5_n128", "c5_n256", "c5_n512", "c5_n1024", "c5_n2048"]


def test_reference_arm_other_ranks_exit_quietly():
    r = subprocess.run([sys.executable, str(REPO / "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--ref-blocks", "1024"], capture_output=True, text=True,
                       timeout=600, cwd=str(REPO),
                       env={**os.environ, "RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_gpus_flag_relaunches_under_torchrun(monkeypatch):
    """--gpus N without WORLD_SIZE starts N ranks through torch.distributed.run."""
    sys.path.insert(0, str(REPO))
    import bench

    seen = {}

    def fake_run(cmd, env=None, **kw):
        seen["cmd"], seen["env"] = cmd, env

        class R:
            returncode = 0
        return R()

    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "run", fake_run)
    assert bench.main(["--gpus", "4", "--steps", "2"]) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "2"][-3:]


def test_sharded_ranges_cover_c5_identically():
    """Strong scaling splits every C5 leg on the same stream bit boundaries, so
    a rank generates one slice of each stream for the whole sweep."""
    from paper_2402_14607_b200 import sharding
    from paper_2402_14607_b200 import workloads as W

    legs = [W.WORKLOADS[f"c5_n{n}"] for n in (128, 256, 512, 1024, 2048)]
    for world in (1, 2, 4, 8):
        for rank in range(world):
            spans = {(s * wl.block_bits, (s + c) * wl.block_bits)
                     for wl in legs for s, c in [sharding.rank_range(wl.num_blocks, rank, world)]}
            assert spans == {(rank * 2**36 // world, (rank + 1) * 2**36 // world)}


@pytest.mark.gpu
def test_our_arm_contract():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--steps", "3", "--warmup", "3", "--no-cpu", "--e2e-steps", "1", "--e2e-warmup", "0"],
             timeout=1200)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "roofline", "cpu_baseline", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3
    assert d["higher_is_better"] is True and d["scaling"] == "strong" and d["vs_baseline"] is None
    assert d["config"]["workload"] == "c5" and len(d["sweep"]) == 5
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert d["e2e"]["h2d_bytes_per_step"] == 5 * 2 * 2**33 and d["e2e"]["bit_exact_vs_device_run"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    assert d["roofline"]["bound"] in ("hbm", "int") and 0.3 < d["roofline"]["frac"] < 1.5
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in d["clocks"], k
    assert d["gpu_launches"] == 3 * 5
    assert d["parity"]["mismatches"] == 0
