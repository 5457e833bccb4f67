"""Full-size configs on the GPU (BASELINE.json configs 2-5 shapes).

* config 2 (c2) in full: reference-identical seeded streams (pinned by
  tests/golden/streams.json), every block vs the CPU oracle, plus the
  reference's own outputs at sampled blocks (tests/golden/sampled.json);
* configs 3, 4, the planner shapes, paper and c5 (first 2^33 bits) in full vs
  the oracle; config 3 and the planner shapes also at sampled reference blocks;
* size-independent properties at full size: bilinearity
  E(x1^x2, y) = E(x1, y) ^ E(x2, y), zero annihilation, segmentation and
  device-sharding invariance.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2402_14607_b200 as bx
from paper_2402_14607_b200 import device as D
from paper_2402_14607_b200 import sharding
from paper_2402_14607_b200 import workloads as W
from oracle import coracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _run(xd, yd, nbytes, wl, nblocks=None):
    nb = nblocks or wl.num_blocks
    out = D.extract_eq(xd, nbytes, yd, nbytes, wl.q, wl.n, nb)
    return out[:(nb * wl.q + 7) // 8]


def _block(outbytes, l, q):
    seg = outbytes[l * q // 8:(l * q + q + 7) // 8 + 1]
    return (int.from_bytes(seg, "little") >> (l * q % 8)) & ((1 << q) - 1)


def test_c2_full_vs_oracle_and_reference_samples(golden):
    wl = W.WORKLOADS["c2"]
    xd, nbytes = W.stream_device(wl.x, wl.samples)
    yd, _ = W.stream_device(wl.y, wl.samples)
    got = _run(xd, yd, nbytes, wl).cpu().numpy().tobytes()
    xh = xd[:nbytes].cpu().numpy()
    yh = yd[:nbytes].cpu().numpy()
    assert got == coracle.extract_eq(xh, yh, wl.q, wl.n, wl.num_blocks)
    for l, z in golden("sampled.json")["c2"]["blocks"]:
        assert _block(got, l, wl.q) == int(z, 16), l


@pytest.mark.parametrize("name", ["c2p", "c3", "c5_n2048", "paper"])
def test_sampled_reference_blocks_full_size(golden, name):
    wl = W.WORKLOADS[name]
    rec = golden("sampled.json")[name]
    samples = wl.samples if name != "c5_n2048" else 2**27   # first 2^30 bits suffice
    xd, nbytes = W.stream_device(wl.x, samples)
    yd, _ = W.stream_device(wl.y, samples)
    nblocks = samples * wl.b // wl.block_bits
    got = _run(xd, yd, nbytes, wl, nblocks).cpu().numpy().tobytes()
    checked = 0
    for l, z in rec["blocks"]:
        if l < nblocks:
            assert _block(got, l, wl.q) == int(z, 16), (name, l)
            checked += 1
    assert checked >= 3


@pytest.mark.parametrize("name", ["c3", "c4", "c2p", "c4p", "paper", "c5_n1024", "c5_n2048"])
def test_full_output_vs_oracle(name):
    """Every block of the config (c5: the first 2^33 bits of each stream) against
    the CPU oracle (PCLMUL mode, all host threads), so each kernel family's
    full-size launch -- the one bench.py times -- is bit-exact end to end."""
    wl = W.WORKLOADS[name]
    samples = wl.samples if not name.startswith("c5") else (2**33) // wl.b
    xd, nbytes = W.stream_device(wl.x, samples)
    yd, _ = W.stream_device(wl.y, samples)
    nblocks = samples * wl.b // wl.block_bits
    got = _run(xd, yd, nbytes, wl, nblocks).cpu().numpy().tobytes()
    xh = xd[:nbytes].cpu().numpy()
    yh = yd[:nbytes].cpu().numpy()
    del xd, yd
    assert got == coracle.extract_eq(xh, yh, wl.q, wl.n, nblocks), name


@pytest.mark.parametrize("q,n", [(4, 64), (4, 128), (2, 64), (8, 64), (16, 64), (32, 64),
                                 (128, 8), (56, 48), (58, 120), (80, 71)])
def test_bilinearity_and_zero_at_scale(q, n):
    nblocks = (1 << 29) // (q * n)          # 2 x 64 MiB inputs
    nbytes = nblocks * q * n // 8
    g = torch.Generator(device="cuda").manual_seed(q * 1000 + n)
    mk = lambda: torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device="cuda", generator=g)
    x1, x2, y = mk(), mk(), mk()
    def run(a, b):
        A = D.empty_stream(nbytes, "cuda"); A[:nbytes] = a
        Bt = D.empty_stream(nbytes, "cuda"); Bt[:nbytes] = b
        return D.extract_eq(A, nbytes, Bt, nbytes, q, n, nblocks)[:(nblocks * q + 7) // 8]
    lhs = run(x1 ^ x2, y)
    rhs = run(x1, y) ^ run(x2, y)
    assert torch.equal(lhs, rhs)
    assert not torch.any(run(torch.zeros_like(y), y))
    # y-linearity too
    assert torch.equal(run(y, x1 ^ x2), run(y, x1) ^ run(y, x2))
    # spot check against the oracle
    xs = x1[:1 << 16].cpu().numpy()
    ys = y[:1 << 16].cpu().numpy()
    k = (1 << 19) // (q * n)
    assert run(x1, y)[:(k * q) // 8].cpu().numpy().tobytes() == \
        coracle.extract_eq(xs, ys, q, n, k)[:(k * q) // 8]


def test_segmentation_and_sharding_invariance():
    q, n = 56, 48
    nblocks = 200_003
    nbytes = nblocks * q * n // 8 + 1
    rng = np.random.default_rng(9)
    xb, yb = rng.bytes(nbytes), rng.bytes(nbytes)
    plan = bx.EqPlan(8, nbytes, bx.params.as_rational("3/4"), bx.params.as_rational("1/2"), n, q,
                     nblocks, nblocks * q, 0.0)
    import io
    outs = []
    for kw in ({}, {"segment_blocks": 4096}, {"devices": [0, 0, 0]}):
        sink = io.BytesIO()
        rep = bx.extract_eq(xb, yb, plan, **kw).run(sink)
        assert rep.blocks_completed == nblocks
        outs.append(sink.getvalue())
    assert outs[0] == outs[1] == outs[2]
    assert outs[0] == coracle.extract_eq(xb, yb, q, n, nblocks)
