"""Source simulators and the packer on the GPU."""
import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2402_14607_b200 import device as D
from paper_2402_14607_b200 import sources as S
from paper_2402_14607_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_generate_matches_reference_prefixes(golden):
    want = golden("streams.json")
    for key, digest in want.items():
        name, side = key.split(".")
        wl = W.WORKLOADS[name]
        spec = wl.x if side == "x" else wl.y
        got = S.generate(W.to_model(spec), 1 << 15)
        assert hashlib.sha256(got).hexdigest() == digest, key


def test_generate_markov_matches_reference(golden):
    for c in golden("markov.json"):
        size = 1 << c["b"]
        tab = np.random.default_rng(c["table_seed"]).random((size, size)) ** 3
        tab /= tab.sum(axis=1, keepdims=True)
        model = S.markov(tab, c["b"], seed=c["seed"])
        assert S.generate(model, c["count"]).hex() == c["out"], c["b"]


def test_pack_samples_matches_reference(golden):
    for c in golden("pack.json"):
        vals = np.array([int(v, 16) for v in c["values"]], dtype=np.uint64)
        assert S._pack_samples(vals, c["b"]).hex() == c["out"]


def test_bernoulli_bits_match_host_restatement():
    for p, seed, bit0, nbits in [(0.5, 1, 0, 4096), (0.2, 7, 512, 100_000), (0.0, 3, 0, 999),
                                 (1.0, 3, 64, 1000), (0.3, 2**40 + 5, 32, 77)]:
        out = D.bernoulli_bits(nbits, p, seed, bit0=bit0)
        nb = (nbits + 7) // 8
        host = np.packbits(W.splitmix_bits_host(seed, bit0, nbits, p), bitorder="little")
        assert out[:nb].cpu().numpy().tobytes() == host.tobytes(), (p, seed, bit0, nbits)


@pytest.mark.parametrize("rows,cols", [(1, 4), (2, 16), (63, 16), (64, 16), (1000, 1), (70_001, 16),
                                       (300_000, 8)])
def test_xor_scan_rows(rows, cols):
    g = torch.Generator(device="cuda").manual_seed(rows)
    m = torch.randint(0, 256, (rows * cols * 4 + 16,), dtype=torch.uint8, device="cuda", generator=g)
    host = m[:rows * cols * 4].cpu().numpy().view(np.uint32).reshape(rows, cols)
    want = np.bitwise_xor.accumulate(host, axis=0)
    D.xor_scan_rows(m, rows, cols * 4)
    got = m[:rows * cols * 4].cpu().numpy().view(np.uint32).reshape(rows, cols)
    assert np.array_equal(got, want)


def test_block_markov_device_equals_host():
    spec = W.block_markov_spec(0.2, 11, 512)
    samples = 512 * 3000
    dev, nbytes = W.stream_device(spec, samples)
    host = W._block_markov_host(spec, samples)
    assert dev[:nbytes].cpu().numpy().tobytes() == host.tobytes()
    # forward-block property sanity: consecutive blocks differ in ~20% of bits
    blocks = host.reshape(-1, 64)
    flips = np.unpackbits(blocks[1:] ^ blocks[:-1]).mean()
    assert 0.18 < flips < 0.22
