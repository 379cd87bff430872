"""Single-GPU ring (W logical peers on one B200) vs the reference's ring
outputs: every golden case of tests/golden/golden.json, bit-exact."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ring as oring
from oracle import simplehash as osh
from tests.golden.gen import RING_CASES, ring_inputs
from tests.gpu_util import bits, need_gpu, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


@pytest.mark.parametrize("idx", range(len(RING_CASES)))
def test_golden_case(golden, idx):
    from paper_2505_14065_b200 import LocalRing

    c = golden["ring"][idx]
    bufs = ring_inputs(c["w"], c["n"], np.dtype(c["dtype"]), c["seed"])
    dev = [to_dev(b) for b in bufs]
    res = LocalRing(c["w"]).run_op(dev, c["op"], quantize=c["quantize"])
    assert all(s == "ok" for s, _ in res)
    for d in dev:
        assert osh.simplehash_c(d.cpu().numpy()) == c["output_hash"]


@pytest.mark.parametrize("quant,key", [(False, "plain"), (True, "quant")])
def test_appendix_c_w8_avg_16m(golden, quant, key):
    from paper_2505_14065_b200 import LocalRing, simplehash_many

    rng = np.random.default_rng(0)
    dev = [to_dev(rng.normal(0, 1, 1 << 24).astype(np.float32)) for _ in range(8)]
    LocalRing(8).run_op(dev, "avg", quantize=quant)
    assert set(simplehash_many(dev)) == {golden["appendix_c_w8_avg_16M"][key]}


@pytest.mark.parametrize("offset", [1, 2, 3])
def test_misaligned_buffers(offset):
    from paper_2505_14065_b200 import LocalRing

    w, n = 4, 100_003
    rng = np.random.default_rng(offset)
    host = [rng.normal(0, 1, n).astype(np.float32) for _ in range(w)]
    for quant in (False, True):
        want = oring.ring_allreduce_chunkwise(host, oring.ReduceOp.AVG, quantize=quant)
        dev = [to_dev(np.concatenate([np.zeros(offset, np.float32), h]))[offset:] for h in host]
        LocalRing(w).run_op(dev, "avg", quantize=quant)
        for d in dev:
            assert bits(d) == bits(want)


def test_nonfinite_quantized_restores():
    from paper_2505_14065_b200 import LocalRing

    w, n = 3, 4096
    rng = np.random.default_rng(1)
    host = [rng.normal(0, 1, n).astype(np.float32) for _ in range(w)]
    host[1][100] = np.inf
    dev = [to_dev(h) for h in host]
    res = LocalRing(w).run_op(dev, "sum", quantize=True)
    assert all(s == "aborted" for s, _ in res)
    for d, h in zip(dev, host):
        assert bits(d) == bits(h)


def test_overflow_mid_ring_restores():
    """SURVEY §0 finding 5: a partial sum overflowing to inf makes the
    reference raise without restoring; this build aborts and restores."""
    from paper_2505_14065_b200 import LocalRing

    w, n = 3, 64
    host = [np.full(n, 3e38, np.float32) for _ in range(w)]
    dev = [to_dev(h) for h in host]
    res = LocalRing(w).run_op(dev, "sum", quantize=True)
    assert all(s == "aborted" for s, _ in res)
    for d, h in zip(dev, host):
        assert bits(d) == bits(h)


def test_repeat_runs_bit_identical():
    from paper_2505_14065_b200 import LocalRing

    w, n = 3, 2048
    rng = np.random.default_rng(12)
    base = [rng.normal(0, 10, n).astype(np.float32) for _ in range(w)]
    ring = LocalRing(w)
    outs = []
    for _ in range(2):
        dev = [to_dev(b) for b in base]
        ring.run_op(dev, "avg")
        outs.append(bits(dev[0]))
    assert outs[0] == outs[1]


def test_large_streaming_oracle_w8():
    """Config-2 shaped (W=8) at 64 Mi elements per rank, checked chunk by chunk."""
    from paper_2505_14065_b200 import LocalRing

    w, n = 8, 1 << 26
    gens = [torch.Generator(device="cuda").manual_seed(r) for r in range(w)]
    dev = [torch.randn(n, generator=g, device="cuda") for g in gens]
    host = [d.cpu().numpy() for d in dev]
    LocalRing(w).run_op(dev, "avg")
    out = dev[3].cpu().numpy()
    for c, (lo, hi) in enumerate(oring.chunk_bounds(n, w)):
        spans = [host[(c + k) % w][lo:hi] for k in range(w)]
        assert out[lo:hi].tobytes() == oring.reduce_chunk(spans, oring.ReduceOp.AVG, False, w).tobytes()
