"""Pin the oracle against the live reference on seeded random cases (beside
the committed golden fixtures): the ring schedule against the reference's own
test oracle (pkg/tests/oracles.py:30-101, which calls the reference's
collective.py kernels) and simplehash against churncomm.sharedstate.simplehash
(sharedstate.py:87-105). Needs /root/reference (this container), skipped
elsewhere; CPU only, a few seconds."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present")


@pytest.fixture(scope="module")
def ref():
    sys.dont_write_bytecode = True  # the reference tree is read-only
    for p in (os.path.join(REF, "src"), os.path.join(REF, "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    import oracles as ref_oracles
    from churncomm import sharedstate as ref_ss
    from churncomm.collective import ReduceOp as RefOp

    return ref_oracles, ref_ss, RefOp


def _cases(count, seed):
    rng = np.random.default_rng(seed)
    for _ in range(count):
        w = int(rng.choice([1, 2, 3, 4, 5, 7, 8]))
        n = int(rng.choice([0, 1, w - 1 if w > 1 else 1, 17, 1000, int(rng.integers(1, 70_000))]))
        op = str(rng.choice(["SUM", "AVG", "MAX", "MIN"]))
        quant = bool(rng.integers(0, 2))
        dtype = np.float32 if quant or rng.integers(0, 4) else np.float64
        scale = float(rng.choice([1e-3, 1.0, 1e3]))
        bufs = [(rng.normal(0, scale, n)).astype(dtype) for _ in range(w)]
        if n and rng.integers(0, 4) == 0:  # signed-zero ties for MAX/MIN
            for b in bufs:
                b[rng.integers(0, n, max(1, n // 10))] = rng.choice([0.0, -0.0])
        yield w, n, op, quant, bufs


@pytest.mark.parametrize("seed", range(6))
def test_ring_oracle_matches_reference_oracle(ref, seed):
    from oracle import ring as oring

    ref_oracles, _, RefOp = ref
    for w, n, op, quant, bufs in _cases(12, 1000 + seed):
        want = ref_oracles.ring_allreduce_oracle([b.copy() for b in bufs], RefOp[op], quantize=quant)
        got = oring.ring_allreduce([b.copy() for b in bufs], oring.ReduceOp[op], quantize=quant)
        for r in range(w):
            assert got[r].tobytes() == want[r].tobytes(), (w, n, op, quant, r)
        # the per-chunk closed form the config-size checks stream through
        closed = oring.ring_allreduce_chunkwise(bufs, oring.ReduceOp[op], quantize=quant)
        assert all(closed.tobytes() == want[r].tobytes() for r in range(w)), (w, n, op, quant)


@pytest.mark.parametrize("seed", range(4))
def test_simplehash_oracles_match_reference(ref, seed):
    from oracle import simplehash as osh

    _, ref_ss, _ = ref
    rng = np.random.default_rng(2000 + seed)
    sizes = [0, 1, 3, 4, 5, 1023, 1024, 1025, 4096 + 3, int(rng.integers(1, 1 << 20))]
    bufs = [rng.integers(0, 256, s, dtype=np.uint8) for s in sizes]
    want = [ref_ss.simplehash(b) for b in bufs]
    assert osh.simplehash_many_c(bufs, threads=2) == want
    assert [osh.simplehash_np(b) for b in bufs] == want
