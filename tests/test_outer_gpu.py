"""Outer-optimizer steps on the GPU vs the reference's NumPy sequence
(algos.py:75-105), bit-exact over several DiLoCo-like outer steps."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import outer as oouter
from tests.gpu_util import bits, need_gpu, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


@pytest.mark.parametrize("n", [1, 7, 4099, 1_000_003])
def test_nesterov_and_sgd_bit_exact(n):
    from paper_2505_14065_b200.outer import NesterovOuter, PlainSGD, pseudo_gradient

    rng = np.random.default_rng(n)
    g = rng.normal(0, 1, n).astype(np.float32)
    vel = np.zeros(n, np.float32)
    dg, dvel_opt = to_dev(g), NesterovOuter(n, lr=0.7, momentum=0.9)
    sgd = PlainSGD(2.0**-6)
    for step in range(4):
        local = g - rng.normal(0, 1e-2, n).astype(np.float32) * np.float32(step + 1)
        # pseudo-gradient + Nesterov step (algos.py:334, :98-100)
        d_np = oouter.pseudo_gradient(g, local)
        d_gpu = pseudo_gradient(dg, to_dev(local))
        assert bits(d_gpu) == bits(d_np)
        oouter.nesterov_step(g, d_np, vel, 0.7, 0.9)
        dvel_opt.step(dg, d_gpu)
        assert bits(dg) == bits(g)
        assert bits(dvel_opt.velocity) == bits(vel)
        # an inner SGD step (algos.py:83-84)
        grad = rng.normal(0, 1, n).astype(np.float32)
        oouter.sgd_step(g, grad, 2.0**-6)
        sgd.step(dg, to_dev(grad))
        assert bits(dg) == bits(g)


def test_misaligned_views():
    from paper_2505_14065_b200.outer import pseudo_gradient

    rng = np.random.default_rng(3)
    a = rng.normal(0, 1, 10_001).astype(np.float32)
    b = rng.normal(0, 1, 10_001).astype(np.float32)
    da, db = to_dev(a)[1:], to_dev(b)[3:]
    out = pseudo_gradient(da[: db.numel()], db)
    assert bits(out) == bits(a[1 : 1 + db.numel()] - b[3:])
