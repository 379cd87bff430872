"""Pin the CPU oracle against the reference's own outputs (golden fixtures
produced by tests/golden/make_golden.py) and the reference's known-answer
tests. CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import ring as oring
from oracle import simplehash as osh
from tests.golden.gen import RING_CASES, hash_bytes, quant_cases, ring_inputs, sha256

OPS = {"sum": oring.ReduceOp.SUM, "avg": oring.ReduceOp.AVG, "max": oring.ReduceOp.MAX, "min": oring.ReduceOp.MIN}


def test_bounds_kats(golden):
    # test_collective_units.py:18-35
    assert oring.chunk_bounds(10, 3) == [tuple(x) for x in golden["bounds"]["10_3"]]
    assert oring.chunk_bounds(5, 8) == [tuple(x) for x in golden["bounds"]["5_8"]]
    b = oring.chunk_bounds(268_435_456, 18)
    assert b == [tuple(x) for x in golden["bounds"]["268435456_18"]]
    sizes = [hi - lo for lo, hi in b]
    assert sizes.count(14_913_081) == 16 and sizes.count(14_913_080) == 2


def _hash_input(k):
    name = k["name"]
    fixed = {
        "empty": b"",
        "one_word": bytes([1, 0, 0, 0]),
        "one_byte": bytes([1]),
        "arange1000_f32": np.arange(1000, dtype=np.float32).tobytes(),
        "zeros4096": bytes(4096),
        "pattern4096": bytes((i * 131 + 4096) % 256 for i in range(4096)),
    }
    if name in fixed:
        return np.frombuffer(fixed[name], dtype=np.uint8)
    if name == "rng2_64MiB":
        return np.random.default_rng(2).integers(0, 256, 64 << 20, dtype=np.uint8)
    return hash_bytes(k["nbytes"])


def test_simplehash_c_matches_reference_kats(golden):
    for k in golden["hash"]:
        buf = _hash_input(k)
        assert sha256(buf) == k["sha256"], k["name"]
        assert osh.simplehash_c(buf) == k["hash"], k["name"]


def test_simplehash_np_and_scalar_match_reference(golden):
    for k in golden["hash"]:
        if k["nbytes"] > (4 << 20):
            continue
        buf = _hash_input(k)
        assert osh.simplehash_np(buf) == k["hash"], k["name"]
        if k["nbytes"] <= 4100:
            assert osh.simplehash_scalar(buf) == k["hash"], k["name"]


def test_simplehash_many_threads(golden):
    ks = [k for k in golden["hash"] if k["nbytes"] <= (4 << 20)]
    bufs = [_hash_input(k) for k in ks]
    assert osh.simplehash_many_c(bufs, threads=4) == [k["hash"] for k in ks]


def test_quantize_matches_reference(golden, quant_npz):
    meta = {m["name"]: m for m in golden["quant"]}
    for name, values in quant_cases():
        m = meta[name]
        assert np.array_equal(quant_npz[f"{name}__x"].view(np.uint32), values.view(np.uint32))
        codes = np.empty(values.size, dtype=np.uint8)
        if "error" in m:
            with pytest.raises(ValueError):
                oring.quantize_chunk(values, codes)
            continue
        with np.errstate(all="ignore"):
            mn, sc = oring.quantize_chunk(values, codes)
            back = np.empty(values.size, dtype=np.float32)
            oring.dequantize_into(codes, mn, sc, back)
        assert (mn, sc) == (m["min"], m["scale"]), name
        assert np.array_equal(codes, quant_npz[f"{name}__q"]), name
        assert back.tobytes() == quant_npz[f"{name}__d"].tobytes(), name


def _case_inputs(c):
    bufs = ring_inputs(c["w"], c["n"], np.dtype(c["dtype"]), c["seed"])
    assert sha256(np.concatenate(bufs) if c["n"] else b"") == c["input_sha256"]
    return bufs


@pytest.mark.parametrize("idx", range(0, len(RING_CASES)))
def test_ring_oracle_matches_reference(golden, idx):
    c = golden["ring"][idx]
    assert (c["w"], c["n"], c["op"], c["quantize"], c["dtype"], c["seed"]) == RING_CASES[idx]
    bufs = _case_inputs(c)
    out = oring.ring_allreduce(bufs, OPS[c["op"]], quantize=c["quantize"])
    assert {osh.simplehash_np(o) for o in out} == {c["output_hash"]}
    # the per-chunk closed form is the same function
    closed = oring.ring_allreduce_chunkwise(bufs, OPS[c["op"]], quantize=c["quantize"])
    assert closed.tobytes() == out[0].tobytes()


def test_appendix_c_goldens(golden):
    rng = np.random.default_rng(0)
    inputs = [rng.normal(0, 1, 1 << 24).astype(np.float32) for _ in range(8)]
    want = golden["appendix_c_w8_avg_16M"]
    for quant, key in ((False, "plain"), (True, "quant")):
        out = oring.ring_allreduce_chunkwise(inputs, oring.ReduceOp.AVG, quantize=quant)
        assert osh.simplehash_c(out) == want[key]


def test_outer_oracle_matches_reference_expressions():
    """oracle/outer.py is the reference's own NumPy sequence (algos.py:93-100);
    check it against a literal transcription on random data."""
    from oracle import outer as oouter

    rng = np.random.default_rng(1)
    p = rng.normal(0, 1, 1001).astype(np.float32)
    d = rng.normal(0, 1, 1001).astype(np.float32)
    v = rng.normal(0, 1, 1001).astype(np.float32)
    p2, v2 = p.copy(), v.copy()
    oouter.nesterov_step(p, d, v, 0.5, 0.9)
    lr, mu = np.float32(0.5), np.float32(0.9)
    v2 = v2 * mu
    v2 = v2 + d
    p2 = p2 - lr * (d + mu * v2)
    assert p.tobytes() == p2.tobytes() and v.tobytes() == v2.tobytes()


def _outer_replay(n, oouter):
    rng = np.random.default_rng(n)
    g = rng.normal(0, 1, n).astype(np.float32)
    vel = np.zeros(n, np.float32)
    for step in range(4):
        local = g - rng.normal(0, 1e-2, n).astype(np.float32) * np.float32(step + 1)
        d = oouter.pseudo_gradient(g, local)
        oouter.nesterov_step(g, d, vel, 0.7, 0.9)
        grad = rng.normal(0, 1, n).astype(np.float32)
        oouter.sgd_step(g, grad, 2.0**-6)
    return g, vel


def test_outer_oracle_matches_reference_run(golden):
    """oracle/outer.py reproduces churncomm.algos' optimizers (golden.json 'outer')."""
    from oracle import outer as oouter

    for n, want in golden["outer"].items():
        g, vel = _outer_replay(int(n), oouter)
        assert osh.simplehash_c(g) == want["params"]
        assert osh.simplehash_c(vel) == want["velocity"]


@pytest.mark.parametrize("w", [2, 3, 4, 8])
@pytest.mark.parametrize("quant", [False, True])
def test_prod_extension_closed_form_matches_ring(w, quant):
    """The PROD extension (parity unpinned: no reference op) is defined as the
    reference's ring with np.multiply; the chunk closed form agrees with the
    full ring simulation, as it does for the reference's own ops."""
    rng = np.random.default_rng(w)
    bufs = [(1.0 + 0.05 * rng.normal(0, 1, 4099)).astype(np.float32) for _ in range(w)]
    ring = oring.ring_allreduce([b.copy() for b in bufs], oring.ReduceOp.PROD, quantize=quant)
    closed = oring.ring_allreduce_chunkwise(bufs, oring.ReduceOp.PROD, quantize=quant)
    for out in ring:
        assert out.tobytes() == closed.tobytes()
