"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the dev container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``churncomm`` from /root/reference/pkg/src and the reference test
helpers (``oracles.py``, ``ring_harness.py``) from /root/reference/pkg/tests,
and records their outputs. The fixtures are committed; nothing at test time
reads /root/reference. Inputs are regenerated from seeds at test time and
checked against the sha256 recorded here.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path[:0] = [REF_SRC, REF_TESTS]
sys.dont_write_bytecode = True

from churncomm.collective import (  # noqa: E402
    ReduceOp,
    compute_chunk_boundaries,
    dequantize_into,
    quantize_chunk,
)
from churncomm.sharedstate import simplehash, simplehash_reference  # noqa: E402
from oracles import ring_allreduce_oracle  # noqa: E402
from ring_harness import run_single_op  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from tests.golden.gen import (  # noqa: E402
    HASH_LENGTHS,
    RING_CASES,
    hash_bytes,
    quant_cases,
    ring_inputs,
    sha256,
    edge_pairs,
)

OPS = {"sum": ReduceOp.SUM, "avg": ReduceOp.AVG, "max": ReduceOp.MAX, "min": ReduceOp.MIN}


def make_hash():
    kats = []
    fixed = {
        "empty": b"",
        "one_word": bytes([1, 0, 0, 0]),
        "one_byte": bytes([1]),
        "arange1000_f32": np.arange(1000, dtype=np.float32).tobytes(),
        "zeros4096": bytes(4096),
        "pattern4096": bytes((i * 131 + 4096) % 256 for i in range(4096)),
    }
    for name, buf in fixed.items():
        h = simplehash_reference(buf)
        assert simplehash(buf) == h
        kats.append({"name": name, "nbytes": len(buf), "sha256": sha256(buf), "hash": h})
    big = np.random.default_rng(2).integers(0, 256, 64 << 20, dtype=np.uint8)
    kats.append({"name": "rng2_64MiB", "nbytes": big.size, "sha256": sha256(big), "hash": simplehash(big)})
    for n in HASH_LENGTHS:
        buf = hash_bytes(n)
        h = simplehash(buf)
        if n <= 4100:
            assert simplehash_reference(buf) == h
        kats.append({"name": f"rand{n}", "nbytes": n, "sha256": sha256(buf), "hash": h})
    return kats


def make_quant():
    out = {}
    meta = []
    for name, values in quant_cases():
        codes = np.empty(values.size, dtype=np.uint8)
        try:
            mn, sc = quantize_chunk(values, codes)
        except ValueError:
            meta.append({"name": name, "error": "ValueError"})
            out[f"{name}__x"] = values
            continue
        back = np.empty(values.size, dtype=np.float32)
        dequantize_into(codes, mn, sc, back)
        out[f"{name}__x"] = values
        out[f"{name}__q"] = codes
        out[f"{name}__d"] = back
        meta.append({"name": name, "min": mn, "scale": sc})
    return out, meta


def make_edges():
    out = {}
    for dt in (np.float32, np.float64):
        a, b = edge_pairs(dt)
        tag = np.dtype(dt).name
        out[f"{tag}__a"] = a
        out[f"{tag}__b"] = b
        for opname, fn in (("add", np.add), ("max", np.maximum), ("min", np.minimum)):
            r = a.copy()
            with np.errstate(all="ignore"):
                fn(r, b, out=r)
            out[f"{tag}__{opname}"] = r
        for w in (3, 7):
            r = a.copy()
            with np.errstate(all="ignore"):
                np.divide(r, r.dtype.type(w), out=r)
            out[f"{tag}__div{w}"] = r
    return out


def make_ring():
    cases = []
    engine_checked = 0
    for case in RING_CASES:
        w, n, opname, quant, dtname, seed = case
        bufs = ring_inputs(w, n, np.dtype(dtname), seed)
        expected = ring_allreduce_oracle([b.copy() for b in bufs], OPS[opname], quantize=quant)
        hashes = [simplehash(e) for e in expected]
        assert len(set(hashes)) == 1
        # pin the oracle to the real threaded engine on small cases
        # (W == 1 never reaches the engine: client.py:896-900 finalizes only)
        if n <= 4099 and 2 <= w <= 5:
            live = [b.copy() for b in bufs]
            res = run_single_op(live, OPS[opname], quantize=quant)
            assert all(s == "ok" for s, _ in res)
            assert [simplehash(x) for x in live] == hashes, case
            engine_checked += 1
        cases.append(
            {
                "w": w,
                "n": n,
                "op": opname,
                "quantize": quant,
                "dtype": dtname,
                "seed": seed,
                "input_sha256": sha256(np.concatenate(bufs) if n else b""),
                "output_hash": hashes[0],
            }
        )
    return cases, engine_checked


def make_appendix_c():
    rng = np.random.default_rng(0)
    inputs = [rng.normal(0, 1, 1 << 24).astype(np.float32) for _ in range(8)]
    res = {}
    for quant in (False, True):
        out = ring_allreduce_oracle(inputs, ReduceOp.AVG, quantize=quant)
        hs = {simplehash(o) for o in out}
        assert len(hs) == 1
        res["quant" if quant else "plain"] = hs.pop()
    return res


def make_outer():
    """Run the reference's own outer optimizers (algos.py:75-105) on seeded
    data: 4 outer steps of pseudo-gradient + Nesterov, each followed by one
    PlainSGD step."""
    from churncomm.algos import NesterovOuter, PlainSGD

    out = {}
    for n in (7, 4099):
        rng = np.random.default_rng(n)
        g = rng.normal(0, 1, n).astype(np.float32)
        opt = NesterovOuter(n, lr=0.7, momentum=0.9)
        sgd = PlainSGD(2.0**-6)
        for step in range(4):
            local = g - rng.normal(0, 1e-2, n).astype(np.float32) * np.float32(step + 1)
            delta = g - local  # algos.py:236
            opt.step(g, delta)
            grad = rng.normal(0, 1, n).astype(np.float32)
            sgd.step(g, grad)
        out[str(n)] = {"params": simplehash(g), "velocity": simplehash(opt.velocity)}
    return out


def main():
    fixtures = {}
    fixtures["bounds"] = {
        "10_3": compute_chunk_boundaries(10, 3),
        "5_8": compute_chunk_boundaries(5, 8),
        "268435456_18": compute_chunk_boundaries(268_435_456, 18),
    }
    fixtures["hash"] = make_hash()
    qarrays, qmeta = make_quant()
    fixtures["quant"] = qmeta
    np.savez_compressed(os.path.join(HERE, "quant.npz"), **qarrays)
    np.savez_compressed(os.path.join(HERE, "edges.npz"), **make_edges())
    ring, engine_checked = make_ring()
    fixtures["ring"] = ring
    fixtures["ring_engine_checked"] = engine_checked
    fixtures["appendix_c_w8_avg_16M"] = make_appendix_c()
    fixtures["outer"] = make_outer()
    fixtures["generator"] = {
        "reference": "/root/reference/pkg (churncomm, pure Python/NumPy)",
        "numpy": np.__version__,
        "python": sys.version.split()[0],
    }
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(fixtures, f, indent=1)
    print(f"ring cases: {len(ring)} (engine-checked {engine_checked}); hash KATs: {len(fixtures['hash'])}")


if __name__ == "__main__":
    main()
