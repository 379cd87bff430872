"""Deterministic input generators shared by make_golden.py and the tests.

The golden fixtures record the reference's outputs together with the sha256
of the inputs generated here, so a test can regenerate the inputs (NumPy
``default_rng`` streams) and verify they are the very bytes the reference saw.
"""

from __future__ import annotations

import hashlib

import numpy as np

# byte lengths for hash KATs: small exhaustive-ish, round boundaries, big
HASH_LENGTHS = (
    list(range(0, 70))
    + [1020, 1021, 1022, 1023, 1024, 1025, 1026, 1027, 1028, 2047, 2048, 2049, 4095, 4096, 4097]
    + [4100, 8191, 65536 + 3, 262144 - 1, 1 << 20, (1 << 20) + 5, 3 * (1 << 20) + 1022]
)


def sha256(buf) -> str:
    if isinstance(buf, np.ndarray):
        buf = np.ascontiguousarray(buf).tobytes()
    return hashlib.sha256(bytes(buf)).hexdigest()


def hash_bytes(n: int) -> np.ndarray:
    return np.random.default_rng(1000 + n).integers(0, 256, n, dtype=np.uint8)


def _ring_cases():
    cases = []
    seed = 0
    for w in (1, 2, 3, 4, 5, 8):
        for n in (0, 1, 2, 7, 1024, 4099):
            for op in ("sum", "avg", "max", "min"):
                for quant in (False, True):
                    seed += 1
                    cases.append((w, n, op, quant, "float32", seed))
    for w in (2, 3, 5):
        for n in (1, 513, 4099):
            for op in ("sum", "avg", "max", "min"):
                seed += 1
                cases.append((w, n, op, False, "float64", seed))
    for op in ("sum", "avg", "max", "min"):
        for quant in (False, True):
            seed += 1
            cases.append((8, (1 << 16) + 3, op, quant, "float32", seed))
    # integer-valued inputs with signed zeros: exercises max/min tie rules
    for w in (2, 3, 5):
        for op in ("max", "min", "sum"):
            seed += 1
            cases.append((w, 1024, op, False, "float32", 100000 + seed))
            seed += 1
            cases.append((w, 1024, op, False, "float64", 100000 + seed))
    return cases


RING_CASES = _ring_cases()


def ring_inputs(w: int, n: int, dtype: np.dtype, seed: int) -> list[np.ndarray]:
    """Per-rank inputs in ring-position order, drawn from one generator."""
    rng = np.random.default_rng(seed)
    if seed >= 100000:  # ties kind
        out = []
        for _ in range(w):
            v = rng.integers(-3, 4, n).astype(dtype)
            neg = rng.random(n) < 0.5
            v[(v == 0) & neg] = -0.0
            out.append(v)
        return out
    return [rng.normal(0, 10, n).astype(dtype) for _ in range(w)]


def quant_cases() -> list[tuple[str, np.ndarray]]:
    f = np.float32
    rng = np.random.default_rng(77)
    cases = [
        ("constant", np.array([5.0, 5.0, 5.0], f)),
        ("arange256", np.arange(256, dtype=f)),
        ("ties", np.array([0.0, 255.0, 0.5, 1.5, 2.5, 254.5, 127.5, 3.5, 4.5], f)),
        ("single", np.array([3.25], f)),
        ("empty", np.array([], f)),
        ("neg_zero", np.array([-0.0, 0.0, 1.0, -1.0, -0.0], f)),
        ("subnormal_range", np.array([1e-45, 2e-45, 1e-45, 0.0], f)),
        ("tiny_range", np.array([1.0, np.nextafter(f(1.0), f(2.0)), 1.0], f)),
        ("huge_range", np.array([-3e38, 3e38, 0.0, 1e38, -1e38], f)),
        ("nonfinite_nan", np.array([1.0, np.nan], f)),
        ("nonfinite_inf", np.array([1.0, np.inf], f)),
    ]
    for i, n in enumerate([1, 2, 3, 7, 63, 64, 65, 1000, 4099, 70001]):
        scale = 10.0 ** rng.uniform(-3, 3)
        cases.append((f"normal{i}_{n}", rng.normal(0, scale, n).astype(f)))
    cases.append(("diloco_delta", rng.normal(0, 1e-2, 65536).astype(f)))
    mags = rng.normal(0, 1, 5000) * 10.0 ** rng.uniform(-30, 30, 5000)
    cases.append(("mixed_magnitudes", mags.astype(f)))
    return cases


def _bits(dt, vals):
    it = np.uint32 if dt == np.float32 else np.uint64
    return np.array(vals, dtype=it).view(dt)


def edge_pairs(dt) -> tuple[np.ndarray, np.ndarray]:
    """(a, b) element pairs covering single-NaN propagation with payloads,
    signed-zero ties, equal values, infinities, subnormals and random values.
    Both-NaN and signalling-NaN pairs are excluded: NumPy's own result for
    them depends on the SIMD lane (parity unpinned)."""
    rng = np.random.default_rng(5)
    if dt == np.float32:
        qa, qb = _bits(dt, [0x7FC00011, 0xFFC01234])
        sub = _bits(dt, [0x00000001, 0x80000005, 0x007FFFFF])
    else:
        qa, qb = _bits(dt, [0x7FF8000000000011, 0xFFF8000000001234])
        sub = _bits(dt, [0x1, 0x8000000000000005, 0x000FFFFFFFFFFFFF])
    inf = dt(np.inf)
    base_a = [qa, 1.0, qb, -2.0, 0.0, -0.0, 0.0, -0.0, inf, inf, -inf, 3.0, 3.0, sub[0], sub[1], sub[2], 1e30, -5.5]
    base_b = [1.0, qa, 7.0, qb, -0.0, 0.0, 0.0, -0.0, -inf, inf, 2.0, 3.0, -3.0, sub[1], sub[2], sub[0], 1e30, -5.5]
    a = np.array(base_a, dtype=dt)
    b = np.array(base_b, dtype=dt)
    # repeat so both SIMD bodies and scalar tails see every pattern
    reps = 73
    a = np.tile(a, reps)
    b = np.tile(b, reps)
    ra = rng.normal(0, 1, 1001).astype(dt)
    rb = rng.normal(0, 1, 1001).astype(dt)
    return np.concatenate([a, ra]), np.concatenate([b, rb])


# Reference wire transcripts (tests/golden/make_wire_golden.py):
# (world, n, op, quantize, dtype, seed, chunk_bytes)
WIRE_CASES = [
    (2, 1000, "sum", False, "float32", 11, 256),
    (3, 1000, "avg", False, "float32", 12, 256),
    (3, 1001, "max", False, "float64", 13, 512),
    (4, 999, "min", False, "float32", 14, 1024),
    (3, 2, "sum", False, "float32", 15, 256),
    (1, 100, "avg", False, "float32", 23, 256),
    (2, 1000, "avg", True, "float32", 16, 256),
    (3, 1000, "sum", True, "float32", 17, 300),
    (4, 1003, "max", True, "float32", 18, 256),
    (3, 2, "avg", True, "float32", 19, 256),
    (3, 997, "min", True, "float32", 100019, 128),
    (5, 5000, "avg", True, "float32", 20, 1024),
    (5, 5000, "avg", False, "float64", 21, 2048),
]
