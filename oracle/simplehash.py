"""simplehash oracle -- TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

``simplehash_np`` restates ``src/churncomm/sharedstate.py:45-105`` in NumPy
(lane matrix rounds, ``:57-72``; tree fold ``:75-84``). ``simplehash_c`` and
``simplehash_many_c`` call the plain-C restatement in ``oracle/simplehash.c``
(built by ``oracle/Makefile`` into ``oracle/_build/liboracle.so``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

FNV_OFFSET = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3
LANES = 256
TREE_DEPTH = 8
ROTATE = 27
_MASK64 = (1 << 64) - 1

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def _as_u8(buffer) -> np.ndarray:
    if isinstance(buffer, np.ndarray):
        return np.ascontiguousarray(buffer).reshape(-1).view(np.uint8)
    return np.frombuffer(memoryview(buffer).cast("B"), dtype=np.uint8)


def simplehash_np(buffer) -> int:
    """sharedstate.py:87-105 with workers=1."""
    data = _as_u8(buffer)
    n = data.size
    full = n // 4
    words = data[: full * 4].view("<u4")
    if n % 4:
        tail = np.zeros(4, dtype=np.uint8)
        tail[: n % 4] = data[full * 4 :]
        words = np.concatenate([words, tail.view("<u4")])
    lanes = np.full(LANES, FNV_OFFSET, dtype=np.uint64)
    prime = np.uint64(FNV_PRIME)
    rounds = words.size // LANES
    if rounds:
        mat = words[: rounds * LANES].reshape(rounds, LANES)
        for r in range(rounds):
            np.bitwise_xor(lanes, mat[r].astype(np.uint64), out=lanes)
            np.multiply(lanes, prime, out=lanes)
    rem = words.size - rounds * LANES
    if rem:
        part = lanes[:rem]
        np.bitwise_xor(part, words[rounds * LANES :].astype(np.uint64), out=part)
        np.multiply(part, prime, out=part)
    level = lanes
    rot, inv = np.uint64(ROTATE), np.uint64(64 - ROTATE)
    for _ in range(TREE_DEPTH):
        a = level[0::2].copy()
        b = level[1::2]
        np.bitwise_xor(a, (b << rot) | (b >> inv), out=a)
        np.multiply(a, prime, out=a)
        level = a
    return int(level[0]) ^ n


def simplehash_scalar(buffer) -> int:
    """sharedstate.py:108-128 (normative scalar form); small inputs only."""
    raw = bytes(_as_u8(buffer))
    n = len(raw)
    if n % 4:
        raw += b"\x00" * (4 - n % 4)
    lanes = [FNV_OFFSET] * LANES
    for i in range(len(raw) // 4):
        w = int.from_bytes(raw[4 * i : 4 * i + 4], "little")
        lanes[i % LANES] = ((lanes[i % LANES] ^ w) * FNV_PRIME) & _MASK64
    level = lanes
    for _ in range(TREE_DEPTH):
        level = [
            ((a ^ (((b << ROTATE) | (b >> (64 - ROTATE))) & _MASK64)) * FNV_PRIME) & _MASK64
            for a, b in zip(level[0::2], level[1::2])
        ]
    return level[0] ^ n


def build() -> str:
    """Compile oracle/simplehash.c (gcc -O2) if needed; returns the .so path."""
    src = os.path.join(_HERE, "simplehash.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.oracle_simplehash.restype = ctypes.c_uint64
        lib.oracle_simplehash.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        lib.oracle_simplehash_many.restype = ctypes.c_int
        lib.oracle_simplehash_many.argtypes = [
            ctypes.POINTER(ctypes.c_void_p),
            ctypes.POINTER(ctypes.c_uint64),
            ctypes.c_uint32,
            ctypes.POINTER(ctypes.c_uint64),
            ctypes.c_int,
        ]
        _lib = lib
    return _lib


def simplehash_c(buffer) -> int:
    data = _as_u8(buffer)
    return int(_load().oracle_simplehash(data.ctypes.data, data.size))


def simplehash_many_c(buffers, threads: int = 1) -> list[int]:
    arrs = [_as_u8(b) for b in buffers]
    n = len(arrs)
    ptrs = (ctypes.c_void_p * n)(*[a.ctypes.data for a in arrs])
    sizes = (ctypes.c_uint64 * n)(*[a.size for a in arrs])
    out = (ctypes.c_uint64 * n)()
    if _load().oracle_simplehash_many(ptrs, sizes, n, out, threads) != 0:
        raise RuntimeError("oracle_simplehash_many failed")
    return [int(v) for v in out]
