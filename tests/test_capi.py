"""C ABI checks that need no GPU: the library loads, exports every symbol
include/pcclb200.h declares, and its host-only helpers agree with the oracle."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from oracle import ring as oring
from paper_2505_14065_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pcclb200.h")


def declared_symbols() -> list[str]:
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^PCCLB_API[^;(]*?\b(pcclb_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_api():
    syms = declared_symbols()
    assert "pcclb_ring_allreduce" in syms and "pcclb_simplehash_multi" in syms
    assert len(syms) >= 25


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, f"not exported: {missing}"


def test_python_signatures_cover_header():
    assert set(declared_symbols()) == set(_native.SIGNATURES)


def test_strerror_and_version():
    lib = _native.lib()
    assert lib.pcclb_strerror(0) == b"ok"
    assert b"sm_100a" in lib.pcclb_version()
    assert _native.strerror(_native.PCCLB_ENONFINITE).startswith("non-finite")


@pytest.mark.parametrize("n,w", [(10, 3), (5, 8), (268_435_456, 18), (0, 4), (1 << 28, 8), (4099, 5), (7, 1)])
def test_chunk_bounds_matches_oracle(n, w):
    out = (ctypes.c_uint64 * (2 * w))()
    assert _native.lib().pcclb_chunk_bounds(n, w, out) == 0
    got = [(out[2 * r], out[2 * r + 1]) for r in range(w)]
    assert got == oring.chunk_bounds(n, w)


def test_chunk_bounds_rejects_zero_world():
    out = (ctypes.c_uint64 * 2)()
    assert _native.lib().pcclb_chunk_bounds(10, 0, out) == _native.PCCLB_EINVAL


def test_mirror_compute_chunk_boundaries():
    from paper_2505_14065_b200.collective import compute_chunk_boundaries

    assert compute_chunk_boundaries(10, 3) == [(0, 4), (4, 7), (7, 10)]
    with pytest.raises(ValueError):
        compute_chunk_boundaries(10, 0)


def test_sass_is_sm100a_and_uses_bulk_copies():
    """The shipped cubin targets sm_100a and the hash stages through TMA bulk
    copies (UBLKCP); checked with cuobjdump when available."""
    import shutil
    import subprocess

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-lelf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass  # simplehash stages via 2-D TMA tensor copies
    # -fmad=false: kernels without a division (whose correctly rounded
    # Newton sequence legitimately uses FFMA) contain no fused multiply-add
    funcs = re.split(r"\n\s*Function : ", sass)
    checked = 0
    for f in funcs:
        name = f.split("\n", 1)[0]
        if "accumulate_kernel" in name or "dequant_acc_kernel" in name:
            assert "FFMA" not in f and "DFMA" not in f, name
            checked += 1
    assert checked >= 4


def test_ring_workspace_bytes_host_only():
    """pcclb_ring_workspace_bytes sizes the engine workspace without a GPU:
    monotone in n, covers the backup copy, and the quantized layout (per-step
    code buffers, gathered codes, ready flags) differs from the plain one."""
    lib = _native.lib()
    f = lib.pcclb_ring_workspace_bytes
    assert f(100, 0, 1, 0) == 0 and f(100, 65, 1, 0) == 0 and f(100, 2, 7, 0) == 0
    for w in (2, 3, 4, 8):
        prev = 0
        for n in (0, 1, 1000, 65536 * w + 5, 1 << 24):
            plain, quant, f64 = f(n, w, 1, 0), f(n, w, 1, 1), f(n, w, 2, 0)
            assert plain >= 16384 + 4 * n and f64 >= 16384 + 8 * n
            assert quant >= 16384 + 4 * n + w * ((n + w - 1) // w)
            assert plain >= prev
            prev = plain
    from paper_2505_14065_b200.ring_ipc import DeviceRing

    assert DeviceRing.required_bytes(1 << 20, 4, 4, True) >= f(1 << 20, 4, 1, 1)
