"""ctypes binding of libpcclb200.so (the C ABI in include/pcclb200.h).

The library is built in-tree by ``paper_2505_14065_b200/csrc/Makefile``
(``python -c "import __graft_entry__ as g; g.build()"``). There is no CPU
fallback: if the library is missing every product entry point raises
``NativeLibraryMissing``.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libpcclb200.so")
CSRC = os.path.join(_HERE, "csrc")

PCCLB_OK = 0
PCCLB_EINVAL = 1
PCCLB_ECUDA = 2
PCCLB_EABORTED = 3
PCCLB_ETIMEOUT = 4
PCCLB_ENONFINITE = 5
PCCLB_EIO = 6
PCCLB_ENOMEM = 7

F32 = 1
F64 = 2


class NativeLibraryMissing(RuntimeError):
    pass


class NativeError(RuntimeError):
    def __init__(self, status: int, what: str, cuda_error: int = 0):
        msg = f"{what}: {strerror(status)} (status {status}"
        if status == PCCLB_ECUDA:
            msg += f", cudaError {cuda_error}"
        super().__init__(msg + ")")
        self.status = status
        self.cuda_error = cuda_error


class Range(ctypes.Structure):
    _fields_ = [
        ("kmin_inv", ctypes.c_uint32),
        ("kmax", ctypes.c_uint32),
        ("nonfinite", ctypes.c_uint32),
        ("seen", ctypes.c_uint32),
    ]


class QMeta(ctypes.Structure):
    _fields_ = [("min_val", ctypes.c_float), ("scale", ctypes.c_float)]


class Stats(ctypes.Structure):
    _fields_ = [
        ("tx_payload_bytes", ctypes.c_uint64),
        ("rx_payload_bytes", ctypes.c_uint64),
        ("n_phases", ctypes.c_uint32),
        ("phase_ms", ctypes.c_float * 47),
    ]


_P = ctypes.c_void_p
_U64 = ctypes.c_uint64
_U32 = ctypes.c_uint32
_I = ctypes.c_int

# name -> (restype, argtypes); mirrors include/pcclb200.h
SIGNATURES = {
    "pcclb_strerror": (ctypes.c_char_p, [_I]),
    "pcclb_last_cuda_error": (_I, []),
    "pcclb_version": (ctypes.c_char_p, []),
    "pcclb_chunk_bounds": (_I, [_U64, _U32, ctypes.POINTER(_U64)]),
    "pcclb_accumulate": (_I, [_P, _P, _U64, _I, _I, _P]),
    "pcclb_finalize": (_I, [_P, _U64, _I, _I, _U32, _P]),
    "pcclb_range_reset": (_I, [_P, _U32, _P]),
    "pcclb_range_f32": (_I, [_P, _U64, _P, _P]),
    "pcclb_quantize_u8": (_I, [_P, _U64, _P, _P, _P, _P, _U32, _P]),
    "pcclb_dequantize_u8": (_I, [_P, _P, _U64, _P, _U32, _P]),
    "pcclb_dequant_accumulate_u8": (_I, [_P, _P, _U64, _P, _I, _P, _P]),
    "pcclb_quantize_ex": (_I, [_P, _U64, _P, _P, _P, _P, _U32, _I, _P]),
    "pcclb_dequantize_ex": (_I, [_P, _P, _U64, _P, _U32, _I, _P]),
    "pcclb_dequant_accumulate_ex": (_I, [_P, _P, _U64, _P, _I, _P, _I, _P]),
    "pcclb_simplehash": (_I, [_P, _U64, _P, _P]),
    "pcclb_simplehash_multi": (_I, [ctypes.POINTER(_P), ctypes.POINTER(_U64), _U32, _P, _P]),
    "pcclb_crc32": (_I, [_P, _U64, _P, _P]),
    "pcclb_crc32_multi": (_I, [ctypes.POINTER(_P), ctypes.POINTER(_U64), _U32, _P, _P]),
    "pcclb_simplehash_init": (_I, [_P, _P]),
    "pcclb_simplehash_update": (_I, [_P, _P, _U64, _P]),
    "pcclb_simplehash_final": (_I, [_P, _U64, _P, _P]),
    "pcclb_pseudo_gradient_f32": (_I, [_P, _P, _P, _U64, _P]),
    "pcclb_outer_sgd_f32": (_I, [_P, _P, _U64, ctypes.c_float, _P]),
    "pcclb_outer_nesterov_f32": (_I, [_P, _P, _P, _U64, ctypes.c_float, ctypes.c_float, _P]),
    "pcclb_local_scratch_bytes": (_U64, [_U32]),
    "pcclb_local_allreduce": (_I, [ctypes.POINTER(_P), _U32, _U64, _I, _I, _I, _P, _P, _P]),
    "pcclb_local_allreduce_ex": (_I, [ctypes.POINTER(_P), _U32, _U64, _I, _I, _I, _P, _P, _P]),
    "pcclb_ring_create": (_I, [_I, _U32, _U32, _U64, ctypes.POINTER(_P)]),
    "pcclb_ring_export": (_I, [_P, _P]),
    "pcclb_ring_import": (_I, [_P, _U32, _P]),
    "pcclb_ring_abort_word": (ctypes.POINTER(ctypes.c_uint64), [_P]),
    "pcclb_ring_capacity": (_U64, [_P, _I, _I]),
    "pcclb_ring_set_slots": (_I, [_P, _U32]),
    "pcclb_ring_set_small_max": (_I, [_P, _U64]),
    "pcclb_ring_workspace_bytes": (_U64, [_U64, _U32, _I, _I]),
    "pcclb_ring_allreduce": (
        _I,
        [_P, _P, _U64, _I, _I, _I, _U64, _I, ctypes.c_double, ctypes.POINTER(Stats), _P],
    ),
    "pcclb_ring_restore": (_I, [_P, _P, _U64, _I, _P]),
    "pcclb_ring_enqueue": (
        _I,
        [_P, _P, _U64, _I, _I, _I, _U64, _I, ctypes.c_double, _P, ctypes.POINTER(_U32)],
    ),
    "pcclb_ring_wait": (_I, [_P, _U32, ctypes.POINTER(Stats)]),
    "pcclb_ring_destroy": (None, [_P]),
    "pcclb_ipc_handle": (_I, [_P, _P, ctypes.POINTER(_U64)]),
    "pcclb_ring_register": (_I, [_P, _U32, _P, _U64, _P, ctypes.POINTER(_U64)]),
    "pcclb_ring_deregister": (_I, [_P, _U32]),
    "pcclb_ipc_open": (_I, [_P, ctypes.POINTER(_P)]),
    "pcclb_ipc_close": (_I, [_P]),
    "pcclb_copy": (_I, [_P, _P, _U64, _P]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """The loaded library (raises NativeLibraryMissing if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} not built; run `make -C {CSRC}` "
                    "(there is no CPU fallback for the pcclb200 data plane)"
                )
            handle = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name, None)
                if fn is None:
                    continue  # reported by tests/test_capi.py
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def strerror(status: int) -> str:
    try:
        return lib().pcclb_strerror(status).decode()
    except NativeLibraryMissing:
        return f"status {status}"


def check(status: int, what: str) -> None:
    if status != PCCLB_OK:
        raise NativeError(status, what, lib().pcclb_last_cuda_error())
