"""pcclb200 -- B200-native data plane for PCCL's collectives.

Drop-in for the hot path of the reference (``churncomm``, arXiv 2505.14065):
the ring all-reduce chunk arithmetic behind ``all_reduce_async`` and the
``simplehash`` behind ``sync_shared_state``, as hand-written sm_100a kernels
behind a C ABI (include/pcclb200.h), bit-identical to the reference.
"""

from .collective import (  # noqa: F401
    CollectiveAborted,
    ReduceOp,
    UsageError,
    accumulate,
    compute_chunk_boundaries,
    dequantize_into,
    finalize_reduction,
    quantize_chunk,
)
from .ring import LocalRing  # noqa: F401
from .sharedstate import SharedStateEntry, crc32, crc32_many, digest_entries, simplehash, simplehash_many  # noqa: F401

__version__ = "0.1.0"
