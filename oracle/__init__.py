"""CPU oracle for the PCCL collective data plane — TEST INFRASTRUCTURE ONLY.

This package restates, in NumPy and plain C, the reference algorithm of the
hot path (ring all-reduce chunk arithmetic and ``simplehash``) so that the
CUDA product can be checked against it. Every function cites the reference
``file:line`` it follows (paths relative to ``/root/reference/pkg``).

Parity pinning: the restatement is checked against golden vectors produced by
running the reference itself (``tests/golden/make_golden.py`` imports
``churncomm`` from ``/root/reference``) and against the reference's own
known-answer tests (``tests/test_hash.py``, ``tests/test_collective_units.py``,
``tests/test_ring_engine.py``). See ``tests/test_oracle_golden.py``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline. The product (``paper_2505_14065_b200``) never imports
it: there is no CPU fallback on the hot path.
"""
