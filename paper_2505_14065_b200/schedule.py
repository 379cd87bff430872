"""The NVLink engine's schedule, stated in Python (csrc/ring_ipc.cu runs it).

Ring positions 0..W-1 follow the committed ring (client.py:902). Chunk c is
``compute_chunk_boundaries(N, W)[c]`` (collective.py:86-101).

Plain ops (2 barriers): position r owns chunk (r + 1) mod W, exactly the chunk
the reference rank owns after its reduce-scatter (collective.py:538). It folds
that chunk from every position's input in the reference's accumulation order
(chain positions own, own+1, ..., own-1 = r; SURVEY §0 finding 2), then every
position copies the W-1 other chunks from their owners.

Quantized ops (W barriers): the reference's ring steps (collective.py:521-565)
with u8 codes as the payload.
"""

from __future__ import annotations


def owned_chunk(pos: int, w: int) -> int:
    return (pos + 1) % w


def owner_of(chunk: int, w: int) -> int:
    return (chunk - 1) % w


def fold_chain(pos: int, w: int) -> list[int]:
    """Positions whose inputs the owner folds, in accumulation order."""
    c = owned_chunk(pos, w)
    return [(c + k) % w for k in range(w)]


def gather_sources(pos: int, w: int) -> list[tuple[int, int]]:
    """(chunk, owner position) pairs a position copies in the gather."""
    own = owned_chunk(pos, w)
    return [(c, owner_of(c, w)) for c in range(w) if c != own]


def quant_steps(pos: int, w: int) -> list[tuple[int, int]]:
    """(tx chunk, rx chunk) per reduce step (collective.py:522-523)."""
    return [((pos - s) % w, (pos - s - 1) % w) for s in range(w - 1)]


def payload_bytes(n: int, w: int, elem_bytes: int, pos: int = 0) -> int:
    """Per-position tx (= rx) payload of one all-reduce: 2(W-1) spans
    (test_ring_engine.py:99-108 traffic identity)."""
    from .collective import compute_chunk_boundaries

    b = compute_chunk_boundaries(n, w)
    size = lambda c: b[c][1] - b[c][0]  # noqa: E731
    tx = sum(size(t) for t, _ in quant_steps(pos, w))
    cur = owned_chunk(pos, w)
    for _ in range(w - 1):
        tx += size(cur)
        cur = (cur - 1) % w
    return tx * elem_bytes
