"""simplehash on the GPU vs the reference's known answers and the oracle."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import simplehash as osh
from tests.golden.gen import hash_bytes
from tests.gpu_util import need_gpu, to_dev
from tests.test_oracle_golden import _hash_input

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu():
    need_gpu()


def test_kats_one_by_one(golden):
    from paper_2505_14065_b200 import simplehash

    for k in golden["hash"]:
        buf = to_dev(_hash_input(k))
        assert simplehash(buf) == k["hash"], k["name"]


def test_kats_multi_entry_single_launch(golden):
    from paper_2505_14065_b200 import simplehash_many

    ks = golden["hash"]
    bufs = [to_dev(_hash_input(k)) for k in ks]
    assert simplehash_many(bufs) == [k["hash"] for k in ks]


@pytest.mark.parametrize("offset", list(range(1, 16)))
def test_misaligned_views(offset):
    from paper_2505_14065_b200 import simplehash

    raw = hash_bytes(300_000 + offset)
    d = to_dev(raw)
    for start in (offset, offset + 1024):
        view = d[start:]
        assert simplehash(view) == osh.simplehash_c(raw[start:])


def test_dtype_agnostic_raw_bytes():
    from paper_2505_14065_b200 import simplehash

    x = torch.randn(12345, dtype=torch.bfloat16, device="cuda")
    raw = x.view(torch.uint8).cpu().numpy()
    assert simplehash(x) == osh.simplehash_c(raw)


def test_host_buffers_stream_through_device(golden):
    from paper_2505_14065_b200 import simplehash
    from paper_2505_14065_b200.sharedstate import StreamingHasher

    k = next(k for k in golden["hash"] if k["name"] == "rng2_64MiB")
    buf = _hash_input(k)
    assert simplehash(buf.tobytes()) == k["hash"]
    small = StreamingHasher(segment_bytes=1 << 20)  # many segments
    assert small.hash(buf) == k["hash"]
    assert small.hash(b"") == next(x["hash"] for x in golden["hash"] if x["name"] == "empty")


def test_llama_like_layout_scaled():
    """Many entries of very different sizes in one launch (config-4 shape, scaled)."""
    from paper_2505_14065_b200 import digest_entries
    from paper_2505_14065_b200.sharedstate import DType, SharedStateEntry

    rng = np.random.default_rng(9)
    shapes = [(1283, 64), (1283, 64)] + [(64, 64), (16, 64), (16, 64), (64, 64), (143, 64), (143, 64), (64, 143), (64,), (64,)] * 8
    entries = []
    host = []
    for i, sh in enumerate(shapes):
        t = torch.from_numpy(rng.normal(0, 1, int(np.prod(sh))).astype(np.float32)).to(torch.bfloat16).cuda()
        entries.append(SharedStateEntry(f"e{i}", DType.U8, t.view(torch.uint8)))
        host.append(t.view(torch.uint8).cpu().numpy())
    got = digest_entries(entries)
    want = osh.simplehash_many_c(host, threads=4)
    assert [h for _, _, h in got] == want


def test_one_bit_drift_detected():
    from paper_2505_14065_b200 import simplehash

    x = torch.randint(0, 256, (1 << 22,), dtype=torch.uint8, device="cuda")
    h0 = simplehash(x)
    x[123457] ^= 4
    assert simplehash(x) != h0


# sizes around the bitsliced kernel's block structure (5 warps x 1024-row
# segments per block): whole / partial last block, partial last segment,
# tail words and tail bytes
BIG_SIZES = [64 << 20, (64 << 20) + 1023, (64 << 20) + 3 * 1024 + 517, (65 << 20), (65 << 20) + 1,
             (66 << 20) + 4096 * 1024 - 1024, (67 << 20) + 7, (69 << 20) + 1024 * 1023 + 3]


@pytest.mark.parametrize("n", BIG_SIZES)
def test_big_entry_sizes(n):
    """Entries >= 64 MiB take the bitsliced big-entry kernel (loscan.cuh: lo
    chain by plane scans, hi chain affine): bit-exact against the oracle."""
    from paper_2505_14065_b200 import simplehash

    raw = np.random.default_rng(n).integers(0, 256, n, dtype=np.uint8)
    assert simplehash(to_dev(raw)) == osh.simplehash_c(raw)


def test_big_entry_structured_words():
    """All-zero, all-ones and alternating words: the carry planes of the
    bitsliced multiply see long runs of identical bits."""
    from paper_2505_14065_b200 import simplehash_many

    n = (65 << 20) + 12
    host = [np.zeros(n, np.uint8), np.full(n, 255, np.uint8),
            np.tile(np.array([0xAA, 0x55, 0xFF, 0x00], np.uint8), n // 4)]
    got = simplehash_many([to_dev(h) for h in host])
    assert got == osh.simplehash_many_c(host, threads=3)


def test_big_entry_unaligned_base_uses_batch_path():
    """A >= 64 MiB view at a byte offset (not 16-byte aligned, no TMA view):
    hashed by the batch kernel's direct loads, same digest as the oracle."""
    from paper_2505_14065_b200 import simplehash

    raw = np.random.default_rng(3).integers(0, 256, (64 << 20) + 9, dtype=np.uint8)
    dev = to_dev(raw)
    assert simplehash(dev[1:]) == osh.simplehash_c(raw[1:])


def test_big_entries_mixed_batch():
    """Two big entries beside many small ones in one call (config-4 shape):
    the big-entry kernel runs concurrently with the batch kernel."""
    from paper_2505_14065_b200 import simplehash_many

    rng = np.random.default_rng(77)
    sizes = [(96 << 20) + 12345, (80 << 20) + 4096] + [int(x) for x in rng.integers(1, 1 << 20, 60)]
    host = [rng.integers(0, 256, s, dtype=np.uint8) for s in sizes]
    got = simplehash_many([to_dev(h) for h in host])
    assert got == osh.simplehash_many_c(host, threads=8)


def test_big_entries_repeated_calls_stable():
    from paper_2505_14065_b200 import simplehash_many

    x = torch.randint(0, 256, (200 << 20,), dtype=torch.uint8, device="cuda")
    views = [x[: 150 << 20], x[150 << 20 :]]
    first = simplehash_many(views)
    for _ in range(3):
        assert simplehash_many(views) == first
    assert first[0] == osh.simplehash_c(views[0].cpu().numpy())
