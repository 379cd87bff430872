"""Parity at the BASELINE configs' full sizes (SURVEY §8c "oracle cost at
scale"): the whole config-4 shared state (291 entries, 16.06 GB, the
Llama-3-8B-like layout bench.py hashes) against the C oracle, and the
reduce/quantize schedules at config-2/3 chunk sizes against the streaming
per-chunk oracle (tests/mp_ring_worker.py, scenario "config")."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _host_free_bytes() -> int:
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def test_config4_full_layout_digests():
    """Every digest of the 16.06 GB config-4 state equals the oracle's."""
    from bench import llama3_8b_layout
    from oracle import simplehash as osh
    from paper_2505_14065_b200 import simplehash_many

    layout = llama3_8b_layout()
    total = sum(n for _, n in layout)
    nbytes = 2 * total
    if torch.cuda.mem_get_info()[0] < nbytes + (4 << 30) or _host_free_bytes() < nbytes + (8 << 30):
        pytest.skip("needs ~20 GB of device and host memory")
    state = torch.empty(total, dtype=torch.bfloat16, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(4)
    state.view(torch.int16).random_(-32768, 32767, generator=g)
    views, off = [], 0
    for _, n in layout:
        views.append(state[off : off + n])
        off += n
    got = simplehash_many(views)
    host = state.view(torch.uint8).cpu().numpy()
    del state, views
    torch.cuda.empty_cache()
    bufs, off = [], 0
    for _, n in layout:
        bufs.append(host[off : off + 2 * n])
        off += 2 * n
    # largest first keeps the two 1.05 GB entries from finishing last
    order = sorted(range(len(bufs)), key=lambda i: -bufs[i].size)
    want = osh.simplehash_many_c([bufs[i] for i in order], threads=os.cpu_count() or 8)
    exp = [0] * len(bufs)
    for i, h in zip(order, want):
        exp[i] = h
    assert got == exp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_ring_config_sizes(tmp_path):
    """W=2 (ranks share the GPU when the box has one): config-2 plain AVG of
    268 435 456 f32 and a u8 AVG with config-3's 150 M-element chunks; every
    rank checks its chunks against oracle.ring.reduce_chunk."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    world = 2
    cmd = [sys.executable, os.path.join(ROOT, "tests", "mp_ring_worker.py"), str(world), str(_free_port()),
           str(tmp_path), "config"]
    proc = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert proc.returncode == 0, proc.stderr[-4000:]
    failures, total = [], 0
    for r in range(world):
        with open(tmp_path / f"rank{r}.json") as f:
            res = json.load(f)
        assert not res["errors"], res["errors"][0]
        total += len(res["checks"])
        failures += [(r, c["name"], c["detail"]) for c in res["checks"] if not c["ok"]]
    assert total > 0
    assert not failures, failures[:20]
