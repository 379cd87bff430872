"""Communicator facade on the NVLink data plane (one process per GPU): usage
errors before native calls, two tags in flight, parameter disagreement,
non-finite abort, shared-state resync (config 4: drifted peer, newcomer) and
churn (config 5: concurrent quantized all-reduces, a dropped peer, retry at
W-1 in a new ring order, rejoin + digest parity)."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3, 4])
def test_communicator(world, tmp_path):
    # fewer GPUs than ranks: ranks share devices over same-device CUDA IPC
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cmd = [sys.executable, os.path.join(ROOT, "tests", "mp_comm_worker.py"), str(world), str(_free_port()), str(tmp_path)]
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


@pytest.mark.parametrize("world", [3])
def test_communicator_config_scale(world, tmp_path):
    """Config 4 (16.06 GB state, one drifted peer, one sync) and config 5 (two
    concurrent 600 M-element u8 AVG all-reduces, a dropped peer) at size."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    free, _ = torch.cuda.mem_get_info()
    per_gpu_ranks = -(-world // torch.cuda.device_count())
    if free < per_gpu_ranks * 26 * (1 << 30):
        pytest.skip("needs ~26 GB of device memory per rank")
    cmd = [sys.executable, os.path.join(ROOT, "tests", "mp_comm_worker.py"), str(world), str(_free_port()),
           str(tmp_path), "sync_scale", "churn_scale"]
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
