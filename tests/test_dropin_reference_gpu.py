"""Drop-in under the reference's own control plane: the unmodified churncomm
MasterServer and client (installed from /root/reference into baseline/_ref by
pip) run config 1 with only the engine seam rebound to the
NVLink engine (tests/dropin_worker.py). Skipped when the
reference package is not installed."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_reference_master_drives_nvlink_engine(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not os.path.isdir(os.path.join(REF, "churncomm")):
        pytest.skip("reference package not installed in baseline/_ref")
    sys.path.insert(0, REF)
    try:
        from churncomm.master import MasterConfig, MasterServer
    finally:
        sys.path.remove(REF)
    server = MasterServer("127.0.0.1", 0, MasterConfig(pool_size=1, probe_bytes=64 * 1024, vote_timeout=15.0)).start()
    world = 2
    try:
        dport = _free_port()
        procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "dropin_worker.py"), str(r), str(world),
                                   str(server.port), str(dport), str(tmp_path)], cwd=ROOT,
                                  stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(world)]
        errs = []
        for p in procs:
            _, err = p.communicate(timeout=300)
            errs.append(err)
            assert p.returncode == 0, err[-3000:]
    finally:
        server.stop()
    failures, total = [], 0
    for r in range(world):
        with open(tmp_path / f"rank{r}.json") as f:
            res = json.load(f)
        assert not res["errors"], res["errors"][0]
        total += len(res["checks"])
        failures += [(r, c["name"], c["detail"]) for c in res["checks"] if not c["ok"]]
    assert total >= 9
    assert not failures, failures
