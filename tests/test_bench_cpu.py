"""bench.py's reference arm (the reference algorithm on host cores) keeps the
driver's JSON contract; runs on CPU."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("workload,world", [("allreduce", 2), ("quant", 4), ("async", 2), ("hash", 1)])
def test_reference_arm_json(workload, world):
    env = dict(os.environ, WORLD_SIZE=str(world), RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", workload,
                          "--gpus", str(world), "--steps", "1", "--warmup", "3"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "impl", "n_gpus", "cpu_baseline", "e2e", "higher_is_better"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["n_gpus"] == world
    cpu = line["cpu_baseline"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and cpu["kind"] in ("port", "reference")
    if cpu["kind"] == "reference":  # the reference's own ring beat the port: both are reported
        assert cpu["value"] == line["value"] and cpu["port"]["kind"] == "port" and cpu["value"] >= cpu["port"]["value"]
    own = line["cpu_baseline"].get("reference_own")
    if workload == "hash" and own is not None and "unavailable" not in own:
        # the reference's own simplehash, timed beside the port, agrees with it
        assert own["digests_equal_port"] and own["value"] > 0


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, WORLD_SIZE="2", RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and out.stdout.strip() == ""
