"""CPU: the reference arm of bench.py (the reference's own CPU implementation,
oracle/_ref or the restatement) prints one contract-shaped JSON line; under
torchrun only rank 0 runs it."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=240):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable] + args, cwd=ROOT, capture_output=True, text=True,
                          timeout=timeout, env=e)


def test_reference_arm_json_line():
    r = _run(["bench.py", "--impl", "reference", "--config", "cfg1", "--steps", "2",
              "--warmup", "0", "--ref-seconds", "0.3", "--warmup-ref", "0"])
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "GFLOP/s" and d["value"] > 0
    assert d["higher_is_better"] is True and d["steps"] == 2
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"] == "cfg1"


def test_reference_arm_rank1_is_silent():
    env = {"RANK": "1", "WORLD_SIZE": "1", "LOCAL_RANK": "1"}
    r = _run(["bench.py", "--impl", "reference", "--config", "cfg1", "--steps", "1",
              "--warmup", "0"], env=env)
    assert r.returncode == 0
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
