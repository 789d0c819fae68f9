"""Repeated runs of every refill form (producer warp / warpgroup, release
counter, deferred-wait row problem) stay bitwise identical
(tools/stress_determinism.py; the reference's determinism test,
tests/test_kernels.cpp:200-210, over many launches)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_repeated_runs_bitwise_identical():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stress_determinism.py"), "10"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("0 failures"), r.stdout + r.stderr
