"""Every kernel family once, bitwise vs the FMA-chain oracle, through
tools/sanitize_cases.py (the driver meant for compute-sanitizer, which is
closed on this pool)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_kernel_family_once():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("0 failures"), r.stdout + r.stderr


def test_every_kernel_family_without_pdl():
    # the same calls launched without programmatic dependent launch
    env = dict(os.environ, LRB_PDL="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0 and r.stdout.strip().endswith("0 failures"), r.stdout + r.stderr
