"""GPU: bench.py's multi-rank path end to end under torchrun, as the driver
launches it for N > 1 — on ONE GPU. LRB_BENCH_SHARE_GPU=1 lets the ranks
share the device (they never wait on one another's kernels: the only
collectives are host-side gloo barriers and gathers), so this is a functional
test of the rank launch, the shard plan, the per-rank timing gather and the
JSON line; the line is tagged `shared_gpu_test` and its numbers mean nothing."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _torchrun(n, extra, timeout=600):
    env = dict(os.environ, LRB_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", str(n)] + extra
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, "rank 0 alone prints the line"
    return json.loads(lines[0])


def test_two_ranks_cfg4_under_torchrun():
    d = _torchrun(2, ["--steps", "3", "--warmup", "3", "--no-cpu", "--e2e-steps", "0"])
    assert d["n_gpus"] == 2 and d["shared_gpu_test"] is True and d["scaling"] == "strong"
    assert d["config"]["workload"] == "cfg4"
    shards = d["config"]["shards"]
    assert len(shards) == 2 and shards[0][0] == 0
    assert shards[0][0] + shards[0][1] == shards[1][0] and shards[1][0] + shards[1][1] == 8192
    per_rank = d["step_ms"]["per_rank"]
    assert [r["rank"] for r in per_rank] == [0, 1] and all(r["ms_median"] > 0 for r in per_rank)
    assert d["gpu_launches"] == 3 and d["value"] > 0 and d["roofline"]["bound"] == "tensor"


def test_reference_arm_under_torchrun_prints_once():
    d = _torchrun(2, ["--impl", "reference", "--steps", "1", "--warmup", "1", "--ref-seconds", "1"])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] in ("reference", "port")
