"""GPU run_bench (reference bench.hpp:175-230; tests/test_harness.cpp:94-114):
the device run produces a consistent result row, with the reference's own
naive_multiply_batch as the baseline callable."""
import pytest

import oracle as O
from paper_2311_07602_b200 import bench_csv as BC

pytestmark = pytest.mark.gpu


def _ref_naive(batch, workers):
    O.ref_lowrank(0, batch.batch_size, batch.block_size, batch.rank_a, batch.a_vt_batch,
                  batch.b_u_batch, batch.a_x_batch, batch.b_x_batch, workers=workers)
    return O.ref_last_seconds()  # the driver alone


def test_run_bench_produces_a_consistent_result_row(ctx):
    cfg = BC.BenchConfig(batch_size=64, block_size=64, rank=8, workers=2, repetitions=3,
                         warmup_reps=1, seed=7)
    baseline = _ref_naive if O.ref_available() else None
    r = BC.run_bench(cfg, ctx=ctx, baseline=baseline)
    assert r.wall_seconds > 0.0
    assert r.gflops_rate == pytest.approx(BC.gflops(64, 8, 64, r.wall_seconds), rel=1e-12)
    phase_sum = r.pack_small_seconds + r.pack_skinny_seconds + r.kernel_seconds
    assert 0.0 <= phase_sum <= r.wall_seconds * 1.5 + 1e-3
    assert r.other_seconds >= 0.0
    assert r.kernel_device_seconds > 0.0 and r.h2d_seconds > 0.0 and r.d2h_seconds > 0.0
    assert r.gpu_launches == 1
    if baseline is not None:
        assert r.baseline_seconds > 0.0
        assert r.speedup == pytest.approx(r.baseline_seconds / r.wall_seconds, rel=1e-12)
    q = BC.parse_bench_csv_row(BC.bench_csv_row(r))
    assert q.batch_size == 64 and q.gpu_launches == 1 and q.device == r.device.replace(",", " ")


def test_write_csv(ctx, tmp_path):
    rows = [BC.run_bench(BC.BenchConfig(batch_size=100, block_size=128, rank=r, repetitions=2,
                                        run_baseline=False), ctx=ctx) for r in (8, 16)]
    path = tmp_path / "bench.csv"
    text = BC.write_csv(rows, str(path))
    lines = path.read_text().splitlines()
    assert lines[0] == BC.bench_csv_header() and len(lines) == 3 and text == path.read_text()
    assert [BC.parse_bench_csv_row(ln).rank for ln in lines[1:]] == [8, 16]
    assert all(BC.parse_bench_csv_row(ln).baseline_seconds == 0.0 for ln in lines[1:])
