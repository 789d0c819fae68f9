"""CPU: the bench CSV and rate formulas (reference bench.hpp:20-170;
tests/test_harness.cpp:15-93), pinned against the reference binary's own
functions when oracle/_ref is built."""
import numpy as np
import pytest

import oracle as O
from paper_2311_07602_b200 import ParseError, ShapeError
from paper_2311_07602_b200 import bench_csv as BC


def _sample():
    # tests/test_harness.cpp:56-75
    return BC.BenchResult(10000, 1024, 8, 4, 5, 1, 42, 0.123456789, 5.4321, 20.125, 20.5, 0.01,
                          0.04, 0.06, 0.013456789, 0.5, 4.05, "NVIDIA B200", 0.002, 0.06, 0.001, 1)


def test_rate_formulas():
    # test_harness.cpp:15-45
    assert BC.gflops(1000, 8, 512, 1.0) == pytest.approx(1000 * (4 * 512 + 2 * 64 * 512) * 1e-9)
    b1 = BC.bandwidth_overlapped_gib_s(100, 8, 512, 1.0)
    b2 = BC.bandwidth_overlapped_gib_s(100, 8, 1024, 1.0)
    assert b2 - b1 == pytest.approx(100.0 * (2.0 * 8 * 512) * 8 / 1073741824.0, rel=1e-12)
    assert (BC.bandwidth_nonoverlapped_gib_s(100, 8, 512, 1.0) - b1 ==
            pytest.approx(100.0 * 64 * 8 / 1073741824.0, rel=1e-12))
    with pytest.raises(ShapeError):
        BC.bandwidth_overlapped_gib_s(1, 0, 1, 1.0)
    with pytest.raises(ShapeError):
        BC.gflops(1, 1, 1, 0.0)


def test_median_of():
    # test_harness.cpp:48-52
    assert BC.median_of([3.0, 1.0, 2.0]) == 2.0
    assert BC.median_of([4.0, 1.0, 2.0, 3.0]) == 2.5
    assert BC.median_of([7.0]) == 7.0
    assert BC.median_of([]) == 0.0


def test_csv_round_trip():
    # test_harness.cpp:55-93, extended by the device columns
    r = _sample()
    q = BC.parse_bench_csv_row(BC.bench_csv_row(r))
    assert (q.batch_size, q.block_size, q.rank, q.workers, q.seed) == (10000, 1024, 8, 4, 42)
    for f in ("wall_seconds", "gflops_rate", "speedup", "baseline_seconds", "h2d_seconds",
              "kernel_device_seconds", "d2h_seconds"):
        assert getattr(q, f) == pytest.approx(getattr(r, f), rel=1e-8)
    assert q.device == "NVIDIA B200" and q.gpu_launches == 1
    assert BC.bench_csv_header().count(",") == BC.bench_csv_row(r).count(",")
    with pytest.raises(ParseError, match="short CSV row"):
        BC.parse_bench_csv_row("1,2,3")
    with pytest.raises(ParseError, match="trailing fields"):
        BC.parse_bench_csv_row(BC.bench_csv_row(r) + ",7")


def test_reference_rows_parse():
    # a row written by the reference (17 fields) reads back with empty device columns
    ref17 = ",".join(BC.bench_csv_row(_sample()).split(",")[:17])
    q = BC.parse_bench_csv_row(ref17)
    assert q.batch_size == 10000 and q.device == "" and q.gpu_launches == 0


def test_first_17_columns_equal_the_reference_binary():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    r = _sample()
    assert BC.bench_csv_header().startswith(O.ref_bench_csv_header() + ",")
    vals = [r.batch_size, r.block_size, r.rank, r.workers, r.repetitions, r.warmup_reps, r.seed,
            r.wall_seconds, r.gflops_rate, r.bandwidth_overlapped, r.bandwidth_nonoverlapped,
            r.pack_small_seconds, r.pack_skinny_seconds, r.kernel_seconds, r.other_seconds,
            r.baseline_seconds, r.speedup]
    ours = BC.bench_csv_row(r).split(",")[:17]
    assert ",".join(ours) == O.ref_bench_csv_row(vals)
    rng = np.random.default_rng(3)
    for _ in range(20):
        vals[7:] = list(rng.uniform(0, 1e4, 10) * 10.0 ** rng.integers(-9, 3, 10))
        r2 = BC.BenchResult(*[int(v) for v in vals[:7]], *vals[7:])
        assert ",".join(BC.bench_csv_row(r2).split(",")[:17]) == O.ref_bench_csv_row(vals)


def test_rates_equal_the_reference_binary():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    for batch, rank, block, sec in ((20000, 8, 1024, 0.0123), (1, 1, 1, 1.0), (64, 32, 2048, 3.5)):
        want = O.ref_bench_rates(batch, rank, block, sec)
        got = (BC.gflops(batch, rank, block, sec),
               BC.bandwidth_overlapped_gib_s(batch, rank, block, sec),
               BC.bandwidth_nonoverlapped_gib_s(batch, rank, block, sec))
        assert got == pytest.approx(want, rel=1e-15)
    assert O.ref_bench_rates(1, 0, 1, 1.0) is None  # ShapeError in the reference too
    for vals in ([3.0, 1.0, 2.0], [4.0, 1.0, 2.0, 3.0], [7.0]):
        assert BC.median_of(vals) == O.ref_median_of(vals)
