"""The reference's benchmark harness and CSV rows, with device columns.

Mirrors proj/include/lrbatch/bench.hpp:20-230: the rate formulas
(``gflops``, ``bandwidth_overlapped_gib_s``, ``bandwidth_nonoverlapped_gib_s``),
``median_of``, ``BenchConfig`` / ``BenchResult``, the 17-column CSV
(``bench_csv_header`` / ``bench_csv_row`` / ``parse_bench_csv_row``) and
``run_bench``, which here times the paper's low-rank product on the GPU.

Column semantics on the device:

* ``wall_s`` is the median repetition of the reference-facing host call
  (``packed_multiply`` on a host ``LowRankBatch``). It includes H2D of the four
  roles, the kernel and D2H of G, exactly what a caller of the drop-in waits for.
* ``pack_small_s`` and ``pack_skinny_s`` are 0: the kernel reads the packed
  roles through TMA, and there is no packing phase.
* ``kernel_s`` is the device time of the same batch already resident in HBM
  (CUDA events, median of the repetitions). ``other_s`` is ``wall_s - kernel_s``
  (transfers and host overhead).
* ``baseline_s`` / ``speedup``: the reference runs naive_multiply_batch on the
  same batch. The product package has no CPU path, so the baseline is an
  optional callable supplied by the caller (tools pass the reference binary).
  Without one, both stay 0, as in the reference with run_baseline = false.

Five device columns follow the reference's 17: ``device``, ``h2d_s``,
``kernel_device_s``, ``d2h_s`` and ``gpu_launches``. ``parse_bench_csv_row``
reads both the reference's 17-field rows and the extended 22-field rows.
"""
from __future__ import annotations

import time
from dataclasses import dataclass
from typing import Callable, List, Optional

import numpy as np

from .lrbatch import Context, ParseError, ShapeError, default_context
from .lowrank import LowRankBatch, flops_per_item, packed_multiply

GIB = 1073741824.0


def gflops(batch_size: int, rank: int, block_size: int, seconds: float) -> float:
    """bench.hpp:21-26"""
    if not seconds > 0.0:
        raise ShapeError("gflops: seconds must be positive")
    return float(batch_size) * float(flops_per_item(rank, block_size)) / seconds * 1e-9


def bandwidth_overlapped_gib_s(batch_size: int, rank: int, block_size: int,
                               seconds: float) -> float:
    """read traffic only, (2r^2 + 2rb) words per item (bench.hpp:28-37)"""
    if not seconds > 0.0:
        raise ShapeError("bandwidth: seconds must be positive")
    if rank < 1:
        raise ShapeError("bandwidth: rank must be >= 1")
    words = 2.0 * rank * rank + 2.0 * rank * block_size
    return float(batch_size) * words * 8 / (seconds * GIB)


def bandwidth_nonoverlapped_gib_s(batch_size: int, rank: int, block_size: int,
                                  seconds: float) -> float:
    """adds the result write: (3r^2 + 2rb) words per item (bench.hpp:39-48)"""
    if not seconds > 0.0:
        raise ShapeError("bandwidth: seconds must be positive")
    if rank < 1:
        raise ShapeError("bandwidth: rank must be >= 1")
    words = 3.0 * rank * rank + 2.0 * rank * block_size
    return float(batch_size) * words * 8 / (seconds * GIB)


def median_of(values) -> float:
    """bench.hpp:82-88"""
    v = sorted(values)
    if not v:
        return 0.0
    mid = len(v) // 2
    return v[mid] if len(v) % 2 == 1 else 0.5 * (v[mid - 1] + v[mid])


@dataclass
class BenchConfig:
    """bench.hpp:90-106 (machine / plan_file do not apply on the GPU)"""

    batch_size: int = 10000
    block_size: int = 1024
    rank: int = 8
    workers: int = 1
    repetitions: int = 5
    warmup_reps: int = 1
    seed: int = 42
    output_path: str = ""
    run_baseline: bool = True

    def validate(self) -> None:
        if self.repetitions < 1:
            raise ShapeError("BenchConfig: repetitions must be >= 1")


@dataclass
class BenchResult:
    """bench.hpp:108-123, plus the device columns"""

    batch_size: int = 0
    block_size: int = 0
    rank: int = 0
    workers: int = 0
    repetitions: int = 0
    warmup_reps: int = 0
    seed: int = 0
    wall_seconds: float = 0.0
    gflops_rate: float = 0.0
    bandwidth_overlapped: float = 0.0
    bandwidth_nonoverlapped: float = 0.0
    pack_small_seconds: float = 0.0
    pack_skinny_seconds: float = 0.0
    kernel_seconds: float = 0.0
    other_seconds: float = 0.0
    baseline_seconds: float = 0.0
    speedup: float = 0.0
    # device columns
    device: str = ""
    h2d_seconds: float = 0.0
    kernel_device_seconds: float = 0.0
    d2h_seconds: float = 0.0
    gpu_launches: int = 0


_REF_COLUMNS = ("batch_size,block_size,rank,workers,repetitions,warmup_reps,seed,wall_s,gflops,"
                "bw_overlapped_gib_s,bw_nonoverlapped_gib_s,pack_small_s,pack_skinny_s,kernel_s,"
                "other_s,baseline_s,speedup")
_DEVICE_COLUMNS = "device,h2d_s,kernel_device_s,d2h_s,gpu_launches"


def bench_csv_header() -> str:
    """the reference's header (bench.hpp:125-129) + the device columns"""
    return _REF_COLUMNS + "," + _DEVICE_COLUMNS


def _g(x: float) -> str:
    return "%.9g" % x


def bench_csv_row(r: BenchResult) -> str:
    """bench.hpp:131-141 (%zu / %llu / %.9g) + the device columns"""
    ref = [str(int(r.batch_size)), str(int(r.block_size)), str(int(r.rank)), str(int(r.workers)),
           str(int(r.repetitions)), str(int(r.warmup_reps)), str(int(r.seed)),
           _g(r.wall_seconds), _g(r.gflops_rate), _g(r.bandwidth_overlapped),
           _g(r.bandwidth_nonoverlapped), _g(r.pack_small_seconds), _g(r.pack_skinny_seconds),
           _g(r.kernel_seconds), _g(r.other_seconds), _g(r.baseline_seconds), _g(r.speedup)]
    dev = [r.device.replace(",", " "), _g(r.h2d_seconds), _g(r.kernel_device_seconds),
           _g(r.d2h_seconds), str(int(r.gpu_launches))]
    return ",".join(ref + dev)


def parse_bench_csv_row(line: str) -> BenchResult:
    """bench.hpp:143-170: ParseError on a short row or trailing fields. Reads
    the reference's 17-field rows and this build's 22-field rows."""
    toks = line.rstrip("\r\n").split(",")
    if len(toks) < 17:
        raise ParseError("short CSV row: " + line)
    if len(toks) not in (17, 22):
        raise ParseError("trailing fields in CSV row: " + line)
    try:
        ints = [int(t) for t in toks[:7]]
        floats = [float(t) for t in toks[7:17]]
    except ValueError as e:
        raise ParseError(f"bad CSV field in row: {line} ({e})") from None
    r = BenchResult(*ints, *floats)
    if len(toks) == 22:
        try:
            r.device = toks[17]
            r.h2d_seconds, r.kernel_device_seconds, r.d2h_seconds = map(float, toks[18:21])
            r.gpu_launches = int(toks[21])
        except ValueError as e:
            raise ParseError(f"bad CSV field in row: {line} ({e})") from None
    return r


def _device_name(ctx: Context) -> str:
    import ctypes

    from .lrbatch import lib

    buf = ctypes.create_string_buffer(256)
    if lib.lrb_device_name(lib.lrb_ctx_device(ctx._h), buf, 256) == 0:
        return buf.value.decode()
    return "cuda"


def run_bench(config: BenchConfig, ctx: Optional[Context] = None,
              baseline: Optional[Callable[[LowRankBatch, int], None]] = None) -> BenchResult:
    """bench.hpp:175-230 on the GPU: a seeded LowRankBatch, warm-up, then the
    median of `repetitions` host calls of packed_multiply; the device-resident
    kernel time, H2D and D2H are measured separately (module docstring).
    `baseline(batch, workers)` runs the comparison (the reference's
    naive_multiply_batch) when config.run_baseline; when it returns a float,
    that is taken as its time."""
    config.validate()
    ctx = ctx or default_context()
    res = BenchResult(config.batch_size, config.block_size, config.rank, config.workers,
                      config.repetitions, config.warmup_reps, config.seed)
    batch = LowRankBatch.random(config.batch_size, config.block_size, config.rank, config.seed)
    n, b, r = config.batch_size, config.block_size, config.rank
    for _ in range(config.warmup_reps):
        packed_multiply(batch, ctx=ctx)
    walls: List[float] = []
    for _ in range(config.repetitions):
        t0 = time.perf_counter()
        packed_multiply(batch, ctx=ctx)
        walls.append(time.perf_counter() - t0)
    wall = median_of(walls)

    # device-resident kernel time and the transfer phases
    from .lowrank import lowrank_multiply_device

    roles = (batch.a_vt_batch, batch.b_u_batch, batch.a_x_batch, batch.b_x_batch)
    d_in = [ctx.empty(a.size) for a in roles]
    d_g = ctx.empty(batch.g_xy_batch.size)
    pins = [ctx.pinned(a.size) for a in roles]
    for p, a in zip(pins, roles):
        p.array[:] = a
    pin_g = ctx.pinned(batch.g_xy_batch.size)
    from .lrbatch import _check, lib

    h2d, d2h, kern = [], [], []
    s = ctx.stream()
    e0, e1 = ctx.event(), ctx.event()
    launches0 = ctx.launch_count
    for rep in range(config.repetitions + 1):
        t0 = time.perf_counter()
        for p, d in zip(pins, d_in):
            _check(lib.lrb_memcpy_h2d(ctx._h, d.ptr, p.ptr, p.nbytes), ctx._h)
        t1 = time.perf_counter()
        e0.record(s)
        lowrank_multiply_device(ctx, n, b, r, *d_in, d_g, stream=s)
        e1.record(s)
        s.synchronize()
        t2 = time.perf_counter()
        _check(lib.lrb_memcpy_d2h(ctx._h, pin_g.ptr, d_g.ptr, pin_g.nbytes), ctx._h)
        t3 = time.perf_counter()
        if rep:  # the first pass is a warm-up
            h2d.append(t1 - t0)
            kern.append(e0.elapsed_ms(e1) * 1e-3)
            d2h.append(t3 - t2)
    res.gpu_launches = (ctx.launch_count - launches0) // (config.repetitions + 1)
    res.wall_seconds = wall
    res.gflops_rate = gflops(n, r, b, wall)
    res.bandwidth_overlapped = bandwidth_overlapped_gib_s(n, r, b, wall)
    res.bandwidth_nonoverlapped = bandwidth_nonoverlapped_gib_s(n, r, b, wall)
    res.kernel_device_seconds = median_of(kern)
    res.kernel_seconds = res.kernel_device_seconds
    res.other_seconds = max(0.0, wall - res.kernel_seconds)
    res.h2d_seconds = median_of(h2d)
    res.d2h_seconds = median_of(d2h)
    res.device = _device_name(ctx)
    if config.run_baseline and baseline is not None:
        for _ in range(config.warmup_reps):
            baseline(batch, config.workers)
        bw = []
        for _ in range(config.repetitions):
            t0 = time.perf_counter()
            t = baseline(batch, config.workers)
            # a callable may report its own time (e.g. the driver alone,
            # without marshalling into the reference's containers)
            bw.append(float(t) if isinstance(t, float) else time.perf_counter() - t0)
        res.baseline_seconds = median_of(bw)
        res.speedup = res.baseline_seconds / res.wall_seconds
    return res


def write_csv(results, path: str = "") -> str:
    """header + one row per result, to `path` (or returned when empty)"""
    text = bench_csv_header() + "\n" + "".join(bench_csv_row(r) + "\n" for r in results)
    if path:
        with open(path, "w") as fh:
            fh.write(text)
    return text
